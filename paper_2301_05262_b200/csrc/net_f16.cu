// fp16 / bf16 hot path: the U-Net of network.forward (network.py:165-209)
// as level-fused tensor-core kernels, with the feature pass
// (raster.assemble_features, raster.py:266-278) fused into the level-0
// encoder so that the 4 feature planes never reach HBM.
//
//   enc0   features + space_to_depth + l0.enc3 + l0.enc1 + avg_pool2  (mma.sync)
//   lv<>   l1 enc / l2 enc / l3 bottleneck / l2 dec / l1 dec          (tcgen05)
//   dec0p  up2 + l0.dec3 + l0.dec1 + head, polyphase on the L1 grid    (tcgen05)
//   ring   the same for the outer level-0 ring (zero padding), fp32    (CUDA cores)
//   recon  bilinear(ch0) + depth_to_space(detail) + sigmoid, crop      (CUDA cores)
//
// Activations live in NHWC 16-bit tensors between kernels (L2-resident for
// a chunk of frames); inside a kernel they live in chunk-planar SMEM tiles
// (tc.cuh) so that every 3x3 tap of the implicit GEMM is an address offset,
// for ldmatrix rows and for UMMA descriptors alike.  Bias, ReLU, pooling,
// upsampling, skip sums, the head and the sigmoid run in fp32 registers.
#include <algorithm>
#include <atomic>
#include <type_traits>
#include <utility>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "net.cuh"
#include "prof.cuh"
#include "tc.cuh"

#include <cudaTypedefs.h>

namespace nsm {

namespace {

// ------------------------------------------------------------------ config
// Experiment switches (chunk size, PDL, the work-skipping attribution modes
// of enc0 / the level kernels, the dec0 ring, per-tile traces) exist only in
// builds with -DNSM_EXPERIMENTS (tools/); the release library ignores every
// NSM_* environment variable.
#ifdef NSM_EXPERIMENTS
constexpr bool kExp = true;
int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
}
#else
constexpr bool kExp = false;
int env_int(const char*, int dflt) { return dflt; }
#endif

// frames per pass through all levels (L2 residency vs. launch fill/drain)
int chunk_frames() {
    static int v = 0;
    if (!v) v = std::max(1, std::min(NSM_MAX_FRAMES_PER_LAUNCH, env_int("NSM_CHUNK_FRAMES", NSM_MAX_FRAMES_PER_LAUNCH)));
    return v;
}
// Kernel launches of the fused path go through launch_pdl: programmatic
// stream serialisation lets each kernel's prologue overlap its predecessor's
// tail (the kernels call pdl_trigger / pdl_wait).
bool pdl_enabled() {
    static int v = -1;
    if (v < 0) v = env_int("NSM_PDL", 1);
    return v != 0;
}

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// One-time per-device setup (cudaFuncSetAttribute applies to the current
// device only): true the first time it is asked for the current device.
struct PerDevice {
    std::atomic<uint64_t> done{0};
    bool first() {
        int dev = 0;
        cudaGetDevice(&dev);
        const uint64_t bit = 1ull << (dev & 63);
        return !(done.fetch_or(bit) & bit);
    }
};

constexpr int E0_TH = 16, E0_TW = 64;  // level-0 output tile (enc0 / dec0)
constexpr int E0_IR = E0_TH + 2, E0_IC = E0_TW + 2;
constexpr int E0_PLANE = plane_bytes(E0_IR * E0_IC, 2);
constexpr int E0_SMEM = 2 * E0_PLANE;
// TMA staging of the G-buffer for half a level-0 tile: 18 full-res rows x
// 132 columns x 7 fp32 planes (d, normal xyz, position xyz), double-buffered
// The TMA inner-dimension start must be 16-B aligned (measured: an fp32 box
// starting at x = -2 raises "illegal instruction", x = -4 works), so each
// staged row holds 136 columns starting 2 columns left of the halo.
constexpr int ST_ROWS = E0_IR, ST_COLS = 2 * E0_IC, ST_PIX = ST_ROWS * ST_COLS;
constexpr int ST_TCOLS = ST_COLS + 4, ST_TPIX = ST_ROWS * ST_TCOLS;
constexpr int ST_PLANE = ST_TPIX * 4;
constexpr int ST_TX = 7 * ST_PLANE;                       // bytes landed per half-tile
constexpr int round128(int v) { return (v + 127) / 128 * 128; }
constexpr int ST_OFF_N = round128(ST_PLANE);              // TMA destinations 128-B aligned
constexpr int ST_OFF_P = ST_OFF_N + round128(3 * ST_PLANE);
constexpr int ST_BYTES = round128(ST_OFF_P + 3 * ST_PLANE);
constexpr int ENC0_SMEM_TMA = 2 * E0_SMEM + 2 * ST_BYTES + 256;   // + 10 mbarriers, tile ring, bias ring
static_assert(E0_SMEM % 128 == 0, "stage base alignment");

struct GbufMaps {
    CUtensorMap d, n, p;   // (W, H, N) and (W, H, 3, N) fp32 tensor maps
};

// packed-weight formats (offsets into the plan's device block)
//  "frag": mma.sync B fragments, [tap][kk][nt][lane][2] u32
//  "umma": K-major core matrices, [tap][kk][2 chunks][N][8] elements
size_t frag_words(int taps, int cin, int cout) {
    return (size_t)taps * ((cin + 15) / 16) * ((cout + 7) / 8) * 64;
}

// l0.enc3 reads a tile whose channel k' = (2dy + dx) * 4 + c holds s2d
// channel 4c + 2dy + dx (space_to_depth, autodiff.py:290-308), so each
// full-resolution pixel writes its 4 features contiguously.
// With a 5th plane (cin4 = 20) the first 16 channels keep this order and
// channels 16-19 (the blocker plane's 2 x 2) follow in s2d order.
int perm_s2d(int kp, int cin4) {
    if ((cin4 != 16 && cin4 != 20) || kp >= 16) return kp;
    return 4 * (kp % 4) + kp / 4;
}

template <typename T>
uint16_t to_bits(float v) {
    T h = (T)v;
    return *reinterpret_cast<uint16_t*>(&h);
}

template <typename T>
void pack_frag(const float* w, int cout, int cin, int k, bool s2d_perm, std::vector<uint32_t>& out,
               float scale = 1.f) {
    const int taps = k * k, KK = (cin + 15) / 16, NT = (cout + 7) / 8;
    out.assign(frag_words(taps, cin, cout), 0u);
    auto B = [&](int tap, int kk, int n) -> float {
        if (n >= cout || kk >= cin) return 0.f;
        const int ci = s2d_perm ? perm_s2d(kk, cin) : kk;
        return scale * w[((size_t)n * cin + ci) * taps + tap];
    };
    for (int tap = 0; tap < taps; ++tap)
        for (int kk = 0; kk < KK; ++kk)
            for (int nt = 0; nt < NT; ++nt)
                for (int l = 0; l < 32; ++l) {
                    const int g = l >> 2, t = l & 3, n = nt * 8 + g, k0 = kk * 16 + 2 * t;
                    const size_t o = ((((size_t)tap * KK + kk) * NT + nt) * 32 + l) * 2;
                    out[o] = to_bits<T>(B(tap, k0, n)) | ((uint32_t)to_bits<T>(B(tap, k0 + 1, n)) << 16);
                    out[o + 1] = to_bits<T>(B(tap, k0 + 8, n)) | ((uint32_t)to_bits<T>(B(tap, k0 + 9, n)) << 16);
                }
}

template <typename T>
void pack_umma(const float* w, int cout, int cin, int k, std::vector<uint16_t>& out) {
    const int taps = k * k, KK = cin / 16;
    out.assign((size_t)taps * cin * cout, 0);
    for (int tap = 0; tap < taps; ++tap)
        for (int kk = 0; kk < KK; ++kk)
            for (int c = 0; c < 2; ++c)
                for (int n = 0; n < cout; ++n)
                    for (int e = 0; e < 8; ++e) {
                        const int ci = kk * 16 + c * 8 + e;
                        out[((((size_t)tap * KK + kk) * 2 + c) * cout + n) * 8 + e] =
                            to_bits<T>(w[((size_t)n * cin + ci) * taps + tap]);
                    }
}

// Tile decode without integer division: q = (n * ceil(2^32 / d)) >> 32 is
// floor(n / d) whenever n * d < 2^32 (tiles and tiles-per-frame < 2^16);
// the multiplier is 2^32 itself for d = 1, hence 64-bit.
struct TileDiv {
    int nx, nxy;
    uint64_t mnx, mnxy;
};

__host__ __device__ inline TileDiv tile_div(int H0, int W0) {
    TileDiv d;
    d.nx = (W0 + E0_TW - 1) / E0_TW;
    d.nxy = d.nx * ((H0 + E0_TH - 1) / E0_TH);
    d.mnx = 0xFFFFFFFFull / (uint64_t)d.nx + 1ull;
    d.mnxy = 0xFFFFFFFFull / (uint64_t)d.nxy + 1ull;
    return d;
}

// ------------------------------------------------------------- level 0 (mma.sync)
struct Enc0Args {
    GBufK g;
    const float* sm;
    int64_t sm_stride;
    FrameTable tab;
    const float* x;       // features (N, 4, H0*2, W0*2) fp32 when not from the G-buffer
    int h, w;             // frame pixels actually present (rows/cols beyond are padding)
    int H0, W0;           // level-0 dims (padded frame / 2)
    const uint2* wb3;     // l0.enc3 fragments [9][2 nt][32]
    const uint2* wb1;     // l0.enc1 fragments [2 nt][32]
    const float* b3;
    const float* b1;
    void* out;            // pooled (N, H0/2, W0/2, 16)
    int64_t* first_bad;
    int32_t* tidx;        // parity hook (nullable): (N, 2, h, w) texel (row, col) of covered pixels
    int dbg;              // experiments only: 1 skip feature math, 2 skip convolutions
    TileDiv td;           // tile decode constants (host-computed, read from the param bank)
    long long* trace;     // experiments only (NSM_ENC0_TRACE): per-CTA globaltimer start / end
    int* tile_ctr;        // TMA kernel: [0] tiles claimed beyond the first round, [1] CTAs done
                          // claiming (zeroed by fill_first_bad; the last CTA re-zeroes both)
};

__device__ __forceinline__ long long globaltimer_ns() {
    long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Stage-1 per-pixel math of the fused kernel: fp64 projection for the texel
// index (bit-exact np.rint), fp32 for the rest (the values are rounded to
// 16 bits right after).  Returns ch0..ch3 (raster.py:262, 272-276).
__device__ __forceinline__ float4 pixel_features(const FrameK& F, const GBufK& g, const float* sm,
                                                 int64_t base, int64_t pix, int fy, int fx,
                                                 int64_t hw, int64_t* first_bad) {
    const float* dp = reinterpret_cast<const float*>(g.d);
    const float d = __ldg(dp + base + pix);
    if (!(d > 0.f)) return make_float4(0.f, 0.f, 0.f, 0.f);
    const float* P = reinterpret_cast<const float*>(g.position) + 3 * base + pix;
    const float* Nn = reinterpret_cast<const float*>(g.normal) + 3 * base + pix;
    const float px = __ldg(P), py = __ldg(P + hw), pz = __ldg(P + 2 * hw);
    const float nx = __ldg(Nn), ny = __ldg(Nn + hw), nz = __ldg(Nn + 2 * hw);
    int ri, ci;
    if (!texel_of(F, px, py, pz, ri, ci)) atomic_min_i64(first_bad, pix);
    const float look = __ldg(sm + (int64_t)ri * F.ws + ci);
    const float tx = (float)(F.ec[0] - (double)px), ty = (float)(F.ec[1] - (double)py),
                tz = (float)(F.ec[2] - (double)pz);
    const float zf = sqrtf(tx * tx + ty * ty + tz * tz);
    const float ce = fminf(fmaxf((nx * tx + ny * ty + nz * tz) / zf, 0.f), 1.f);
    const float u = ((fx + 0.5f) / F.cw * 2.f - 1.f) * (float)F.half_w;
    const float v = (1.f - (fy + 0.5f) / F.ch * 2.f) * (float)F.half_h;
    const float rx = (float)F.cf[0] + u * (float)F.cr[0] + v * (float)F.cu[0];
    const float ry = (float)F.cf[1] + u * (float)F.cr[1] + v * (float)F.cu[1];
    const float rz = (float)F.cf[2] + u * (float)F.cr[2] + v * (float)F.cu[2];
    const float cc = fminf(fmaxf(-(nx * rx + ny * ry + nz * rz) * rsqrtf(rx * rx + ry * ry + rz * rz), 0.f), 1.f);
    float ch0 = 0.f, ch1 = 1.f;
    if (isfinite(look)) {
        const float m = fminf(look, zf);
        ch0 = (m - zf) + (float)F.bias;
        ch1 = (m + (float)F.bias) / zf;
    }
    return make_float4(ch0, ch1, ce + (float)F.size_index, cc / d);
}

// Sliding-window 3x3 conv on a 16-pixel strip: every input row's three
// dx-shifted A fragments are loaded once and applied to the three output
// rows that need them, so ldmatrix traffic is 3 instead of 9 loads per row.
// Accumulators start at the conv bias (saves the epilogue's bias adds).
struct NoRowHook {
    __device__ void operator()(int) const {}
};

// hook(ir) runs before input row ir is read (e.g. to wait for the producers
// to finish the half of the tile that holds it).  kPairRows maps MMA row r
// to strip pixel 2r (r < 8) / 2(r-8)+1, so each thread's accumulator holds
// the horizontal neighbours 2g, 2g+1 (a 2x2 pool needs no shuffles).
template <typename T, int ROWS, bool kPairRows = false, class Epi, class Hook = NoRowHook>
__device__ __forceinline__ void conv3_strip16(uint32_t sbase, int plane, int rowpix, int r0, int sx,
                                              const uint32_t (&B3)[9][2][2], const float (&binit)[2][2],
                                              Epi&& epi, Hook&& hook = Hook{}) {
    const int lane = threadIdx.x & 31;
    const int lm = lane >> 3, li = lane & 7;
    const uint32_t a_off = (lm >> 1) * plane + (kPairRows ? 2 * li + (lm & 1) : li + 8 * (lm & 1)) * 16;
    float acc[3][2][4];
    // A fragments double-buffered: row ir+1 is loaded before row ir's MMAs
    uint32_t Ab[2][3][4];
    auto load_row = [&](int ir, uint32_t (&A)[3][4]) {
        hook(ir);
#pragma unroll
        for (int dx = 0; dx < 3; ++dx)
            ldsm_x4(sbase + a_off + ((r0 + ir) * rowpix + sx + dx) * 16, A[dx]);
    };
    load_row(0, Ab[0]);
#pragma unroll
    for (int ir = 0; ir < ROWS + 2; ++ir) {
        if (ir + 1 < ROWS + 2) load_row(ir + 1, Ab[(ir + 1) & 1]);
        uint32_t (&A)[3][4] = Ab[ir & 1];
        // dx outer, (ky, n) inner: consecutive MMAs go to up to 6 different
        // accumulators, so no MMA waits on the one just issued
#pragma unroll
        for (int dx = 0; dx < 3; ++dx)
#pragma unroll
            for (int ky = 0; ky < 3; ++ky) {
                const int oo = ir - ky;
                if (oo >= 0 && oo < ROWS) {
#pragma unroll
                    for (int n = 0; n < 2; ++n) {
                        if (ky == 0 && dx == 0)          // first tap of output row oo: C = bias
                            mma16816_c<T>(acc[oo % 3][n], A[dx], B3[ky * 3 + dx][n][0], B3[ky * 3 + dx][n][1],
                                          binit[n][0], binit[n][1], binit[n][0], binit[n][1]);
                        else
                            mma16816<T>(acc[oo % 3][n], A[dx], B3[ky * 3 + dx][n][0], B3[ky * 3 + dx][n][1]);
                    }
                }
            }
        if (ir >= 2) {
            const int oo = ir - 2;
            epi(oo, acc[oo % 3]);
        }
    }
}

// relu(acc) of a 16x16 m16n8 pair packed to 16 bits (ReLU after the rounding:
// the two commute), as the A fragment of the next 1x1 conv.
template <typename T>
__device__ __forceinline__ void relu_pack_a(const float (&acc)[2][4], uint32_t a[4]) {
    a[0] = Elem<T>::relu2(Elem<T>::pack(acc[0][0], acc[0][1]));
    a[1] = Elem<T>::relu2(Elem<T>::pack(acc[0][2], acc[0][3]));
    a[2] = Elem<T>::relu2(Elem<T>::pack(acc[1][0], acc[1][1]));
    a[3] = Elem<T>::relu2(Elem<T>::pack(acc[1][2], acc[1][3]));
}

// relu(acc + bias) of a 16x16 m16n8 pair, packed as the A fragment of the
// next 1x1 conv (accumulator layout == A-operand layout).
template <typename T>
__device__ __forceinline__ void acc_to_a(const float (&acc)[2][4], const float (&bias)[2][2], bool relu,
                                         uint32_t a[4]) {
    float v[2][4];
#pragma unroll
    for (int n = 0; n < 2; ++n)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            v[n][e] = acc[n][e] + bias[n][e & 1];
            if (relu) v[n][e] = fmaxf(v[n][e], 0.f);
        }
    a[0] = Elem<T>::pack(v[0][0], v[0][1]);
    a[1] = Elem<T>::pack(v[0][2], v[0][3]);
    a[2] = Elem<T>::pack(v[1][0], v[1][1]);
    a[3] = Elem<T>::pack(v[1][2], v[1][3]);
}

__device__ __forceinline__ void nbar_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Persistent, warp-specialised level-0 kernels: warps 0-7 produce the
// halo'd input tile of the next tile into one of two SMEM buffers while
// warps 8-15 run the tensor-core convolutions on the other.  Named barriers
// 1/2 = buffer full, 3/4 = buffer empty.
constexpr int kL0Threads = 512, kL0Prod = 256;

template <class Produce>
__device__ __forceinline__ void l0_produce_loop(int total, Produce&& produce) {   // all 512 threads meet at 1-4
    extern __shared__ __align__(128) uint8_t smem[];
    for (int k = 0;; ++k) {
        const int tile = blockIdx.x + k * gridDim.x;
        if (tile >= total) break;
        const int s = k & 1;
        if (k >= 2) nbar_sync(3 + s, kL0Threads);
        produce(smem + s * E0_SMEM, tile);
        nbar_arrive(1 + s, kL0Threads);
    }
}

template <int NT = kL0Threads, class Consume>
__device__ __forceinline__ void l0_consume_loop(int total, Consume&& consume) {
    extern __shared__ __align__(128) uint8_t smem[];
    for (int k = 0;; ++k) {
        const int tile = blockIdx.x + k * gridDim.x;
        if (tile >= total) break;
        const int s = k & 1;
        nbar_sync(1 + s, NT);
        consume(smem + s * E0_SMEM, tile);
        if (tile + 2 * (int)gridDim.x < total) nbar_arrive(3 + s, NT);
    }
}

struct L0Tile {
    int f, ty0, tx0;
};

__device__ __forceinline__ L0Tile l0_tile(int tile, int H0, int W0) {
    const int nx = (W0 + E0_TW - 1) / E0_TW, ny = (H0 + E0_TH - 1) / E0_TH;
    L0Tile t;
    t.tx0 = (tile % nx) * E0_TW;
    t.ty0 = ((tile / nx) % ny) * E0_TH;
    t.f = tile / (nx * ny);
    return t;
}

__device__ __forceinline__ L0Tile l0_tile(int tile, const TileDiv& d) {
    L0Tile t;
    t.f = (int)(((uint64_t)(uint32_t)tile * d.mnxy) >> 32);
    const int r = tile - t.f * d.nxy;
    const int ty = (int)(((uint64_t)(uint32_t)r * d.mnx) >> 32);
    t.ty0 = ty * E0_TH;
    t.tx0 = (r - ty * d.nx) * E0_TW;
    return t;
}

// Features of a halo'd level-0 tile, s2d-packed: 4 full-resolution pixels
// per thread per batch, all G-buffer loads issued before any use.
template <typename T, bool kFromGBuffer>
__device__ __forceinline__ void produce_features(const Enc0Args& a, uint8_t* buf, const L0Tile& tl) {
    constexpr int RC = 2 * E0_IC, NPX = 2 * E0_IR * RC, K = 4;
    const int ptid = threadIdx.x;
    const int64_t hw = (int64_t)a.h * a.w;
    const int64_t base = (int64_t)tl.f * a.g.frame_stride;
    const float* gd = reinterpret_cast<const float*>(a.g.d) + base;
    const float* gp = reinterpret_cast<const float*>(a.g.position) + 3 * base;
    const float* gn = reinterpret_cast<const float*>(a.g.normal) + 3 * base;
    for (int i0 = ptid; i0 < NPX; i0 += kL0Prod * K) {
        float d[K], px[K], py[K], pz[K], nx[K], ny[K], nz[K];
        int fy[K], fx[K];
        bool in[K];
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const int i = i0 + j * kL0Prod;
            const int ry = i / RC, rx = i - ry * RC;
            fy[j] = 2 * (tl.ty0 - 1) + ry;
            fx[j] = 2 * (tl.tx0 - 1) + rx;
            in[j] = i < NPX && fy[j] >= 0 && fx[j] >= 0 && fy[j] < a.h && fx[j] < a.w;
            d[j] = px[j] = py[j] = pz[j] = nx[j] = ny[j] = nz[j] = 0.f;
            if (in[j]) {
                const int64_t pix = (int64_t)fy[j] * a.w + fx[j];
                if (kFromGBuffer) {
                    d[j] = __ldg(gd + pix);
                    px[j] = __ldg(gp + pix);
                    py[j] = __ldg(gp + hw + pix);
                    pz[j] = __ldg(gp + 2 * hw + pix);
                    nx[j] = __ldg(gn + pix);
                    ny[j] = __ldg(gn + hw + pix);
                    nz[j] = __ldg(gn + 2 * hw + pix);
                } else {
                    const float* xp = a.x + (int64_t)tl.f * 4 * hw + pix;
                    px[j] = __ldg(xp);
                    py[j] = __ldg(xp + hw);
                    pz[j] = __ldg(xp + 2 * hw);
                    nx[j] = __ldg(xp + 3 * hw);
                }
            }
        }
        float4 v[K];
        if (kFromGBuffer) {
            const FrameK& F = a.tab.f[tl.f];
            const float* smf = a.sm + tl.f * a.sm_stride;
            float look[K];
#pragma unroll
            for (int j = 0; j < K; ++j) {
                look[j] = 0.f;
                if (d[j] > 0.f) {
                    int ri, ci;
                    if (!texel_of(F, px[j], py[j], pz[j], ri, ci))
                        atomic_min_i64(a.first_bad + tl.f, (int64_t)fy[j] * a.w + fx[j]);
                    look[j] = __ldg(smf + (int64_t)ri * F.ws + ci);
                    if (a.tidx) {
                        int32_t* ti = a.tidx + (int64_t)tl.f * 2 * hw + (int64_t)fy[j] * a.w + fx[j];
                        ti[0] = ri;
                        ti[hw] = ci;
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < K; ++j) {
                v[j] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (d[j] > 0.f) {
                    const float tx = (float)(F.ec[0] - (double)px[j]), ty = (float)(F.ec[1] - (double)py[j]),
                                tz = (float)(F.ec[2] - (double)pz[j]);
                    const float izf = rsqrtf(tx * tx + ty * ty + tz * tz);
                    const float zf = 1.f / izf;
                    const float ce = fminf(fmaxf((nx[j] * tx + ny[j] * ty + nz[j] * tz) * izf, 0.f), 1.f);
                    const float u = ((fx[j] + 0.5f) / F.cw * 2.f - 1.f) * (float)F.half_w;
                    const float w = (1.f - (fy[j] + 0.5f) / F.ch * 2.f) * (float)F.half_h;
                    const float rx = (float)F.cf[0] + u * (float)F.cr[0] + w * (float)F.cu[0];
                    const float ry = (float)F.cf[1] + u * (float)F.cr[1] + w * (float)F.cu[1];
                    const float rz = (float)F.cf[2] + u * (float)F.cr[2] + w * (float)F.cu[2];
                    const float cc = fminf(fmaxf(-(nx[j] * rx + ny[j] * ry + nz[j] * rz) *
                                                     rsqrtf(rx * rx + ry * ry + rz * rz), 0.f), 1.f);
                    float ch0 = 0.f, ch1 = 1.f;
                    if (isfinite(look[j])) {                    // raster.py:262
                        const float m = fminf(look[j], zf);
                        ch0 = (m - zf) + (float)F.bias;
                        ch1 = (m + (float)F.bias) * izf;
                    }
                    v[j] = make_float4(ch0, ch1, ce + (float)F.size_index, cc / d[j]);
                }
            }
        } else {
#pragma unroll
            for (int j = 0; j < K; ++j) v[j] = make_float4(px[j], py[j], pz[j], nx[j]);
        }
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const int i = i0 + j * kL0Prod;
            if (i < NPX) {
                const int ry = i / RC, rx = i - ry * RC;
                const int p = (ry >> 1) * E0_IC + (rx >> 1);
                *reinterpret_cast<uint2*>(buf + (ry & 1) * E0_PLANE + p * 16 + (rx & 1) * 8) =
                    make_uint2(Elem<T>::pack(v[j].x, v[j].y), Elem<T>::pack(v[j].z, v[j].w));
            }
        }
    }
}

// TMA producer: one elected thread streams half-tiles of the seven G-buffer
// planes into two SMEM stages (mbarrier complete_tx); the producer warps turn
// each staged half into features while the next half is in flight.
// Each producer thread owns 4 pixels of one staged row of a half-tile:
// threads 0-575 an interior quad (halo cols 4k-2 .. 4k+1, k = 1..32: level-0
// pixels 2k-1 and 2k), warp 18 the row's two edge pairs (halo cols 0,1 and
// 130,131: level-0 pixels 0 and 65).  A half is then one vectorised pass
// (LDS.128 per plane) over 18 x 33 threads with all index math hoisted.
// Warp roles: 0-18 feature producers, 19 the TMA issuer, 20-23 tensor-core
// consumers.  All hand-offs are mbarriers with one arrival per warp, so a
// warp only ever waits for the data it needs, never for its peers:
//   full[s]     TMA -> producers       (complete_tx: staged half-tile landed)
//   empty[s]    producers -> TMA       (19 arrivals: stage s read by phase A)
//   half[b][h]  producers -> consumers (19: rows of half h of tile buffer b)
//   freed[b]    consumers -> producers (4: tile buffer b consumed)
// The TMA thread also picks the tiles: blockIdx.x first, then one global
// counter (tiles differ in cost with their coverage, and static round-robin
// left the slowest CTA 14 % above the mean); the k-th tile's index goes into
// a shared ring (tring[k & 7], -1 = none) that the producers read after
// full[] and the consumers after half[].
// setmaxnreg moves registers from the producer/TMA warps (-> 72) to the MMA
// warps (-> 112); the budget is checked against the kernel's launch
// register count on the host (run_l0).
constexpr int kE0Feat = 608, kE0Prod = 640, kE0Threads = 768;
constexpr int kE0FeatWarps = kE0Feat / 32, kE0MmaWarps = (kE0Threads - kE0Prod) / 32;
constexpr int kE0ProdRegs = 72, kE0MmaRegs = 112;
constexpr int ST_QC = E0_TW / 2;                     // interior quads per staged row (32)
static_assert(ST_ROWS * (ST_QC + 1) <= kE0Feat, "one quad per producer thread per half-tile");
static_assert(ST_ROWS * ST_QC % 32 == 0, "edge threads form their own warp");
static_assert(ST_ROWS % 2 == 0, "a half-tile holds whole level-0 rows");

// Per-quad producer state carried from the A to the B phase of a half-tile:
// the gathered occluder depth (< 0: uncovered).  Phase A already writes
// (ch2, ch3) into the tile and parks z_f (fp32) in the (ch0, ch1) slot.
struct QuadRegs {
    float look[4];
};

// Phase-A results bound for the tile buffer: (z_f, (ch2, ch3)) per pixel.
// A tile's first half parks them in registers until the consumers release
// the buffer, so that waiting never delays the previous tile's last half.
struct QuadPark {
    uint2 v[4];
};

template <typename T, bool kIdx>
__device__ __forceinline__ void produce_features_tma(const Enc0Args& a, const GbufMaps& tm, int total) {
    // Software pipeline over half-tiles q (two per tile):
    //   A(q): staged planes -> texel (fp64), z_f, (c_e + s, c_c / d) packed,
    //         the shadow-map gather issued (LDG in flight)
    //   TMA(q+2) into the stage A(q) just released
    //   B(q-1): gathered occluder depth -> ch0, ch1, pack, STS into the
    //         tile's feature buffer
    // so the gather latency of half q overlaps B(q-1) and A(q+1), and the
    // G-buffer of half q+2 streams in meanwhile.
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* stage = smem + 2 * E0_SMEM;
    uint64_t* full = reinterpret_cast<uint64_t*>(stage + 2 * ST_BYTES);
    uint64_t* empty = full + 2;
    uint64_t* half = full + 4;     // [buffer][half]
    uint64_t* freed = full + 8;
    int* tring = reinterpret_cast<int*>(full + 10);   // tile of the CTA's k-th tile (k & 7), -1: none
    float* tbias = reinterpret_cast<float*>(full + 14);   // and its frame's shadow bias (phase B)
    const int ptid = threadIdx.x;
    const int lane = ptid & 31;
    if (ptid >= kE0Feat) {                         // TMA warp
        if (lane == 0) {
            const uint64_t pol = l2_evict_first_policy();      // the G-buffer is read once
            // The CTA's tiles: the first is blockIdx.x, the rest come from
            // one counter, claimed when the tile is due (claiming earlier
            // balances worse: measured), so CTAs whose tiles turn out cheap
            // (uncovered) take more of them
            int cur = -1;
            for (int q = 0;; ++q) {
                const int sidx = q & 1;
                if (q >= 2) mbar_wait(&empty[sidx], ((q - 2) >> 1) & 1);
                if (!(q & 1)) {
                    const int k = q >> 1;
                    if (k == 0) {
                        cur = blockIdx.x;                        // grid <= total
                    } else {
                        if (k == 1) pdl_wait();                  // the counter was zeroed by fill_first_bad
                        cur = (int)gridDim.x + atomicAdd(a.tile_ctr, 1);
                        if (cur >= total) cur = -1;
                    }
                    tring[k & 7] = cur;
                    if (cur >= 0) tbias[k & 7] = a.tab.f[l0_tile(cur, a.td).f].fbias;
                    if (cur < 0) {
                        mbar_arrive(&full[sidx]);                // no data: the producers read the sentinel
                        // the last CTA done claiming re-zeroes the counters for the next launch
                        if (atomicAdd(a.tile_ctr + 1, 1) == (int)gridDim.x - 1) {
                            a.tile_ctr[0] = 0;
                            a.tile_ctr[1] = 0;
                        }
                        break;
                    }
                }
                const L0Tile tl = l0_tile(cur, a.td);
                const uint32_t dst = smem_u32(stage + sidx * ST_BYTES);
                const int x = 2 * tl.tx0 - 4, y = 2 * tl.ty0 - 2 + ST_ROWS * (q & 1);
                mbar_expect_tx(&full[sidx], ST_TX);
                tma_load_3d_stream(dst, &tm.d, x, y, tl.f, &full[sidx], pol);
                tma_load_4d_stream(dst + ST_OFF_N, &tm.n, x, y, 0, tl.f, &full[sidx], pol);
                tma_load_4d_stream(dst + ST_OFF_P, &tm.p, x, y, 0, tl.f, &full[sidx], pol);
            }
        }
        return;
    }
    // tile-invariant geometry of this thread's 4 pixels: halo columns
    // hc_lo + {0, 1} (level-0 halo pixel lo) and hc_hi + {0, 1} (pixel hi)
    const bool edge = ptid >= ST_ROWS * ST_QC;
    const bool active = ptid < ST_ROWS * (ST_QC + 1);
    const int qy = edge ? ptid - ST_ROWS * ST_QC : ptid / ST_QC;
    const int qk = edge ? 0 : ptid - qy * ST_QC + 1;
    const int px_lo = edge ? 0 : 2 * qk - 1, px_hi = edge ? E0_IC - 1 : 2 * qk;
    // staged col = halo col + 2; halo col of pixel e: 2 px + (e & 1)
    const int lds_lo = qy * ST_TCOLS * 4 + 8 + 8 * px_lo, lds_hi = qy * ST_TCOLS * 4 + 8 + 8 * px_hi;
    const int sts_row = (qy & 1) * E0_PLANE + (qy >> 1) * E0_IC * 16;
    const int slot_lo = sts_row + px_lo * 16, slot_hi = sts_row + px_hi * 16;
    auto park = [&](int q, const QuadPark& P) {
        if (!active) return;
        uint8_t* tdst = smem + ((q >> 1) & 1) * E0_SMEM + (q & 1) * (ST_ROWS / 2) * E0_IC * 16;
#pragma unroll
        for (int e = 0; e < 4; ++e)
            *reinterpret_cast<uint2*>(tdst + (e < 2 ? slot_lo : slot_hi) + (e & 1) * 8) = P.v[e];
    };
    auto phaseA = [&](int q, int tile, QuadRegs& R, QuadPark& P) {
        const L0Tile tl = l0_tile(tile, a.td);
        const int sidx = q & 1;
        if (!active) return;
        const FrameK& F = a.tab.f[tl.f];
        // 32-bit texel index: NSM_MAX_FRAMES_PER_LAUNCH maps of <= 2^26 texels
        const int sm_off = tl.f * (int)a.sm_stride;
        const uint8_t* sb = stage + sidx * ST_BYTES;
        float dv[4], xv[4], yv[4], zv[4], nxv[4], nyv[4], nzv[4];
        auto ld4 = [&](int off, float (&v)[4]) {
            if (!edge) {                                   // warp-uniform
                const float4 t = *reinterpret_cast<const float4*>(sb + off + lds_lo);
                v[0] = t.x, v[1] = t.y, v[2] = t.z, v[3] = t.w;
            } else {
                const float2 l = *reinterpret_cast<const float2*>(sb + off + lds_lo);
                const float2 r = *reinterpret_cast<const float2*>(sb + off + lds_hi);
                v[0] = l.x, v[1] = l.y, v[2] = r.x, v[3] = r.y;
            }
        };
        ld4(0, dv);
        if (!(dv[0] > 0.f || dv[1] > 0.f || dv[2] > 0.f || dv[3] > 0.f)) {   // nothing covered
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                R.look[e] = -1.f;
                P.v[e] = make_uint2(0u, 0u);
            }
            return;
        }
        ld4(ST_OFF_P, xv);
        ld4(ST_OFF_P + ST_PLANE, yv);
        ld4(ST_OFF_P + 2 * ST_PLANE, zv);
        ld4(ST_OFF_N, nxv);
        ld4(ST_OFF_N + ST_PLANE, nyv);
        ld4(ST_OFF_N + 2 * ST_PLANE, nzv);
        const float ecx = F.fec[0], ecy = F.fec[1], ecz = F.fec[2];
        const float cpx = F.fcp[0], cpy = F.fcp[1], cpz = F.fcp[2];
        const float size = F.fsize;
        const int ws = F.ws;
        int bad = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float d = dv[e], px = xv[e], py = yv[e], pz = zv[e];
            const bool cov = d > 0.f;
            int ri, ci;
            const bool ok = texel_fused(F, px, py, pz, ri, ci);
            bad |= (cov && !ok) << e;
            R.look[e] = cov ? __ldg(a.sm + (sm_off + ri * ws + ci)) : -1.f;   // consumed one phase later
            if (kIdx && cov) {      // parity hook (own kernel variant): the texel this pixel gathered
                const int64_t hw = (int64_t)a.h * a.w;
                int32_t* ti = a.tidx + (int64_t)tl.f * 2 * hw +
                              (int64_t)(2 * tl.ty0 - 2 + ST_ROWS * (q & 1) + qy) * a.w +
                              (2 * tl.tx0 - 2 + 2 * (e < 2 ? px_lo : px_hi) + (e & 1));
                ti[0] = ri;
                ti[hw] = ci;
            }
            const float tx = ecx - px, ty = ecy - py, tz = ecz - pz;
            const float l2 = fmaf(tx, tx, fmaf(ty, ty, tz * tz));
            const float izf = rsqrtf(l2);
            // c_c = clip(n . -ray): the pixel ray is the direction camera -> hit
            // point (render_gbuffer places p on it), fp32 is ample here
            const float dx = cpx - px, dy = cpy - py, dz = cpz - pz;
            const float nx = nxv[e], ny = nyv[e], nz = nzv[e];
            const float cc = __saturatef(fmaf(nx, dx, fmaf(ny, dy, nz * dz)) *
                                         rsqrtf(fmaf(dx, dx, fmaf(dy, dy, dz * dz))));
            const float c2 = __saturatef(fmaf(nx, tx, fmaf(ny, ty, nz * tz)) * izf) + size;
            P.v[e] = make_uint2(__float_as_uint(l2 * izf), cov ? Elem<T>::pack(c2, __fdividef(cc, d)) : 0u);
        }
        if (bad) {   // FrustumError: the quad's leftmost bad pixel (raster.py:251-255)
            const int e = __ffs(bad) - 1;
            atomic_min_i64(a.first_bad + tl.f, (int64_t)(2 * tl.ty0 - 2 + ST_ROWS * (q & 1) + qy) * a.w +
                                                   (2 * tl.tx0 - 2 + 2 * (e < 2 ? px_lo : px_hi) + (e & 1)));
        }
    };
    auto phaseB = [&](int q, const QuadRegs& R) {
        if (!active) return;
        const float bias = tbias[(q >> 1) & 7];
        uint8_t* dst = smem + ((q >> 1) & 1) * E0_SMEM + (q & 1) * (ST_ROWS / 2) * E0_IC * 16;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            uint32_t* slot = reinterpret_cast<uint32_t*>(dst + (e < 2 ? slot_lo : slot_hi) + (e & 1) * 8);
            const float look = R.look[e], zf = __uint_as_float(*slot);
            float ch0 = 0.f, ch1 = look >= 0.f ? 1.f : 0.f;
            if (look >= 0.f && look < INFINITY) {           // raster.py:262 (finite lookup)
                const float m = fminf(look, zf);
                ch0 = (m - zf) + bias;
                ch1 = __fdividef(m + bias, zf);
            }
            *slot = Elem<T>::pack(ch0, ch1);
        }
    };
    // live: half q belongs to a claimed tile (the TMA thread's sentinel, -1,
    // ends the loop after the last half's phase B)
    auto step = [&](int q, int tile, QuadRegs& RA, QuadRegs& RB) {
        const bool live = tile >= 0;
        QuadPark P;
        if (live) {
            if (!(kExp && (a.dbg & 1))) phaseA(q, tile, RA, P);
            else for (int e = 0; e < 4; ++e) RA.look[e] = -1.f, P.v[e] = make_uint2(0u, 0u);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[q & 1]);                   // stage read
            if (q & 1) park(q, P);            // second half: the buffer is ours already
        }
        if (q >= 1) {
            const int qb = q - 1, k = qb >> 1;
            phaseB(qb, RB);
            __syncwarp();
            if (lane == 0) mbar_arrive(&half[(k & 1) * 2 + (qb & 1)]);   // rows of half qb&1 done
        }
        if (!live) {
            // no tile k: wake the consumers, which read the sentinel
            __syncwarp();
            if (lane == 0) mbar_arrive(&half[((q >> 1) & 1) * 2]);
        }
        if (live && !(q & 1)) {
            // a tile's first half: wait for the consumers to release the
            // buffer (after finishing the previous tile above), then park
            const int k = q >> 1;
            if (k >= 2) mbar_wait_backoff(&freed[k & 1], ((k - 2) >> 1) & 1);
            park(q, P);
        }
    };
    QuadRegs RA, RB;
#pragma unroll 1
    for (int q = 0;; ++q) {
        mbar_wait(&full[q & 1], (q >> 1) & 1);             // data (or the sentinel) for half q
        const int tile = tring[(q >> 1) & 7];
        step(q, tile, RA, RB);
        if (tile < 0) break;
        const QuadRegs t = RA;
        RA = RB;
        RB = t;
    }
}

// kSrc: 0 = features planes, 1 = G-buffer (LDG), 2 = G-buffer (TMA).  kIdx:
// the parity-hook variant that also writes each covered pixel's texel index
// (a separate instantiation, so the production kernel keeps its registers).
template <typename T, int kSrc, bool kIdx = false>
__global__ void __launch_bounds__(kSrc == 2 ? kE0Threads : kL0Threads, 1) enc0_kernel(
    const __grid_constant__ Enc0Args a, const __grid_constant__ GbufMaps tm, int total) {
    constexpr int kProd = kSrc == 2 ? kE0Prod : kL0Prod;
    constexpr int kThreads = kSrc == 2 ? kE0Threads : kL0Threads;
    if (threadIdx.x == 0) pdl_trigger();
    if (kExp && a.trace && threadIdx.x == 0 && blockIdx.x < 512) {
        a.trace[2 * blockIdx.x] = globaltimer_ns();
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        a.trace[1024 + blockIdx.x] = smid;
    }
    if constexpr (kSrc == 2) {
        extern __shared__ __align__(128) uint8_t smem[];
        uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * E0_SMEM + 2 * ST_BYTES);
        if (threadIdx.x == 0) {
            mbar_init(&bars[0], 1);                 // full[2]
            mbar_init(&bars[1], 1);
            for (int i = 2; i < 8; ++i) mbar_init(&bars[i], kE0FeatWarps);   // empty[2], half[2][2]
            mbar_init(&bars[8], kE0MmaWarps);      // freed[2]
            mbar_init(&bars[9], kE0MmaWarps);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
    }
    // The G-buffer is an input, not the previous kernel's output: the TMA
    // warp starts streaming it before the grid dependency resolves; every
    // other thread waits (first_bad, the pooled output).
    if (kSrc != 2 || threadIdx.x / 32 != kE0FeatWarps) pdl_wait();
    if (kSrc == 2) {
        static_assert(kE0ProdRegs == 72 && kE0MmaRegs == 112, "keep the asm immediates in sync");
        if (threadIdx.x < kProd) asm volatile("setmaxnreg.dec.sync.aligned.u32 72;");
        else asm volatile("setmaxnreg.inc.sync.aligned.u32 112;");
    }
    constexpr int kRows = kSrc == 2 ? 16 : 8;        // output rows per consumer warp
    if (threadIdx.x < kProd) {
        if (kSrc == 2) {
            produce_features_tma<T, kIdx>(a, tm, total);
        } else {
            l0_produce_loop(total, [&](uint8_t* buf, int tile) {
                produce_features<T, kSrc == 1>(a, buf, l0_tile(tile, a.td));
            });
        }
        return;
    }
    const int H1 = a.H0 / 2, W1 = a.W0 / 2;
    const int cw = (threadIdx.x - kProd) >> 5;       // consumer warp
    const int lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int sx = (cw & 3) * 16, r0 = (cw >> 2) * kRows;
    uint32_t B3[9][2][2], B1[2][2];
    float bias3[2][2], bias1[2][2];
    {
#pragma unroll
        for (int tap = 0; tap < 9; ++tap)
#pragma unroll
            for (int n = 0; n < 2; ++n) {
                const uint2 v = __ldg(a.wb3 + (tap * 2 + n) * 32 + lane);
                B3[tap][n][0] = v.x;
                B3[tap][n][1] = v.y;
            }
#pragma unroll
        for (int n = 0; n < 2; ++n) {
            const uint2 v = __ldg(a.wb1 + n * 32 + lane);
            B1[n][0] = v.x;
            B1[n][1] = v.y;
        }
#pragma unroll
        for (int n = 0; n < 2; ++n)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                bias3[n][e] = __ldg(a.b3 + n * 8 + 2 * t + e);
                bias1[n][e] = 0.25f * __ldg(a.b1 + n * 8 + 2 * t + e);   // pool scale folded (see pack_f16)
            }
    }
    T* out = reinterpret_cast<T*>(a.out);
    auto consume = [&](uint8_t* buf, int tile, auto&& hook) {
            const L0Tile tl = l0_tile(tile, a.td);
            float pp[2][2];
            // pooled pixel ((ty0 + r0) / 2 + oo / 2, (tx0 + sx) / 2 + g): one 64-bit
            // base per tile, 32-bit row offsets
            const int px = ((tl.tx0 + sx) >> 1) + g;
            const bool px_ok = px < W1;
            T* obase = out + (((int64_t)tl.f * H1 + ((tl.ty0 + r0) >> 1)) * W1 + px) * 16 + 2 * t;
            if (a.dbg & 2) {          // experiments only (dbg is 0 in release builds)
                hook(E0_IR / 2);
                return;
            }
            conv3_strip16<T, kRows, true>(smem_u32(buf), E0_PLANE, E0_IC, r0, sx, B3, bias3, [&](int oo, float (&acc)[2][4]) {
                uint32_t a1[4];
                relu_pack_a<T>(acc, a1);
                float u[2][4];
#pragma unroll
                for (int n = 0; n < 2; ++n) {
                    mma16816_c<T>(u[n], a1, B1[n][0], B1[n][1], bias1[n][0], bias1[n][1], bias1[n][0], bias1[n][1]);
                }
                // avg_pool2: rows oo-1, oo summed in registers; the x
                // neighbours are this thread's e and e + 2 (kPairRows)
#pragma unroll
                for (int n = 0; n < 2; ++n)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const float v = fmaxf(u[n][e], 0.f) + fmaxf(u[n][e + 2], 0.f);
                        if (oo & 1) pp[n][e] += v;
                        else pp[n][e] = v;
                    }
                if (oo & 1) {                                           // avg_pool2 of rows oo-1, oo
                    if (((tl.ty0 + r0 + oo) >> 1) < H1 && px_ok) {
                        T* o = obase + (oo >> 1) * W1 * 16;
#pragma unroll
                        for (int n = 0; n < 2; ++n)
                            *reinterpret_cast<uint32_t*>(o + n * 8) = Elem<T>::pack(pp[n][0], pp[n][1]);
                    }
                }
            }, hook);
    };
    if constexpr (kSrc == 2) {
        extern __shared__ __align__(128) uint8_t smem[];
        uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * E0_SMEM + 2 * ST_BYTES);
        uint64_t* half = bars + 4;
        uint64_t* freed = bars + 8;
        // the producers signal each half of a tile (level-0 rows 0-8 and
        // 9-17), so the convolution starts one half-tile earlier
        const int* tring = reinterpret_cast<const int*>(bars + 10);
        for (int k = 0;; ++k) {
            const int s = k & 1;
            const uint32_t par = (k >> 1) & 1;
            mbar_wait(&half[s * 2], par);
            const int tile = tring[k & 7];
            if (tile < 0) break;
            consume(smem + s * E0_SMEM, tile, [&](int ir) {
                if (ir == E0_IR / 2) mbar_wait(&half[s * 2 + 1], par);
            });
            __syncwarp();
            if (lane == 0) mbar_arrive(&freed[s]);
        }
        if (kExp && a.trace && threadIdx.x == kProd && blockIdx.x < 512) a.trace[2 * blockIdx.x + 1] = globaltimer_ns();
    } else {
        l0_consume_loop<kThreads>(total, [&](uint8_t* buf, int tile) { consume(buf, tile, NoRowHook{}); });
    }
}

// ------------------------------------------------ level 0 of the 5-plane net
// enc0_s2d: l0.enc3 (20 -> 16, 3x3) + l0.enc1 + avg_pool2 from the 16-bit
// chunk-planar s2d tensor (N, 3, H0, W0, 8) written by feat5_kernel (the 4
// reference planes and the blocker-search plane).  A TMA warp streams halo'd
// 18 x 66 tiles (three 22-pixel boxes: a TMA box row holds at most 256
// elements) into a 3-stage ring; 8 warps run the convolutions: the K = 16
// chunks 0-1 as m16n8k16 and chunk 2 (4 blocker channels + 4 zero) as
// m16n8k8 per tap, the rest exactly as enc0 (pair-row pixel order, enc1 on
// the accumulator as A fragment, the 2x2 pool in registers).
constexpr int S24_BOXW = 22, S24_NBOX = 3;
static_assert(S24_BOXW * S24_NBOX == E0_IC, "boxes tile the halo'd row");
constexpr int S24_ROWB = S24_BOXW * 16;               // one box row of one chunk
constexpr int S24_CSTR = E0_IR * S24_ROWB;             // one chunk of one box
constexpr int S24_BOXB = round128(3 * S24_CSTR);       // one box, 3 chunks (TMA destinations 128-B aligned)
constexpr int S24_TILE = S24_NBOX * S24_BOXB;          // 57,216 B per tile
constexpr int S24_NS = 3;                              // ring stages
constexpr int kS24Mma = 8, kS24Threads = 32 * (kS24Mma + 1);
constexpr int S24_SMEM = S24_NS * S24_TILE + 64;

__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t r[2]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];\n" : "=r"(r[0]), "=r"(r[1]) : "r"(addr));
}

template <typename T>
__device__ __forceinline__ void mma1688(float c[4], const uint32_t a[2], uint32_t b0) {
    if constexpr (std::is_same<T, __half>::value)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                     : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
                     : "r"(a[0]), "r"(a[1]), "r"(b0));
    else
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                     : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
                     : "r"(a[0]), "r"(a[1]), "r"(b0));
}

// conv3_strip16 on the box-split 24-channel tile: the same sliding-window
// schedule (each input row's three dx-shifted fragments loaded once), plus
// the k8 chunk.  Lane addresses carry the box split (x / 22, x % 22).
template <typename T, int ROWS, class Epi>
__device__ __forceinline__ void conv3_strip24(uint32_t sbase, int r0, int sx, const uint32_t (&B3)[9][2][2],
                                              const uint32_t (&B3c)[9][2], const float (&binit)[2][2],
                                              Epi&& epi) {
    const int lane = threadIdx.x & 31;
    const int lm = lane >> 3, li = lane & 7;
    uint32_t xo[3], xoc[3];
#pragma unroll
    for (int dx = 0; dx < 3; ++dx) {
        const int x = sx + 2 * li + (lm & 1) + dx;           // pair-row pixel order (kPairRows)
        const int bx = (x * 373) >> 13;                       // x / 22 for x < 66
        const uint32_t o = bx * S24_BOXB + (x - bx * S24_BOXW) * 16;
        xo[dx] = o + (lm >> 1) * S24_CSTR;
        xoc[dx] = o + 2 * S24_CSTR;
    }
    float acc[3][2][4];
    uint32_t Ab[2][3][4], Ac[2][3][2];
    auto load_row = [&](int ir, uint32_t (&A)[3][4], uint32_t (&C)[3][2]) {
        const uint32_t ro = sbase + (r0 + ir) * S24_ROWB;
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) {
            ldsm_x4(ro + xo[dx], A[dx]);
            ldsm_x2(ro + xoc[dx], C[dx]);
        }
    };
    load_row(0, Ab[0], Ac[0]);
#pragma unroll
    for (int ir = 0; ir < ROWS + 2; ++ir) {
        if (ir + 1 < ROWS + 2) load_row(ir + 1, Ab[(ir + 1) & 1], Ac[(ir + 1) & 1]);
        uint32_t (&A)[3][4] = Ab[ir & 1];
        uint32_t (&Cc)[3][2] = Ac[ir & 1];
#pragma unroll
        for (int dx = 0; dx < 3; ++dx)
#pragma unroll
            for (int ky = 0; ky < 3; ++ky) {
                const int oo = ir - ky;
                if (oo >= 0 && oo < ROWS) {
#pragma unroll
                    for (int n = 0; n < 2; ++n) {
                        const int tap = ky * 3 + dx;
                        if (ky == 0 && dx == 0)
                            mma16816_c<T>(acc[oo % 3][n], A[dx], B3[tap][n][0], B3[tap][n][1], binit[n][0],
                                          binit[n][1], binit[n][0], binit[n][1]);
                        else
                            mma16816<T>(acc[oo % 3][n], A[dx], B3[tap][n][0], B3[tap][n][1]);
                        mma1688<T>(acc[oo % 3][n], Cc[dx], B3c[tap][n]);
                    }
                }
            }
        if (ir >= 2) {
            const int oo = ir - 2;
            epi(oo, acc[oo % 3]);
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(kS24Threads, 1) enc0_s2d_kernel(const __grid_constant__ Enc0Args a,
                                                                  const __grid_constant__ CUtensorMap xm, int total) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S24_NS * S24_TILE);
    uint64_t* empty = full + S24_NS;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S24_NS; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], kS24Mma);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) pdl_trigger();
    pdl_wait();                                 // the s2d tensor is the previous kernel's output
    if (warp == kS24Mma) {                      // TMA producer
        if (lane == 0) {
            const uint64_t pol = l2_evict_first_policy();      // read once
            for (int k = 0;; ++k) {
                const int tile = blockIdx.x + k * gridDim.x;
                if (tile >= total) break;
                const int s = k % S24_NS;
                if (k >= S24_NS) mbar_wait(&empty[s], ((k / S24_NS) - 1) & 1);
                const L0Tile tl = l0_tile(tile, a.td);
                const uint32_t dst = smem_u32(smem + s * S24_TILE);
                mbar_expect_tx(&full[s], S24_NBOX * 3 * S24_CSTR);   // bytes the three boxes deliver
#pragma unroll
                for (int b = 0; b < S24_NBOX; ++b)
                    tma_load_3d_stream(dst + b * S24_BOXB, &xm, (tl.tx0 - 1 + b * S24_BOXW) * 8, tl.ty0 - 1,
                                       tl.f * 3, &full[s], pol);
            }
        }
        return;
    }
    const int H1 = a.H0 / 2, W1 = a.W0 / 2;
    const int g = lane >> 2, t = lane & 3;
    const int sx = (warp & 3) * 16, r0 = (warp >> 2) * 8;
    uint32_t B3[9][2][2], B3c[9][2], B1[2][2];
    float bias3[2][2], bias1[2][2];
#pragma unroll
    for (int tap = 0; tap < 9; ++tap)
#pragma unroll
        for (int n = 0; n < 2; ++n) {
            const uint2 v = __ldg(a.wb3 + ((tap * 2 + 0) * 2 + n) * 32 + lane);   // K-step 0: chunks 0-1
            B3[tap][n][0] = v.x;
            B3[tap][n][1] = v.y;
            B3c[tap][n] = __ldg(a.wb3 + ((tap * 2 + 1) * 2 + n) * 32 + lane).x;  // K-step 1, k 0-7: chunk 2
        }
#pragma unroll
    for (int n = 0; n < 2; ++n) {
        const uint2 v = __ldg(a.wb1 + n * 32 + lane);
        B1[n][0] = v.x;
        B1[n][1] = v.y;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            bias3[n][e] = __ldg(a.b3 + n * 8 + 2 * t + e);
            bias1[n][e] = 0.25f * __ldg(a.b1 + n * 8 + 2 * t + e);   // pool scale folded (pack_f16)
        }
    }
    T* out = reinterpret_cast<T*>(a.out);
    for (int k = 0;; ++k) {
        const int tile = blockIdx.x + k * gridDim.x;
        if (tile >= total) break;
        const int s = k % S24_NS;
        mbar_wait(&full[s], (k / S24_NS) & 1);
        const L0Tile tl = l0_tile(tile, a.td);
        float pp[2][2];
        const int px = ((tl.tx0 + sx) >> 1) + g;
        const bool px_ok = px < W1;
        T* obase = out + (((int64_t)tl.f * H1 + ((tl.ty0 + r0) >> 1)) * W1 + px) * 16 + 2 * t;
        conv3_strip24<T, 8>(smem_u32(smem + s * S24_TILE), r0, sx, B3, B3c, bias3, [&](int oo, float (&acc)[2][4]) {
            uint32_t a1[4];
            relu_pack_a<T>(acc, a1);
            float u[2][4];
#pragma unroll
            for (int n = 0; n < 2; ++n)
                mma16816_c<T>(u[n], a1, B1[n][0], B1[n][1], bias1[n][0], bias1[n][1], bias1[n][0], bias1[n][1]);
#pragma unroll
            for (int n = 0; n < 2; ++n)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const float v = fmaxf(u[n][e], 0.f) + fmaxf(u[n][e + 2], 0.f);
                    if (oo & 1) pp[n][e] += v;
                    else pp[n][e] = v;
                }
            if (oo & 1) {
                if (((tl.ty0 + r0 + oo) >> 1) < H1 && px_ok) {
                    T* o = obase + (oo >> 1) * W1 * 16;
#pragma unroll
                    for (int n = 0; n < 2; ++n)
                        *reinterpret_cast<uint32_t*>(o + n * 8) = Elem<T>::pack(pp[n][0], pp[n][1]);
                }
            }
        });
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
}

// fp32 planes (N, 5, H, W) -> the chunk-planar s2d tensor enc0_s2d reads
// (nsm_forward of a 5-plane plan); one thread per level-0 pixel.
template <typename T>
__global__ void pack_s2d24_kernel(const float* __restrict__ x, int H, int W, int nf, T* __restrict__ out) {
    const int H0 = H / 2, W0 = W / 2;
    const int64_t n0 = (int64_t)H0 * W0;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n0 * nf) return;
    const int f = (int)(i / n0);
    const int64_t r = i - f * n0;
    const int Y = (int)(r / W0), X = (int)(r - (int64_t)Y * W0);
    const int64_t hw = (int64_t)H * W;
    const float* xf = x + (int64_t)f * 5 * hw;
    float v[4][5];
#pragma unroll
    for (int e = 0; e < 4; ++e)
#pragma unroll
        for (int c = 0; c < 5; ++c) v[e][c] = __ldg(xf + c * hw + (int64_t)(2 * Y + (e >> 1)) * W + 2 * X + (e & 1));
    uint4 c0, c1, c2;
    c0 = make_uint4(Elem<T>::pack(v[0][0], v[0][1]), Elem<T>::pack(v[0][2], v[0][3]), Elem<T>::pack(v[1][0], v[1][1]),
                    Elem<T>::pack(v[1][2], v[1][3]));
    c1 = make_uint4(Elem<T>::pack(v[2][0], v[2][1]), Elem<T>::pack(v[2][2], v[2][3]), Elem<T>::pack(v[3][0], v[3][1]),
                    Elem<T>::pack(v[3][2], v[3][3]));
    c2 = make_uint4(Elem<T>::pack(v[0][4], v[1][4]), Elem<T>::pack(v[2][4], v[3][4]), 0u, 0u);
    const int64_t plane = n0 * 8;
    T* o = out + ((int64_t)f * 3 * n0 + r) * 8;
    *reinterpret_cast<uint4*>(o) = c0;
    *reinterpret_cast<uint4*>(o + plane) = c1;
    *reinterpret_cast<uint4*>(o + 2 * plane) = c2;
}

// Bilinear 2x of an NHWC 16-bit tensor at one output pixel, 8 channels
// (bilinear_upsample2 + _upsample_taps, autodiff.py:258-274: rows then cols).
template <typename T>
__device__ __forceinline__ void up2_chunk(const T* x, int hl, int wl, int C, int oy, int ox, int chunk,
                                          float v[8]) {
    const float sy = fminf(fmaxf((oy + 0.5f) * 0.5f - 0.5f, 0.f), (float)(hl - 1));
    const float sx = fminf(fmaxf((ox + 0.5f) * 0.5f - 0.5f, 0.f), (float)(wl - 1));
    const int y0 = (int)sy, x0 = (int)sx;
    const int y1 = min(y0 + 1, hl - 1), x1 = min(x0 + 1, wl - 1);
    const float wy = sy - y0, wx = sx - x0;
    const uint4 q00 = __ldg(reinterpret_cast<const uint4*>(x + ((int64_t)y0 * wl + x0) * C + chunk * 8));
    const uint4 q10 = __ldg(reinterpret_cast<const uint4*>(x + ((int64_t)y1 * wl + x0) * C + chunk * 8));
    const uint4 q01 = __ldg(reinterpret_cast<const uint4*>(x + ((int64_t)y0 * wl + x1) * C + chunk * 8));
    const uint4 q11 = __ldg(reinterpret_cast<const uint4*>(x + ((int64_t)y1 * wl + x1) * C + chunk * 8));
    const uint32_t* a00 = &q00.x;
    const uint32_t* a10 = &q10.x;
    const uint32_t* a01 = &q01.x;
    const uint32_t* a11 = &q11.x;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 p00 = Elem<T>::unpack(a00[i]), p10 = Elem<T>::unpack(a10[i]);
        const float2 p01 = Elem<T>::unpack(a01[i]), p11 = Elem<T>::unpack(a11[i]);
        const float c0x = p00.x * (1.f - wy) + p10.x * wy, c1x = p01.x * (1.f - wy) + p11.x * wy;
        const float c0y = p00.y * (1.f - wy) + p10.y * wy, c1y = p01.y * (1.f - wy) + p11.y * wy;
        v[2 * i] = c0x * (1.f - wx) + c1x * wx;
        v[2 * i + 1] = c0y * (1.f - wx) + c1y * wx;
    }
}

// 2x bilinear upsampling of one 8-channel chunk for the 2x2 output block of
// a low-res pixel: q[u][v] = the chunk at column u, row v of its clamped 3x3
// neighbourhood; out[2 aa + bb] = the output (2i + aa, 2j + bb), packed.
// Rows then columns with weights (1/4, 3/4) like _upsample_taps
// (autodiff.py:258-287).  fp16: packed half2 arithmetic (each FMA rounds to
// fp16, the result is stored as fp16 anyway); bf16: fp32 arithmetic, one
// rounding at the end (bf16 has too few mantissa bits to round twice).
template <typename T>
__device__ __forceinline__ void up2_block(const uint4 (&q)[3][3], uint4 (&out)[4]) {
    if constexpr (std::is_same<T, __half>::value) {
        const __half2 w1 = __float2half2_rn(0.25f), w3 = __float2half2_rn(0.75f);
        __half2 top[3][4], bot[3][4];
#pragma unroll
        for (int u = 0; u < 3; ++u) {
            const __half2* s0 = reinterpret_cast<const __half2*>(&q[u][0]);
            const __half2* s1 = reinterpret_cast<const __half2*>(&q[u][1]);
            const __half2* s2 = reinterpret_cast<const __half2*>(&q[u][2]);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                top[u][e] = __hfma2(s1[e], w3, __hmul2(s0[e], w1));
                bot[u][e] = __hfma2(s1[e], w3, __hmul2(s2[e], w1));
            }
        }
#pragma unroll
        for (int ab = 0; ab < 4; ++ab) {
            const __half2(&vr)[3][4] = (ab >> 1) ? bot : top;
            __half2* o = reinterpret_cast<__half2*>(&out[ab]);
#pragma unroll
            for (int e = 0; e < 4; ++e)
                o[e] = (ab & 1) ? __hfma2(vr[1][e], w3, __hmul2(vr[2][e], w1))
                                : __hfma2(vr[1][e], w3, __hmul2(vr[0][e], w1));
        }
    } else {
        float top[3][8], bot[3][8];
#pragma unroll
        for (int u = 0; u < 3; ++u) {
            float sv[3][8];
#pragma unroll
            for (int v = 0; v < 3; ++v) {
                const uint32_t* qw = &q[u][v].x;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float2 f2 = Elem<T>::unpack(qw[e]);
                    sv[v][2 * e] = f2.x;
                    sv[v][2 * e + 1] = f2.y;
                }
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                top[u][e] = 0.25f * sv[0][e] + 0.75f * sv[1][e];
                bot[u][e] = 0.75f * sv[1][e] + 0.25f * sv[2][e];
            }
        }
#pragma unroll
        for (int ab = 0; ab < 4; ++ab) {
            const float(&vr)[3][8] = (ab >> 1) ? bot : top;
            uint32_t* qo = &out[ab].x;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float x0 = (ab & 1) ? 0.75f * vr[1][2 * e] + 0.25f * vr[2][2 * e]
                                          : 0.25f * vr[0][2 * e] + 0.75f * vr[1][2 * e];
                const float x1 = (ab & 1) ? 0.75f * vr[1][2 * e + 1] + 0.25f * vr[2][2 * e + 1]
                                          : 0.25f * vr[0][2 * e + 1] + 0.75f * vr[1][2 * e + 1];
                qo[e] = Elem<T>::pack(x0, x1);
            }
        }
    }
}

// a + b of two packed 8-channel chunks (the decoder skip sum): half2 adds on
// fp16 plans, fp32 with one rounding on bf16.
template <typename T>
__device__ __forceinline__ uint4 add_packed(uint4 a, uint4 b) {
    uint4 r;
    const uint32_t *pa = &a.x, *pb = &b.x;
    uint32_t* pr = &r.x;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        if constexpr (std::is_same<T, __half>::value) {
            const __half2 v = __hadd2(*reinterpret_cast<const __half2*>(&pa[e]), *reinterpret_cast<const __half2*>(&pb[e]));
            pr[e] = *reinterpret_cast<const uint32_t*>(&v);
        } else {
            const float2 x = Elem<T>::unpack(pa[e]), y = Elem<T>::unpack(pb[e]);
            pr[e] = Elem<T>::pack(x.x + y.x, x.y + y.y);
        }
    }
    return r;
}

// Head reconstruction (network.py:199-209) + sigmoid, cropped to (h, w):
// out(2Y+sy, 2X+sx) = sigmoid(up2(y0) + [sy,sx != 0,0] * y_{2sy+sx}(Y, X)).
// The 2x half-pixel bilinear of y0 at the 4 outputs of L0 pixel (Y, X) uses
// rows/cols Y-1..Y+1 with weights (1/4, 3/4); clamping the neighbour indices
// reproduces the reference's edge clamp (_upsample_taps, autodiff.py:258-264).
__device__ __forceinline__ float sigmoid_fast(float v) {
    // logistic (autodiff.py:200-209) as 1/2 + tanh(v/2)/2: one MUFU.TANH
    // (max relative error ~2^-11, saturating, so no overflow for large |v|)
    float t;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.5f * v));
    return fmaf(0.5f, t, 0.5f);
}

// Each thread reconstructs 4 consecutive level-0 pixels (8 x 2 outputs):
// ch0 of rows Y-1..Y+1 at columns X0-1..X0+4 (8-B + 2 edge loads per row),
// the 3 detail channels as 8-B loads of the fp16 Y planes, two 16-B rows of
// fp16 out.
constexpr int kReconPx = 4;
__global__ void __launch_bounds__(128) recon_kernel(const __half* __restrict__ y, int H0, int W0, int h,
                                                     int w, int n, void* __restrict__ out, int f16) {
    if (threadIdx.x == 0) pdl_trigger();
    pdl_wait();
    const int X0 = (blockIdx.x * blockDim.x + threadIdx.x) * kReconPx;
    const int Y = blockIdx.y;
    const int f = blockIdx.z;
    if (X0 >= W0) return;
    const int hw0 = H0 * W0;
    const __half* y0 = y + (int64_t)f * 4 * hw0;
    auto ld4 = [](const __half* p, float (&v)[4]) {    // 4 consecutive fp16 (8-B aligned)
        const uint2 q = __ldg(reinterpret_cast<const uint2*>(p));
        const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&q.x));
        const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&q.y));
        v[0] = a.x, v[1] = a.y, v[2] = b.x, v[3] = b.y;
    };
    const int rows[3] = {max(Y - 1, 0), Y, min(Y + 1, H0 - 1)};
    const int xm = max(X0 - 1, 0), xp = min(X0 + kReconPx, W0 - 1);
    float r[3][kReconPx + 2];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const __half* row = y0 + rows[i] * W0;
        float c[4];
        ld4(row + X0, c);
        r[i][0] = __half2float(row[xm]);
        r[i][1] = c[0], r[i][2] = c[1], r[i][3] = c[2], r[i][4] = c[3];
        r[i][5] = __half2float(row[xp]);
    }
    float det[3][kReconPx];
#pragma unroll
    for (int c = 0; c < 3; ++c) ld4(y0 + (c + 1) * hw0 + Y * W0 + X0, det[c]);
#pragma unroll
    for (int sy = 0; sy < 2; ++sy) {
        const int oy = 2 * Y + sy;
        if (oy >= h) break;
        // rows: sy = 0 -> (Y-1, Y) weights (1/4, 3/4); sy = 1 -> (Y, Y+1) weights (3/4, 1/4)
        float cr[kReconPx + 2];
#pragma unroll
        for (int j = 0; j < kReconPx + 2; ++j)
            cr[j] = sy ? r[1][j] * 0.75f + r[2][j] * 0.25f : r[0][j] * 0.25f + r[1][j] * 0.75f;
        float o[2 * kReconPx];
#pragma unroll
        for (int k = 0; k < kReconPx; ++k)
#pragma unroll
            for (int sx = 0; sx < 2; ++sx) {
                const float base = sx ? cr[k + 1] * 0.75f + cr[k + 2] * 0.25f : cr[k] * 0.25f + cr[k + 1] * 0.75f;
                // depth_to_space detail: channel 2sy + sx, zero for (0, 0)
                const float d = (sy | sx) ? det[2 * sy + sx - 1][k] : 0.f;
                o[2 * k + sx] = sigmoid_fast(base + d);
            }
        const int64_t ob = ((int64_t)f * h + oy) * w + 2 * X0;
        if (2 * X0 + 2 * kReconPx <= w && !(w & 7)) {
            if (f16) {
                uint4 v;
                v.x = Elem<__half>::pack(o[0], o[1]), v.y = Elem<__half>::pack(o[2], o[3]);
                v.z = Elem<__half>::pack(o[4], o[5]), v.w = Elem<__half>::pack(o[6], o[7]);
                *reinterpret_cast<uint4*>(reinterpret_cast<__half*>(out) + ob) = v;
            } else {
                float4* po = reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + ob);
                po[0] = make_float4(o[0], o[1], o[2], o[3]);
                po[1] = make_float4(o[4], o[5], o[6], o[7]);
            }
        } else {
#pragma unroll
            for (int k = 0; k < 2 * kReconPx; ++k) {
                if (2 * X0 + k >= w) break;
                if (f16) reinterpret_cast<__half*>(out)[ob + k] = __float2half_rn(o[k]);
                else reinterpret_cast<float*>(out)[ob + k] = o[k];
            }
        }
    }
}

// ------------------------------------------------------------- levels 1-3 (tcgen05)
enum { SRC_TENSOR = 0, SRC_UP = 1 };
// DST_PADREP: the stored tensor is chunk-planar (N, 2, H + 2, W + 2, 8)
// (C1 = 16) with a one-pixel border that replicates the edge (the polyphase level-0 decoder reads the
// edge-clamped upsampling source from it without bounds logic)
enum { DST_STORE = 1, DST_POOL = 2, DST_PADREP = 4 };

struct LevelArgs {
    const void* x;       // SRC_TENSOR: (N, H, W, CIN); SRC_UP: (N, H/2, W/2, CIN)
    const void* skip;    // SRC_UP: (N, H, W, CIN) or null
    int H, W;
    const void* w3;      // umma layout [9][CIN/16][2][C3][8]
    const float* b3;
    const void* w1;      // umma layout [1][C3/16][2][C1][8]
    const float* b1;
    void* out;           // (N, H, W, C1)
    void* pool;          // (N, H/2, W/2, C1)
    int dbg;             // experiments only: 1 skip producer math, 2 skip epilogue math, 4 skip MMAs
    long long* trace;    // experiments only (NSM_LEVEL_TRACE=<name>): CTA 0 per-tile clock64 events
};

template <int CIN, int C3, int C1, int NB, int NIN, int NMID, int STG>
struct LvGeom {
    static constexpr int TH = 16, TW = 8 * NB;
    static constexpr int IR = TH + 2, IC = TW + 2;
    static constexpr int NCI = CIN / 8, NC3 = C3 / 8, KK = CIN / 16;
    // SRC_UP (STG): the low-res tile is always staged (double-buffered).  The
    // skip tile is staged pixel-major and double-buffered when shared memory
    // allows (STAGED), else TMA'd straight into the input buffer, whose box is
    // then padded by a row and a column so that the chunk-plane stride is an
    // odd multiple of 16 B (the producers' per-chunk accesses hit all banks)
    static constexpr int LR = TH / 2 + 2, LC = TW / 2 + 2;
    static constexpr int LOB = STG ? LR * LC * CIN * 2 : 0, SKB = STG ? IR * IC * CIN * 2 : 0;
    static constexpr int MIDC_ = NB * C3 / 2, ACCM_ = 2 * NB * (C3 + C1);
    static constexpr bool MIDT_ = ACCM_ + NMID * MIDC_ <= 512;
    static constexpr int FIXED = NIN * round128(NCI * IR * IC * 16) + (MIDT_ ? 0 : NMID * round128(NC3 * plane_bytes(TH * TW, NC3))) +
                                 9 * CIN * C3 * 2 + C3 * C1 * 2 + 128 + round128(2 * LOB) + (C3 + C1) * 4 + 16 + 256;
    static constexpr bool STAGED = STG && FIXED + 2 * round128(SKB) <= 232448;
    static constexpr int PADIN = (STG && !STAGED) ? 1 : 0;
    static constexpr int ICB = IC + PADIN, IRB = IR + PADIN, NPI = IRB * ICB;
    static constexpr int PIN = NPI * 16;                       // dense: the TMA box layout
    static constexpr int INB = round128(NCI * PIN);
    static constexpr int PMID = plane_bytes(TH * TW, NC3);
    // conv1's A operand (relu(conv3) packed to 16 bits) lives in TMEM when the
    // columns allow (the accumulators of both convs are double-buffered):
    // lane = pixel, 2 channels per column; otherwise in a chunk-planar SMEM tile
    static constexpr int ACCM = 2 * NB * (C3 + C1), MIDC = NB * C3 / 2;
    static constexpr bool MIDT = ACCM + NMID * MIDC <= 512;
    static constexpr int MIDB = MIDT ? 0 : round128(NC3 * PMID);
    static constexpr int W3B = 9 * CIN * C3 * 2, W1B = C3 * C1 * 2;
    static constexpr int OFF_MID = NIN * INB;
    static constexpr int OFF_W3 = OFF_MID + NMID * MIDB;
    static constexpr int OFF_W1 = OFF_W3 + W3B;
    static constexpr int SKBR = round128(SKB);
    static constexpr int OFF_SK = round128(OFF_W1 + W1B);
    static constexpr int OFF_LO = round128(OFF_SK + (STAGED ? 2 * SKBR : 0));
    static constexpr int OFF_B = round128(OFF_LO + 2 * LOB);   // low-res staging double-buffered
    static constexpr int OFF_BAR = (OFF_B + (C3 + C1) * 4 + 15) / 16 * 16;
    static constexpr int SMEM = OFF_BAR + 256;
    static constexpr int ACC3 = 0, ACC1 = 2 * NB * C3;         // TMEM columns (both double-buffered)
    static constexpr int TCOLS = tmem_cols(ACCM + (MIDT ? NMID * MIDC : 0));
    static constexpr int TX_BYTES = NCI * PIN;
};

__device__ __forceinline__ void copy_smem16(uint8_t* dst, const uint8_t* src, int bytes) {
    for (int i = threadIdx.x * 16; i < bytes; i += blockDim.x * 16)
        *reinterpret_cast<uint4*>(dst + i) = __ldg(reinterpret_cast<const uint4*>(src + i));
}

__device__ __forceinline__ void tma_load_5d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            int c3, int c4, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], "
        "[%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_load_5d_stream(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                                   int c3, int c4, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
        "[%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar)),
        "l"(pol)
        : "memory");
}

// 1-D bulk copy global -> SMEM (TMA engine, no tensor map), 16-B granules.
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// Persistent, warp-specialised level kernel (levels 1-3):
//   producer warps  - TMA (SRC_TENSOR: a 5-D box turns NHWC into the
//                     chunk-planar tile, zero-filled halo) or up2(low)+skip
//                     in fp32 (SRC_UP) into NIN input buffers
//   MMA warp        - one thread issues conv3x3 as 9 taps x CIN/16 UMMAs per
//                     128-pixel M-block (A = shifted views of the input tile,
//                     B = resident weights) into one of two TMEM accumulators,
//                     then conv1x1 on the 16-bit mid tile into two more
//   epilogue warps  - TMEM -> bias+ReLU -> mid tile; TMEM -> bias+ReLU ->
//                     NHWC store and/or 2x2 average pool
// All hand-offs are mbarriers (tcgen05.commit on the tensor-core side), so
// conv3 of tile k+1 overlaps the epilogues of tile k.
// MMA issuer warps: SRC_UP kernels (up to 72 conv3 UMMAs per tile) issue each
// M-block's conv3 from its own warp and conv1 from another, since one thread
// issues a UMMA only every ~50-70 cycles; SRC_TENSOR kernels keep one issuer
// (their epilogues need the registers).
template <int SRC, int NB>
__host__ __device__ constexpr int lv_mma_warps() { return SRC == SRC_UP ? NB + 1 : 1; }
// epilogue warps: 4 per TMEM lane quadrant where the warp budget allows
// (the epilogue is latency-bound), else 2; they split the accumulator columns
template <int SRC>
__host__ __device__ constexpr int lv_epi_warps() { return SRC == SRC_TENSOR ? 16 : 8; }
template <int SRC, int NB, int NPW>
__host__ __device__ constexpr int lv_threads() {
    return (NPW + lv_epi_warps<SRC>() + lv_mma_warps<SRC, NB>() + (SRC == SRC_UP)) * 32;
}

template <typename T, int CIN, int C3, int C1, int SRC, int DST, int NB, int NIN, int NMID, int NPW>
__global__ void __launch_bounds__(lv_threads<SRC, NB, NPW>(), 1) level_kernel(const __grid_constant__ LevelArgs a,
                                                                   const __grid_constant__ CUtensorMap tin,
                                                                   const __grid_constant__ CUtensorMap tlo,
                                                                   int total) {
    using G = LvGeom<CIN, C3, C1, NB, NIN, NMID, SRC == SRC_UP>;
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + G::OFF_BAR);
    static_assert(NIN <= 4 && NMID <= 2, "barrier slots");
    uint64_t* in_full = bar + 0;      // [NIN]
    uint64_t* in_empty = bar + 4;     // [NIN]
    uint64_t* a3_full = bar + 8;
    uint64_t* a3_empty = bar + 10;
    uint64_t* mid_full = bar + 12;
    uint64_t* mid_empty = bar + 14;
    uint64_t* a1_full = bar + 16;
    uint64_t* a1_empty = bar + 18;
    uint64_t* wbar = bar + 20;        // weights landed
    uint64_t* skf = bar + 21;         // SRC_UP: skip tile landed in in[s] [NIN <= 3]
    uint64_t* lof = bar + 24;         // SRC_UP: low-res tile landed, double-buffered [2]
    uint64_t* lo_empty = bar + 26;    // SRC_UP: producers done with low-res buffer [2]
    static_assert(SRC != SRC_UP || G::STAGED || NIN <= 3, "skip barrier slots");
    uint32_t* tptr = reinterpret_cast<uint32_t*>(smem + G::OFF_BAR + 224);
    float* sb3 = reinterpret_cast<float*>(smem + G::OFF_B);
    float* sb1 = sb3 + C3;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int NE = lv_epi_warps<SRC>(), NG = NE / 4;   // epilogue warps, column groups
    constexpr int EW0 = NPW, MW = NPW + NE;         // first epilogue warp, first MMA warp
    static_assert((NB * C3 / 16) % NG == 0 && (NB * C1 / 16) % NG == 0, "column slices per epilogue warp");
    constexpr int NMW = lv_mma_warps<SRC, NB>();
    constexpr bool kSplit = NMW > 1;                // MW + b: conv3 of M-block b; MW + NB: conv1
    constexpr int TW_ = MW + NMW;                   // SRC_UP: TMA warp
    constexpr int NPT = NPW * 32;
    const uint32_t sbase = smem_u32(smem);
    const int ntx = (a.W + G::TW - 1) / G::TW, nty = (a.H + G::TH - 1) / G::TH;
    const int mytiles = (int)blockIdx.x < total ? (total - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
    auto tr = [&](int k, int ev) {     // experiments: CTA 0's per-tile timeline
        if (kExp && a.trace && blockIdx.x == 0 && k < 32) a.trace[k * 8 + ev] = clock64();
    };
    auto tile_of = [&](int k, int& f, int& y0, int& x0) {
        const int t = blockIdx.x + k * gridDim.x;
        x0 = (t % ntx) * G::TW;
        y0 = ((t / ntx) % nty) * G::TH;
        f = t / (ntx * nty);
    };

    if (tid == 0) pdl_trigger();
    if (kExp && a.trace && tid == 0 && blockIdx.x < 256) a.trace[256 + 2 * blockIdx.x] = globaltimer_ns();
    if (warp == EW0) tmem_alloc<G::TCOLS>(tptr);
    if (tid == 0) {
        for (int i = 0; i < NIN; ++i) {
            mbar_init(&in_full[i], SRC == SRC_TENSOR ? 1 : NPT);
            mbar_init(&in_empty[i], kSplit ? NB : 1);          // one commit per conv3 issuer
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&a3_full[i], kSplit ? NB : 1);
            mbar_init(&a3_empty[i], NE * 32);
            mbar_init(&mid_full[i], NE * 32);
            mbar_init(&mid_empty[i], 1);
            mbar_init(&a1_full[i], 1);
            mbar_init(&a1_empty[i], NE * 32);
        }
        mbar_init(wbar, 1);
        for (int i = 0; i < 3; ++i) mbar_init(&skf[i], 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&lof[i], 1);
            mbar_init(&lo_empty[i], NPW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        // resident weights: two async bulk copies, waited on by the MMA warp only
        mbar_expect_tx(wbar, G::W3B + G::W1B);
        bulk_g2s(sbase + G::OFF_W3, a.w3, G::W3B, wbar);
        bulk_g2s(sbase + G::OFF_W1, a.w1, G::W1B, wbar);
    }
    for (int i = tid; i < C3; i += blockDim.x) sb3[i] = a.b3[i];
    for (int i = tid; i < C1; i += blockDim.x) sb1[i] = a.b1[i];
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tptr;
    pdl_wait();                      // prologue above overlaps the previous kernel's tail

    if (warp < NPW) {
        // ------------------------------------------------------------ producer
        if (SRC == SRC_TENSOR) {
            if (tid == 0) {
                for (int k = 0; k < mytiles; ++k) {
                    const int s = k % NIN;
                    mbar_wait(&in_empty[s], ((k / NIN) & 1) ^ 1);
                    int f, y0, x0;
                    tile_of(k, f, y0, x0);
                    mbar_expect_tx(&in_full[s], G::TX_BYTES);
                    tma_load_5d_stream(sbase + s * G::INB, &tin, 0, x0 - 1, y0 - 1, 0, f, &in_full[s], l2_evict_first_policy());
                }
            }
        } else if constexpr (G::STAGED) {
            // up2(low) + skip from TMA-staged pixel-major tiles (skip: the halo'd
            // tile; low: (TH/2+2) x (TW/2+2) source pixels, edge-clamped indices).
            // The skip tile streams in two row halves and the low-res tile is
            // double-buffered, so the next tile's staging lands while this one
            // is computed: skip rows 0-8 of tile k+1 are issued as soon as the
            // producers finish rows 0-8 of tile k, the low tile of k+2 when
            // tile k is done.
            const int hl = a.H / 2, wl = a.W / 2;
            // (NIN = 1: the input buffer is single, the producers wait for the
            // MMA anyway, so the skip tile is one piece issued per tile)
            constexpr bool kSk2 = true;                         // skip double-buffered with the low tile
            constexpr int NH = kSk2 ? 1 : (NIN == 2 ? 2 : 1);   // skip pieces per tile
            constexpr int HR = G::IR / NH;                      // rows per skip piece
            constexpr int SKH = HR * G::IC * CIN * 2;           // bytes per skip piece
            static_assert(G::IR % NH == 0, "skip halves");
            auto stage_skip = [&](int k, int h) {               // thread 0 only
                int f, y0, x0;
                tile_of(k, f, y0, x0);
                mbar_expect_tx(&skf[h], SKH);
                tma_load_4d_stream(sbase + G::OFF_SK + h * SKH, &tin, 0, x0 - 1, y0 - 1 + h * HR, f, &skf[h], l2_evict_first_policy());
            };
            auto stage_lo = [&](int k) {                        // thread 0 only
                int f, y0, x0;
                tile_of(k, f, y0, x0);
                const bool sk2 = kSk2 && a.skip;
                mbar_expect_tx(&lof[k & 1], G::LOB + (sk2 ? G::SKB : 0));
                tma_load_4d_stream(sbase + G::OFF_LO + (k & 1) * G::LOB, &tlo, 0, x0 / 2 - 1, y0 / 2 - 1, f, &lof[k & 1],
                                   l2_evict_first_policy());
                if (sk2)
                    tma_load_4d_stream(sbase + G::OFF_SK + (k & 1) * G::SKBR, &tin, 0, x0 - 1, y0 - 1, f, &lof[k & 1],
                                       l2_evict_first_policy());
            };
            if (tid == 0) {
                if (mytiles > 0) {
                    if (!kSk2)
                        for (int h = 0; h < NH; ++h)
                            if (a.skip) stage_skip(0, h);
                    stage_lo(0);
                }
                if (mytiles > 1) stage_lo(1);
            }
            for (int k = 0; k < mytiles; ++k) {
                const int s = k % NIN;
                int f, y0, x0;
                tile_of(k, f, y0, x0);
                const int ly0 = y0 / 2 - 1, lx0 = x0 / 2 - 1;
                const uint8_t* lo = smem + G::OFF_LO + (k & 1) * G::LOB;
                const uint8_t* sk = smem + G::OFF_SK + (kSk2 ? (k & 1) * G::SKBR : 0);
                mbar_wait(&in_empty[s], ((k / NIN) & 1) ^ 1);
                mbar_wait(&lof[k & 1], (k >> 1) & 1);
                if (tid == 0) tr(k, 0);
                uint8_t* in = smem + s * G::INB;
#pragma unroll 1
                for (int h = 0; h < NH; ++h) {
                    if (a.skip && !kSk2) mbar_wait(&skf[h], k & 1);
                    // one item = one 2x2 block of outputs (the children of low-res
                    // pixel (bi, bj)) x one 8-channel chunk: the block reads its 3x3
                    // low-res neighbourhood once with the fixed (1/4, 3/4) weights
                    // (autodiff.py:258-287); clamping the source indices reproduces
                    // the reference's edge clamp.  Block rows 5h .. 5h+4 hold the
                    // tile's halo rows 9h .. 9h+8.
                    constexpr int BR = G::IR / 2 + 1, BC = G::IC / 2 + 1;
                    constexpr int BRH = BR / NH;                // block rows per piece
                    static_assert(BR % NH == 0 && (NH == 1 || BRH * 2 == HR + 1), "block rows per skip piece");
                    constexpr int HI = BRH * BC * G::NCI;       // items per piece
                    for (int it = h * HI + tid; it < ((kExp && (a.dbg & 1)) ? 0 : (h + 1) * HI); it += NPT) {
                        const int c = it % G::NCI, blk = it / G::NCI;
                        const int bil = blk / BC, bjl = blk - bil * BC;
                        const int bi = ly0 + bil, bj = lx0 + bjl;      // low-res pixel of the block
                        int rs[3], cs[3];
#pragma unroll
                        for (int u = 0; u < 3; ++u) {
                            rs[u] = min(max(min(max(bi - 1 + u, 0), hl - 1) - ly0, 0), G::LR - 1);
                            cs[u] = min(max(min(max(bj - 1 + u, 0), wl - 1) - lx0, 0), G::LC - 1);
                        }
                        uint4 qn[3][3], ob[4];
#pragma unroll
                        for (int u = 0; u < 3; ++u)
#pragma unroll
                            for (int v = 0; v < 3; ++v)
                                qn[u][v] = *reinterpret_cast<const uint4*>(lo + ((rs[v] * G::LC + cs[u]) * CIN + c * 8) * 2);
                        up2_block<T>(qn, ob);
#pragma unroll
                        for (int ab = 0; ab < 4; ++ab) {
                            const int aa = ab >> 1, bb = ab & 1;
                            const int yy = 2 * bi + aa, xx = 2 * bj + bb;       // output pixel
                            const int ti = yy - (y0 - 1), tj = xx - (x0 - 1);
                            if (ti < 0 || ti >= G::IR || tj < 0 || tj >= G::IC) continue;
                            const int p = ti * G::IC + tj;
                            uint4 q = make_uint4(0u, 0u, 0u, 0u);
                            if (yy >= 0 && xx >= 0 && yy < a.H && xx < a.W) {
                                q = ob[ab];
                                if (a.skip) {          // up2(low) + skip (network.py:189-194)
                                    const uint4 qs = *reinterpret_cast<const uint4*>(sk + (p * CIN + c * 8) * 2);
                                    q = add_packed<T>(q, qs);
                                }
                            }
                            *reinterpret_cast<uint4*>(in + c * G::PIN + p * 16) = q;
                        }
                    }
                    if (h == NH - 1) {
                        fence_proxy_async();
                        mbar_arrive(&in_full[s]);
                        if (tid == 0) tr(k, 1);
                    }
                    nbar_sync(1, NPT);             // all producers done with skip piece h (and, last, the low tile)
                    if (tid == 0) {
                        if (a.skip && !kSk2 && k + 1 < mytiles) stage_skip(k + 1, h);
                        if (h == NH - 1 && k + 2 < mytiles) stage_lo(k + 2);
                    }
                }
            }
        } else {
            // up2(low) + skip.  The TMA warp lands the skip tile straight into
            // the input buffer in[s] (chunk-planar, zero halo outside the
            // frame) and the low-res tile ((TH/2+2) x (TW/2+2) source pixels,
            // pixel-major) into one of two staging buffers, a tile ahead; the
            // producers add up2(low) in place.  Per-warp arrivals (lo_empty)
            // release the staging buffers, so no producer waits for a peer.
            const int hl = a.H / 2, wl = a.W / 2;
            for (int k = 0; k < mytiles; ++k) {
                const int s = k % NIN;
                int f, y0, x0;
                tile_of(k, f, y0, x0);
                const int ly0 = y0 / 2 - 1, lx0 = x0 / 2 - 1;
                const uint8_t* lo = smem + G::OFF_LO + (k & 1) * G::LOB;
                if (a.skip) mbar_wait(&skf[s], (k / NIN) & 1);             // skip landed in in[s] (in[s] free)
                else mbar_wait(&in_empty[s], ((k / NIN) & 1) ^ 1);
                mbar_wait(&lof[k & 1], (k >> 1) & 1);
                if (tid == 0) tr(k, 0);
                uint8_t* in = smem + s * G::INB;
                {
                    // one item = one 2x2 block of outputs (the children of low-res
                    // pixel (bi, bj)) x one 8-channel chunk: the block reads its 3x3
                    // low-res neighbourhood once with the fixed (1/4, 3/4) weights
                    // (autodiff.py:258-287); clamping the source indices reproduces
                    // the reference's edge clamp.
                    constexpr int BR = G::IR / 2 + 1, BC = G::IC / 2 + 1;
                    constexpr int NITEM = BR * BC * G::NCI;
                    for (int it = tid; it < ((kExp && (a.dbg & 1)) ? 0 : NITEM); it += NPT) {
                        const int c = it % G::NCI, blk = it / G::NCI;
                        const int bil = blk / BC, bjl = blk - bil * BC;
                        const int bi = ly0 + bil, bj = lx0 + bjl;      // low-res pixel of the block
                        int rs[3], cs[3];
#pragma unroll
                        for (int u = 0; u < 3; ++u) {
                            rs[u] = min(max(min(max(bi - 1 + u, 0), hl - 1) - ly0, 0), G::LR - 1);
                            cs[u] = min(max(min(max(bj - 1 + u, 0), wl - 1) - lx0, 0), G::LC - 1);
                        }
                        uint4 qn[3][3], ob[4];
#pragma unroll
                        for (int u = 0; u < 3; ++u)
#pragma unroll
                            for (int v = 0; v < 3; ++v)
                                qn[u][v] = *reinterpret_cast<const uint4*>(lo + ((rs[v] * G::LC + cs[u]) * CIN + c * 8) * 2);
                        up2_block<T>(qn, ob);
#pragma unroll
                        for (int ab = 0; ab < 4; ++ab) {
                            const int aa = ab >> 1, bb = ab & 1;
                            const int yy = 2 * bi + aa, xx = 2 * bj + bb;       // output pixel
                            const int ti = yy - (y0 - 1), tj = xx - (x0 - 1);
                            if (ti < 0 || ti >= G::IR || tj < 0 || tj >= G::IC) continue;
                            uint4* dst = reinterpret_cast<uint4*>(in + c * G::PIN + (ti * G::ICB + tj) * 16);
                            uint4 q = make_uint4(0u, 0u, 0u, 0u);
                            if (yy >= 0 && xx >= 0 && yy < a.H && xx < a.W)
                                q = a.skip ? add_packed<T>(ob[ab], *dst) : ob[ab];   // up2(low) + skip (network.py:189-194)
                            *dst = q;
                        }
                    }
                }
                fence_proxy_async();
                mbar_arrive(&in_full[s]);
                __syncwarp();
                if (lane == 0) mbar_arrive(&lo_empty[k & 1]);              // this warp is done with low tile k
                if (tid == 0) tr(k, 1);
            }
        }
    } else if (SRC == SRC_UP && warp == TW_) {
        // ------------------------------------------------------------ TMA warp (SRC_UP, in-place skip)
        if (!G::STAGED && lane == 0) {
            for (int k = 0; k < mytiles; ++k) {
                const int s = k % NIN;
                int f, y0, x0;
                tile_of(k, f, y0, x0);
                if (a.skip) {
                    mbar_wait(&in_empty[s], ((k / NIN) & 1) ^ 1);           // conv3 of tile k - NIN done with in[s]
                    mbar_expect_tx(&skf[s], G::TX_BYTES);
                    tma_load_5d_stream(sbase + s * G::INB, &tin, 0, x0 - 1, y0 - 1, 0, f, &skf[s], l2_evict_first_policy());
                }
                if (k >= 2) mbar_wait(&lo_empty[k & 1], ((k - 2) >> 1) & 1);
                mbar_expect_tx(&lof[k & 1], G::LOB);
                tma_load_4d_stream(sbase + G::OFF_LO + (k & 1) * G::LOB, &tlo, 0, x0 / 2 - 1, y0 / 2 - 1, f, &lof[k & 1],
                                   l2_evict_first_policy());
            }
        }
    } else if (warp >= MW && warp < MW + NMW) {
        // ------------------------------------------------------------ MMA issuer(s)
        const int mi = warp - MW;                   // kSplit: M-block of this conv3 issuer, NB = conv1
        if (lane == 0) {
            constexpr uint32_t idesc3 = umma_idesc(128, C3, Elem<T>::kUmmaFmt);
            constexpr uint32_t idesc1 = umma_idesc(128, C1, Elem<T>::kUmmaFmt);
            auto conv1 = [&](int j) {
                const int m = j % NMID, a1 = j & 1;
                mbar_wait(&mid_full[m], (j / NMID) & 1);
                mbar_wait(&a1_empty[a1], ((j >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint64_t db0 = umma_desc(sbase + G::OFF_W1, C1 * 16, 128);
                const uint64_t dm0 = umma_desc(sbase + G::OFF_MID + m * G::MIDB, G::PMID, G::TW * 16);
#pragma unroll
                for (int b = 0; b < NB; ++b)
#pragma unroll
                    for (int kk = 0; kk < C3 / 16; ++kk) {
                        const uint64_t db = db0 + (uint64_t)((kk * C1 * 32) >> 4);
                        if constexpr (G::MIDT) {
                            umma_f16_ts(tmem + G::ACC1 + (a1 * NB + b) * C1,
                                        tmem + G::ACCM + (m * NB + b) * G::MIDC / NB + kk * 8, db, idesc1, kk ? 1u : 0u);
                        } else {
                            const uint64_t da = dm0 + (uint64_t)(((2 * kk) * G::PMID + (b * 8) * 16) >> 4);
                            umma_f16(tmem + G::ACC1 + (a1 * NB + b) * C1, da, db, idesc1, kk ? 1u : 0u);
                        }
                    }
                umma_commit(&mid_empty[m]);
                umma_commit(&a1_full[a1]);
                tr(j, 3);
            };
            mbar_wait(wbar, 0);
            if (kSplit && mi == NB) {
                for (int j = 0; j < mytiles; ++j) conv1(j);
            } else for (int k = 0; k < mytiles; ++k) {
                const int s = k % NIN, a3 = k & 1;
                mbar_wait(&in_full[s], (k / NIN) & 1);
                mbar_wait(&a3_empty[a3], ((k >> 1) & 1) ^ 1);
                tc_fence_after();
                tr(k, 2);
                // Descriptors: one base per operand, every tap / block / K-step a
                // compile-time offset in 16-B units added to the start-address
                // field (building each descriptor in the loop costs ~70 issue
                // cycles per UMMA: the single MMA thread, not the tensor core,
                // was the limit; tools/umma_layout_probe.cu)
                const uint64_t da0 = umma_desc(sbase + s * G::INB, G::PIN, G::ICB * 16);
                const uint64_t db0 = umma_desc(sbase + G::OFF_W3, C3 * 16, 128);
                if (!(kExp && (a.dbg & 4))) {
                    // SRC_TENSOR kernels have the registers to unroll the taps
                    // (constant descriptor offsets: ~51 vs ~71 issue cycles per UMMA)
#pragma unroll (SRC == SRC_TENSOR ? 9 : 1)
                    for (int tap = 0; tap < 9; ++tap) {
                        const int dy = tap / 3, dx = tap - 3 * dy;
                        const uint64_t dat = da0 + (uint64_t)(dy * G::ICB + dx);           // 16-B units
                        const uint64_t dbt = db0 + (uint64_t)(tap * G::KK * C3 * 2);
#pragma unroll
                        for (int b = 0; b < NB; ++b)
#pragma unroll
                            for (int kk = 0; kk < G::KK; ++kk) {
                                if (kSplit && b != mi) continue;
                                // M-block b: 16 output rows x 8 px; core matrix i = output row i
                                const uint64_t da = dat + (uint64_t)(((2 * kk) * G::PIN + b * 8 * 16) >> 4);
                                const uint64_t db = dbt + (uint64_t)((kk * C3 * 32) >> 4);
                                umma_f16(tmem + G::ACC3 + (a3 * NB + b) * C3, da, db, idesc3, (tap | kk) ? 1u : 0u);
                            }
                    }
                }
                if (SRC == SRC_TENSOR) tr(k, 1);            // conv3 UMMAs issued (SRC_TENSOR: slot 1 is free)
                umma_commit(&in_empty[s]);
                umma_commit(&a3_full[a3]);
                if (!kSplit && k >= 1) conv1(k - 1);
            }
            if (!kSplit && mytiles > 0) conv1(mytiles - 1);
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const int q = warp & 3;                      // TMEM lane quadrant of this warp
        const int grp = (warp - EW0) >> 2;           // NG warps per quadrant split the columns
        const int m = q * 32 + lane;                 // M row == TMEM lane
        const int pi = m >> 3, pj = m & 7;           // pixel row / column inside an M-block
        const uint32_t tl = (uint32_t)(q * 32) << 16;
        auto epi1 = [&](int k) {
            const int a3 = k & 1, mm = k % NMID;
            mbar_wait(&a3_full[a3], (k >> 1) & 1);
            mbar_wait(&mid_empty[mm], ((k / NMID) & 1) ^ 1);
            tc_fence_after();
            if (warp == EW0 && lane == 0) tr(k, 4);
            uint8_t* mid = smem + G::OFF_MID + mm * G::MIDB;
            // this warp's NB * C3 / 32 accumulator slices: all TMEM loads in
            // flight before one wait (a wait per load serialised the epilogue)
            constexpr int NIT1 = NB * (C3 / 16) / NG;
            constexpr bool kPre = SRC == SRC_TENSOR;     // register room (no producer warps)
            uint32_t r1[kPre ? NIT1 : 1][16];
            if (kPre && !(kExp && (a.dbg & 2))) {
#pragma unroll
                for (int i = 0; i < NIT1; ++i) {
                    const int it = grp + NG * i, b = it / (C3 / 16), c0 = (it % (C3 / 16)) * 16;
                    tmem_ld16_nw(tmem + tl + G::ACC3 + (a3 * NB + b) * C3 + c0, r1[i]);
                }
                tmem_ld_wait();
            }
#pragma unroll
            for (int i = 0; i < NIT1; ++i) {
                if (kExp && (a.dbg & 2)) break;
                const int it = grp + NG * i, b = it / (C3 / 16), c0 = (it % (C3 / 16)) * 16;
                {
                    float v[16];
                    if constexpr (!kPre) {
                        tmem_ld16_nw(tmem + tl + G::ACC3 + (a3 * NB + b) * C3 + c0, r1[0]);
                        tmem_ld_wait();
                    }
#pragma unroll
                    for (int e = 0; e < 16; ++e) v[e] = __uint_as_float(r1[kPre ? i : 0][e]);
                    uint4 qv[2];
                    uint32_t* qp = &qv[0].x;
#pragma unroll
                    for (int e = 0; e < 8; ++e)
                        qp[e] = Elem<T>::pack(fmaxf(v[2 * e] + sb3[c0 + 2 * e], 0.f),
                                              fmaxf(v[2 * e + 1] + sb3[c0 + 2 * e + 1], 0.f));
                    if constexpr (G::MIDT) {
                        tmem_st8(tmem + tl + G::ACCM + (mm * NB + b) * G::MIDC / NB + c0 / 2, qp);
                    } else {
                        const int p = pi * G::TW + b * 8 + pj;
                        *reinterpret_cast<uint4*>(mid + (c0 / 8) * G::PMID + p * 16) = qv[0];
                        *reinterpret_cast<uint4*>(mid + (c0 / 8 + 1) * G::PMID + p * 16) = qv[1];
                    }
                }
            }
            if constexpr (G::MIDT) tmem_st_wait();
            fence_proxy_async();
            tc_fence_before();
            mbar_arrive(&a3_empty[a3]);
            mbar_arrive(&mid_full[mm]);
            if (warp == EW0 && lane == 0) tr(k, 5);
        };
        auto epi2 = [&](int j) {
            const int a1 = j & 1;
            int f, y0, x0;
            tile_of(j, f, y0, x0);
            mbar_wait(&a1_full[a1], (j >> 1) & 1);
            tc_fence_after();
            if (warp == EW0 && lane == 0) tr(j, 6);
            const int oy = y0 + pi;
            constexpr int NIT2 = NB * (C1 / 16) / NG;
            constexpr bool kPre = SRC == SRC_TENSOR;
            uint32_t r2[kPre ? NIT2 : 1][16];
            if (kPre && !(kExp && (a.dbg & 2))) {
#pragma unroll
                for (int i = 0; i < NIT2; ++i) {
                    const int it = grp + NG * i, b = it / (C1 / 16), c0 = (it % (C1 / 16)) * 16;
                    tmem_ld16_nw(tmem + tl + G::ACC1 + (a1 * NB + b) * C1 + c0, r2[i]);
                }
                tmem_ld_wait();
            }
#pragma unroll
            for (int i = 0; i < NIT2; ++i) {
                if (kExp && (a.dbg & 2)) break;
                const int it = grp + NG * i, b = it / (C1 / 16), c0 = (it % (C1 / 16)) * 16;
                const int ox = x0 + b * 8 + pj;
                const bool inside = oy < a.H && ox < a.W;
                {
                    float v[16];
                    if constexpr (!kPre) {
                        tmem_ld16_nw(tmem + tl + G::ACC1 + (a1 * NB + b) * C1 + c0, r2[0]);
                        tmem_ld_wait();
                    }
#pragma unroll
                    for (int e = 0; e < 16; ++e) v[e] = __uint_as_float(r2[kPre ? i : 0][e]);
#pragma unroll
                    for (int e = 0; e < 16; ++e) v[e] = fmaxf(v[e] + sb1[c0 + e], 0.f);
                    if (DST & DST_STORE) {
                        if (inside) {
                            uint4 qv[2];
                            uint32_t* qp = &qv[0].x;
#pragma unroll
                            for (int e = 0; e < 8; ++e) qp[e] = Elem<T>::pack(v[2 * e], v[2 * e + 1]);
                            if constexpr (DST & DST_PADREP) {
                                // chunk-planar (N, 2, H + 2, W + 2, 8): the consumer's TMA
                                // box rows are then 10 contiguous pixels of one chunk
                                static_assert(C1 == 16, "DST_PADREP stores one 16-channel slice as 2 chunk planes");
                                const int wp = a.W + 2;
                                const int64_t cpl = (int64_t)(a.H + 2) * wp * 8;      // one chunk plane
                                T* fb = reinterpret_cast<T*>(a.out) + (int64_t)f * 2 * cpl;
                                const int ys[2] = {oy + 1, oy == 0 ? 0 : (oy == a.H - 1 ? a.H + 1 : -1)};
                                const int xs[2] = {ox + 1, ox == 0 ? 0 : (ox == a.W - 1 ? a.W + 1 : -1)};
#pragma unroll
                                for (int iy = 0; iy < 2; ++iy)
#pragma unroll
                                    for (int ix = 0; ix < 2; ++ix)
                                        if (ys[iy] >= 0 && xs[ix] >= 0) {
                                            T* px = fb + ((int64_t)ys[iy] * wp + xs[ix]) * 8;
                                            *reinterpret_cast<uint4*>(px) = qv[0];
                                            *reinterpret_cast<uint4*>(px + cpl) = qv[1];
                                        }
                            } else {
                                // one 256-bit store: a full 32-B sector per lane
                                st_global_256(reinterpret_cast<T*>(a.out) + (((int64_t)f * a.H + oy) * a.W + ox) * C1 + c0,
                                              qv[0], qv[1]);
                            }
                        }
                    }
                    if (DST & DST_POOL) {
                        // 2x2 average pool as a transposing reduction: the x-partner
                        // (lane^1) and y-partner (lane^8) each take half of the
                        // channels, 12 shuffles instead of 32; every thread of the
                        // 2x2 group then owns 4 channels of the pooled pixel.
                        const bool xo = pj & 1, yo = pi & 1;
                        float h8[8], h4[4];
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            const float send = xo ? v[e] : v[e + 8];
                            const float keep = xo ? v[e + 8] : v[e];
                            h8[e] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
                        }
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float send = yo ? h8[e] : h8[e + 4];
                            const float keep = yo ? h8[e + 4] : h8[e];
                            h4[e] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
                        }
                        if (inside) {
                            const int H2 = a.H / 2, W2 = a.W / 2;
                            const int cb = c0 + (xo ? 8 : 0) + (yo ? 4 : 0);
                            uint2 qv = make_uint2(Elem<T>::pack(h4[0] * 0.25f, h4[1] * 0.25f),
                                                  Elem<T>::pack(h4[2] * 0.25f, h4[3] * 0.25f));
                            *reinterpret_cast<uint2*>(reinterpret_cast<T*>(a.pool) +
                                                      (((int64_t)f * H2 + oy / 2) * W2 + ox / 2) * C1 + cb) = qv;
                        }
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(&a1_empty[a1]);
            if (warp == EW0 && lane == 0) tr(j, 7);
        };
        for (int k = 0; k < mytiles; ++k) {
            epi1(k);
            if (k >= 1) epi2(k - 1);
        }
        if (mytiles > 0) epi2(mytiles - 1);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == EW0) tmem_dealloc<G::TCOLS>(tmem);
    if (kExp && a.trace && tid == 0 && blockIdx.x < 256) a.trace[257 + 2 * blockIdx.x] = globaltimer_ns();
}

// ------------------------------------------------------------- level 0 decoder, polyphase (tcgen05)
// dec0 = head(relu(dec1(relu(conv3(up2(D1)))))) evaluated on the level-1
// grid: up2 with an edge clamp is up2 of the replicate-padded D1 (written by
// lv1_dec, DST_PADREP), so conv3(up2(D1)) is, for each of the 4 output
// phases (a, b), a 3x3 convolution of D1 with combined taps (pack_f16).  One
// M-block = 16 x 8 level-1 pixels (128 lanes); N = 4 phases x 16 channels:
//   conv3  9 UMMAs  N = 64, K = 16   (A: shifted views of the D1 tile)
//   dec1   4 UMMAs  N = 64, K = 64   (A in TMEM, phase-block-diagonal B)
//   head   4 UMMAs  N = 16, K = 64   (A in TMEM)
// Epilogues: bias + ReLU + pack into TMEM (the next A), and the head's 16
// values (4 phases x 4 channels) into the fp16 Y planes.  The zero padding
// of the level-0 conv differs from the replicate padding only on the outer
// ring of level-0 pixels, which dec0_ring_kernel recomputes exactly.
// Warps: 0 TMA, 1-4 conv3 epilogue, 5-8 dec1 epilogue, 9-12 head epilogue
// (one warp per TMEM lane quadrant in each group), 13-15 one MMA issuer per
// GEMM.  Every TMEM stage is double buffered and every stage has its own
// warps, so the MMA/epilogue round trips of consecutive tiles overlap.
struct Dec0pArgs {
    const void* w3;      // umma [9][1][2][64][8]
    const void* w1;      // umma [1][4][2][64][8]
    const void* wh;      // umma [1][4][2][16][8]
    const float* b3;     // (16,)  l0.dec3 bias (replicated per phase)
    const float* b1;     // (16,)  l0.dec1 bias
    const float* bh;     // (4,)   head bias
    __half* y;           // (N, 4, H0, W0)
    int H1, W1, H0, W0;
    long long* trace;    // experiments only (NSM_DEC0_TRACE): CTA 0 per-tile clock64 events
};
constexpr int D0P_IR = 18, D0P_IC = 10, D0P_NIN = 4;
constexpr int D0P_PIN = D0P_IR * D0P_IC * 16, D0P_INB = round128(2 * D0P_PIN);
constexpr int D0P_W3B = 9 * 2 * 64 * 16, D0P_W1B = 4 * 2 * 64 * 16, D0P_WHB = 4 * 2 * 16 * 16;
constexpr int D0P_OFF_W3 = D0P_NIN * D0P_INB, D0P_OFF_W1 = D0P_OFF_W3 + D0P_W3B, D0P_OFF_WH = D0P_OFF_W1 + D0P_W1B;
constexpr int D0P_OFF_B = D0P_OFF_WH + D0P_WHB, D0P_OFF_BAR = D0P_OFF_B + 48 * 4;
constexpr int D0P_SMEM = D0P_OFF_BAR + 256;
constexpr int D0P_THREADS = 512;
constexpr int D0P_ACC3 = 0, D0P_ACC1 = 128, D0P_ACCH = 256, D0P_MID = 288, D0P_MID2 = 352;   // MID/MID2: 2 x 32

template <typename T>
__global__ void __launch_bounds__(D0P_THREADS, 1) dec0p_kernel(const __grid_constant__ Dec0pArgs a,
                                                       const __grid_constant__ CUtensorMap tin, int total) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + D0P_OFF_BAR);
    uint64_t* in_full = bar + 0;     // [4]
    uint64_t* in_empty = bar + 4;    // [4]
    uint64_t* a3_full = bar + 8;     // [2]
    uint64_t* a3_empty = bar + 10;
    uint64_t* a1_full = bar + 12;
    uint64_t* a1_empty = bar + 14;
    uint64_t* ah_full = bar + 16;
    uint64_t* ah_empty = bar + 18;
    uint64_t* mid_full = bar + 20;   // [2]
    uint64_t* mid_empty = bar + 22;
    uint64_t* mid2_full = bar + 24;
    uint64_t* mid2_empty = bar + 26;
    uint64_t* wbar = bar + 28;
    uint32_t* tptr = reinterpret_cast<uint32_t*>(smem + D0P_OFF_BAR + 240);
    float* sbias = reinterpret_cast<float*>(smem + D0P_OFF_B);     // b3[16] b1[16] bh[4]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t sbase = smem_u32(smem);
    const int ntx = (a.W1 + 7) / 8, nty = (a.H1 + 15) / 16;
    const int mytiles = (int)blockIdx.x < total ? (total - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
    auto tile_of = [&](int k, int& f, int& y0, int& x0) {   // level-1 tile origin
        const int t = blockIdx.x + k * gridDim.x;
        x0 = (t % ntx) * 8;
        y0 = ((t / ntx) % nty) * 16;
        f = t / (ntx * nty);
    };
    auto tr = [&](int k, int ev) {       // experiments: CTA 0's per-tile timeline
        if (kExp && a.trace && blockIdx.x == 0 && k < 64) a.trace[k * 8 + ev] = clock64();
    };
    if (tid == 0) pdl_trigger();
    if (warp == 13) tmem_alloc<512>(tptr);
    if (tid == 0) {
        for (int i = 0; i < D0P_NIN; ++i) {
            mbar_init(&in_full[i], 1);
            mbar_init(&in_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {                 // epilogue arrivals: every thread of a 4-warp group
            mbar_init(&a3_full[i], 1);
            mbar_init(&a3_empty[i], 128);
            mbar_init(&a1_full[i], 1);
            mbar_init(&a1_empty[i], 128);
            mbar_init(&ah_full[i], 1);
            mbar_init(&ah_empty[i], 128);
            mbar_init(&mid_full[i], 128);
            mbar_init(&mid_empty[i], 1);
            mbar_init(&mid2_full[i], 128);
            mbar_init(&mid2_empty[i], 1);
        }
        mbar_init(wbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        mbar_expect_tx(wbar, D0P_W3B + D0P_W1B + D0P_WHB);
        bulk_g2s(sbase + D0P_OFF_W3, a.w3, D0P_W3B, wbar);
        bulk_g2s(sbase + D0P_OFF_W1, a.w1, D0P_W1B, wbar);
        bulk_g2s(sbase + D0P_OFF_WH, a.wh, D0P_WHB, wbar);
    }
    if (tid < 16) sbias[tid] = a.b3[tid];
    else if (tid < 32) sbias[tid] = a.b1[tid - 16];
    else if (tid < 36) sbias[tid] = a.bh[tid - 32];
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tptr;
    pdl_wait();

    if (warp == 0) {
        // ------------------------------------------------------------ TMA
        if (lane == 0) {
            for (int k = 0; k < mytiles; ++k) {
                const int s = k % D0P_NIN;
                mbar_wait(&in_empty[s], ((k / D0P_NIN) & 1) ^ 1);
                int f, y0, x0;
                tile_of(k, f, y0, x0);
                mbar_expect_tx(&in_full[s], 2 * D0P_PIN);
                // padded coordinates: real (y0 - 1, x0 - 1) is padded (y0, x0)
                tma_load_3d_stream(sbase + s * D0P_INB, &tin, 8 * x0, y0, 2 * f, &in_full[s], l2_evict_first_policy());   // both chunk planes
                tr(k, 0);
            }
        }
    } else if (warp >= 13) {
        // ------------------------------------------------------------ MMA issuers, one per GEMM
        if (lane == 0) {
            constexpr uint32_t id64 = umma_idesc(128, 64, Elem<T>::kUmmaFmt);
            constexpr uint32_t id16 = umma_idesc(128, 16, Elem<T>::kUmmaFmt);
            mbar_wait(wbar, 0);
            if (warp == 13) {
                const uint64_t dw3 = umma_desc(sbase + D0P_OFF_W3, 64 * 16, 128);
                for (int k = 0; k < mytiles; ++k) {                  // conv3(k)
                    const int s = k % D0P_NIN, a3 = k & 1;
                    mbar_wait(&in_full[s], (k / D0P_NIN) & 1);
                    mbar_wait(&a3_empty[a3], ((k >> 1) & 1) ^ 1);
                    tc_fence_after();
                    const uint64_t da0 = umma_desc(sbase + s * D0P_INB, D0P_PIN, D0P_IC * 16);
#pragma unroll
                    for (int tap = 0; tap < 9; ++tap)
                        umma_f16(tmem + D0P_ACC3 + a3 * 64, da0 + (uint64_t)((tap / 3) * D0P_IC + tap % 3),
                                 dw3 + (uint64_t)(tap * 128), id64, tap ? 1u : 0u);
                    umma_commit(&in_empty[s]);
                    umma_commit(&a3_full[a3]);
                    tr(k, 1);
                }
            } else if (warp == 14) {
                const uint64_t dw1 = umma_desc(sbase + D0P_OFF_W1, 64 * 16, 128);
                for (int j = 0; j < mytiles; ++j) {                  // dec1(j)
                    const int a1 = j & 1;
                    mbar_wait(&mid_full[a1], (j >> 1) & 1);
                    mbar_wait(&a1_empty[a1], ((j >> 1) & 1) ^ 1);
                    tc_fence_after();
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        umma_f16_ts(tmem + D0P_ACC1 + a1 * 64, tmem + D0P_MID + a1 * 32 + kk * 8, dw1 + (uint64_t)(kk * 128),
                                    id64, kk ? 1u : 0u);
                    umma_commit(&mid_empty[a1]);
                    umma_commit(&a1_full[a1]);
                    tr(j, 3);
                }
            } else {
                const uint64_t dwh = umma_desc(sbase + D0P_OFF_WH, 16 * 16, 128);
                for (int j = 0; j < mytiles; ++j) {                  // head(j)
                    const int ah = j & 1;
                    mbar_wait(&mid2_full[ah], (j >> 1) & 1);
                    mbar_wait(&ah_empty[ah], ((j >> 1) & 1) ^ 1);
                    tc_fence_after();
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        umma_f16_ts(tmem + D0P_ACCH + ah * 16, tmem + D0P_MID2 + ah * 32 + kk * 8, dwh + (uint64_t)(kk * 32),
                                    id16, kk ? 1u : 0u);
                    umma_commit(&mid2_empty[ah]);
                    umma_commit(&ah_full[ah]);
                    tr(j, 5);
                }
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const int q = warp & 3;                               // TMEM lane quadrant
        const int m = q * 32 + lane, pi = m >> 3, pj = m & 7;
        const uint32_t tl = (uint32_t)(q * 32) << 16;
        const int64_t plane = (int64_t)a.H0 * a.W0;
        // bias + ReLU of 64 accumulator columns -> 32 packed columns of the next A
        auto relu_to_tmem = [&](uint32_t src, uint32_t dst, const float* bias) {
            uint32_t r[4][16];
#pragma unroll
            for (int h = 0; h < 4; ++h) tmem_ld16_nw(src + h * 16, r[h]);
            tmem_ld_wait();
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                uint32_t pk[8];
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    pk[e] = Elem<T>::pack(fmaxf(__uint_as_float(r[h][2 * e]) + bias[(2 * e) & 15], 0.f),
                                          fmaxf(__uint_as_float(r[h][2 * e + 1]) + bias[(2 * e + 1) & 15], 0.f));
                tmem_st8(dst + h * 8, pk);
            }
            tmem_st_wait();
        };
        if (warp <= 4) {
            for (int k = 0; k < mytiles; ++k) {                      // conv3(k) -> MID[k & 1]
                const int a3 = k & 1;
                mbar_wait(&a3_full[a3], (k >> 1) & 1);
                mbar_wait(&mid_empty[a3], ((k >> 1) & 1) ^ 1);
                tc_fence_after();
                if (warp == 1 && lane == 0) tr(k, 7);
                relu_to_tmem(tmem + tl + D0P_ACC3 + a3 * 64, tmem + tl + D0P_MID + a3 * 32, sbias);
                tc_fence_before();
                mbar_arrive(&a3_empty[a3]);
                mbar_arrive(&mid_full[a3]);
                if (warp == 1 && lane == 0) tr(k, 2);
            }
        } else if (warp <= 8) {
            for (int k = 0; k < mytiles; ++k) {                      // dec1(k) -> MID2[k & 1]
                const int a1 = k & 1;
                mbar_wait(&a1_full[a1], (k >> 1) & 1);
                mbar_wait(&mid2_empty[a1], ((k >> 1) & 1) ^ 1);
                tc_fence_after();
                relu_to_tmem(tmem + tl + D0P_ACC1 + a1 * 64, tmem + tl + D0P_MID2 + a1 * 32, sbias + 16);
                tc_fence_before();
                mbar_arrive(&a1_empty[a1]);
                mbar_arrive(&mid2_full[a1]);
                if (warp == 5 && lane == 0) tr(k, 4);
            }
        } else {
            for (int j = 0; j < mytiles; ++j) {                      // head(j) -> Y
                const int ah = j & 1;
                int f, y0, x0;
                tile_of(j, f, y0, x0);
                mbar_wait(&ah_full[ah], (j >> 1) & 1);
                tc_fence_after();
                uint32_t r[16];                                      // phases (a, b) x 4 channels
                tmem_ld16_nw(tmem + tl + D0P_ACCH + ah * 16, r);
                tmem_ld_wait();
                tc_fence_before();
                mbar_arrive(&ah_empty[ah]);
                if (warp == 9 && lane == 0) tr(j, 6);
                // level-0 pixels (oy, ox) and (oy, ox + 1); dec0_ring_kernel
                // overwrites the outer ring afterwards
                const int ox = 2 * (x0 + pj);
#pragma unroll
                for (int ph = 0; ph < 2; ++ph) {
                    const int oy = 2 * (y0 + pi) + ph;
                    if (oy < a.H0 && ox < a.W0) {
                        __half* yp = a.y + (int64_t)f * 4 * plane + (int64_t)oy * a.W0 + ox;
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const float v0 = __uint_as_float(r[ph * 8 + c]) + sbias[32 + c];
                            const float v1 = __uint_as_float(r[ph * 8 + 4 + c]) + sbias[32 + c];
                            if (ox + 1 < a.W0) *reinterpret_cast<__half2*>(yp + c * plane) = __floats2half2_rn(v0, v1);
                            else yp[c * plane] = __float2half_rn(v0);
                        }
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 13) tmem_dealloc<512>(tmem);
}

// The outer ring of level-0 pixels (rows 0 and H0-1, columns 0 and W0-1),
// where the level-0 conv's zero padding differs from dec0p's replicate
// padding: l0.dec3 (zero padding of the up2 image), l0.dec1 and the head
// straight from D1 (autodiff.py:258-287; network.py:199-205), overwriting
// dec0p's values.  One warp per run of 30 pixels along one side: the up2
// values of the two image lines the side's taps touch are staged in shared
// memory for 34 positions (chunk-planar, 16-bit like every level-0 operand),
// and the 6 in-image taps are m16n8k16 MMAs on ldmatrix views shifted by
// -1, 0, +1 positions (the sliding window of conv3_strip16); dec1 and the
// head reuse the accumulators as A fragments.  The taps outside the image
// are simply not issued, which is the zero padding.
constexpr int kRingPos = 34, kRingWarpBytes = 2 * 2 * kRingPos * 16;
template <typename T>
__global__ void __launch_bounds__(128) dec0_ring_kernel(const T* __restrict__ d1p, int H1, int W1, int H0, int W0,
                                                        const uint2* __restrict__ wb3, const uint2* __restrict__ wb1,
                                                        const uint2* __restrict__ wbh, const float* __restrict__ b3,
                                                        const float* __restrict__ b1, const float* __restrict__ bh,
                                                        __half* __restrict__ y, int nf) {
    __shared__ __align__(128) uint8_t su[4 * kRingWarpBytes];
    if (threadIdx.x == 0) pdl_trigger();
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    uint32_t B3[9][2][2], B1[2][2], BH[2];
    float bias3[2][2], bias1[2][2], biash[2];
#pragma unroll
    for (int tap = 0; tap < 9; ++tap)
#pragma unroll
        for (int n = 0; n < 2; ++n) {
            const uint2 v = __ldg(wb3 + (tap * 2 + n) * 32 + lane);
            B3[tap][n][0] = v.x;
            B3[tap][n][1] = v.y;
        }
#pragma unroll
    for (int n = 0; n < 2; ++n) {
        const uint2 v = __ldg(wb1 + n * 32 + lane);
        B1[n][0] = v.x;
        B1[n][1] = v.y;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            bias3[n][e] = __ldg(b3 + n * 8 + 2 * t + e);
            bias1[n][e] = __ldg(b1 + n * 8 + 2 * t + e);
        }
    }
    {
        const uint2 v = __ldg(wbh + lane);
        BH[0] = v.x;
        BH[1] = v.y;
        biash[0] = t < 2 ? __ldg(bh + 2 * t) : 0.f;
        biash[1] = t < 2 ? __ldg(bh + 2 * t + 1) : 0.f;
    }
    pdl_wait();
    uint8_t* u = su + wib * kRingWarpBytes;               // [line][chunk][position] x 16 B
    const uint32_t ub = smem_u32(u);
    const int Wp = W1 + 2;
    const int64_t plane = (int64_t)H0 * W0;
    const int runs_h = (W0 + 29) / 30, runs_v = (H0 - 2 + 29) / 30, per_frame = 2 * (runs_h + runs_v);
    const int nwarps = gridDim.x * 4;
    for (int item = blockIdx.x * 4 + wib; item < per_frame * nf; item += nwarps) {
        const int f = item / per_frame;
        int r = item - f * per_frame, side, run;
        if (r < 2 * runs_h) side = r / runs_h, run = r % runs_h;              // 0 top, 1 bottom
        else r -= 2 * runs_h, side = 2 + r / runs_v, run = r % runs_v;         // 2 left, 3 right
        const bool horiz = side < 2;
        // output row m (0..31) is position p0 - 1 + m along the side (a column,
        // or a row in 1..H0-2); staged position j is p0 - 2 + j
        const int p0 = horiz ? run * 30 : run * 30 + 1;
        const int extent = horiz ? W0 : H0;
        // D1 is chunk-planar (N, 2, H1 + 2, W1 + 2, 8): one uint4 per pixel and chunk
        const int64_t cpl = (int64_t)(H1 + 2) * Wp;
        const uint4* x = reinterpret_cast<const uint4*>(d1p) + (int64_t)f * 2 * cpl;
        __syncwarp();                                    // the previous run's ldmatrix reads are done
        for (int it = lane; it < 2 * 2 * kRingPos; it += 32) {
            const int j = it % kRingPos, kc = it / kRingPos, k = kc >> 1, c = kc & 1;
            const int sp = p0 - 2 + j;
            const int line = side == 0 ? k : side == 1 ? H0 - 2 + k : side == 2 ? k : W0 - 2 + k;
            const int rr = horiz ? line : sp, cc = horiz ? sp : line;
            uint4 q = make_uint4(0u, 0u, 0u, 0u);
            if (sp >= 0 && sp < extent) {                // 0 outside the image: the conv's zero padding
                const float sy = fminf(fmaxf((rr + 0.5f) * 0.5f - 0.5f, 0.f), (float)(H1 - 1));
                const float sx = fminf(fmaxf((cc + 0.5f) * 0.5f - 0.5f, 0.f), (float)(W1 - 1));
                const int y0 = (int)sy, x0 = (int)sx;
                const float wy = sy - y0, wx = sx - x0;
                const int y1 = min(y0 + 1, H1 - 1), x1 = min(x0 + 1, W1 - 1);
                const float cw[4] = {(1.f - wy) * (1.f - wx), (1.f - wy) * wx, wy * (1.f - wx), wy * wx};
                float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int cr = 0; cr < 4; ++cr) {
                    const uint4 s4 = __ldg(x + (int64_t)c * cpl + (int64_t)((cr >> 1 ? y1 : y0) + 1) * Wp + ((cr & 1 ? x1 : x0) + 1));
                    const uint32_t w4[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float2 h2 = Elem<T>::unpack(w4[e]);
                        v[2 * e] = fmaf(cw[cr], h2.x, v[2 * e]);
                        v[2 * e + 1] = fmaf(cw[cr], h2.y, v[2 * e + 1]);
                    }
                }
                q = make_uint4(Elem<T>::pack(v[0], v[1]), Elem<T>::pack(v[2], v[3]), Elem<T>::pack(v[4], v[5]),
                               Elem<T>::pack(v[6], v[7]));
            }
            *reinterpret_cast<uint4*>(u + (kc * kRingPos + j) * 16) = q;
        }
        __syncwarp();
        // A fragment rows: position m0 + row + d + 1 of line k (both chunks)
        const int lm = lane >> 3, li = lane & 7;
        const uint32_t a_off = ((lm >> 1) * kRingPos + li + 8 * (lm & 1)) * 16;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
            float acc[2][4];
            bool first = true;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int across = (side == 0 || side == 2) ? k + 1 : k;      // dy (horiz) / dx (vert) of line k
#pragma unroll
                for (int d = -1; d <= 1; ++d) {
                    const int tap = horiz ? across * 3 + d + 1 : (d + 1) * 3 + across;
                    uint32_t A[4];
                    ldsm_x4(ub + a_off + ((2 * k) * kRingPos + mt * 16 + d + 1) * 16, A);
#pragma unroll
                    for (int n = 0; n < 2; ++n) {
                        if (first)
                            mma16816_c<T>(acc[n], A, B3[tap][n][0], B3[tap][n][1], bias3[n][0], bias3[n][1],
                                          bias3[n][0], bias3[n][1]);
                        else
                            mma16816<T>(acc[n], A, B3[tap][n][0], B3[tap][n][1]);
                    }
                    first = false;
                }
            }
            uint32_t a1[4], a2[4];
            relu_pack_a<T>(acc, a1);
            float hv[2][4];
#pragma unroll
            for (int n = 0; n < 2; ++n)
                mma16816_c<T>(hv[n], a1, B1[n][0], B1[n][1], bias1[n][0], bias1[n][1], bias1[n][0], bias1[n][1]);
            relu_pack_a<T>(hv, a2);
            float yh[4];
            mma16816_c<T>(yh, a2, BH[0], BH[1], biash[0], biash[1], biash[0], biash[1]);
            // head channels 2t, 2t+1 (t < 2) of rows g, g + 8
            if (t < 2) {
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const int m = mt * 16 + g + 8 * hh, sp = p0 - 1 + m;
                    if (m >= 1 && m <= 30 && (horiz ? sp < W0 : sp <= H0 - 2)) {
                        const int R = horiz ? (side == 0 ? 0 : H0 - 1) : sp, C = horiz ? sp : (side == 2 ? 0 : W0 - 1);
                        __half* yp = y + ((int64_t)f * 4 + 2 * t) * plane + (int64_t)R * W0 + C;
                        yp[0] = __float2half_rn(yh[2 * hh]);
                        yp[plane] = __float2half_rn(yh[2 * hh + 1]);
                    }
                }
            }
        }
    }
}

// first_bad[i] = INT64_MAX ("no frustum error"), PDL-chained so that enc0's
// prologue overlaps it
__global__ void fill_first_bad(int64_t* p, int n, int* tile_ctr) {
    // trigger only after the grid dependency resolved: enc0's TMA warp
    // streams the G-buffer before its own griddepcontrol.wait, so whatever
    // wrote the G-buffer must be complete and visible once this kernel
    // lets enc0 start
    pdl_wait();
    pdl_trigger();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = INT64_MAX;
    if (tile_ctr && i < 2) tile_ctr[i] = 0;     // enc0's dynamic tile counters (first launch)
}

// ------------------------------------------------------------------ host side
int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    }
    return n;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (the
// library links cudart statically and never links libcuda directly).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    }
    return fn;
}

// 5-D view of an NHWC 16-bit tensor (8 elems, x, y, chunk, frame) whose
// TMA box lands in SMEM as [chunk][y][x][8], i.e. the chunk-planar tile.
bool encode_nhwc_map(const void* base, bool bf16, int C, int H, int W, int nf, int box_w, int box_h,
                     CUtensorMap* m) {
    auto enc = tensor_map_encoder();
    if (!enc || ((uintptr_t)base % 16)) return false;
    const cuuint64_t dims[5] = {8, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)(C / 8), (cuuint64_t)nf};
    const cuuint64_t strides[4] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, 16, (cuuint64_t)H * W * C * 2};
    const cuuint32_t box[5] = {8, (cuuint32_t)box_w, (cuuint32_t)box_h, (cuuint32_t)(C / 8), 1};
    const cuuint32_t es[5] = {1, 1, 1, 1, 1};
    return enc(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 5,
               const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 3-D view (x * 8 + channel, y, frame * 2 + chunk) of a chunk-planar 16-bit
// tensor (N, 2, H, W, 8): a box row is box_w contiguous pixels of one chunk
// (box_w * 16 B), not one 16-B pixel chunk as in encode_nhwc_map.
bool encode_cplanar_map(const void* base, bool bf16, int H, int W, int nf, int box_w, int box_h, CUtensorMap* m) {
    auto enc = tensor_map_encoder();
    if (!enc || ((uintptr_t)base % 16)) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)W * 8, (cuuint64_t)H, (cuuint64_t)nf * 2};
    const cuuint64_t strides[2] = {(cuuint64_t)W * 16, (cuuint64_t)H * W * 16};
    const cuuint32_t box[3] = {(cuuint32_t)box_w * 8, (cuuint32_t)box_h, 2};
    const cuuint32_t es[3] = {1, 1, 1};
    return enc(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3,
               const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 4-D pixel-major view (C elems, x, y, frame) of an NHWC 16-bit tensor.
bool encode_nhwc_map4(const void* base, bool bf16, int C, int H, int W, int nf, int box_w, int box_h,
                      CUtensorMap* m, int pad = 0) {
    // pad: the tensor lives inside a (H + 2 pad, W + 2 pad) allocation (the map
    // covers the interior, so out-of-range boxes still read zeros)
    auto enc = tensor_map_encoder();
    const int Wa = W + 2 * pad, Ha = H + 2 * pad;
    base = (const char*)base + ((size_t)pad * Wa + pad) * C * 2;
    if (!enc || ((uintptr_t)base % 16)) return false;
    const cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)nf};
    const cuuint64_t strides[3] = {(cuuint64_t)C * 2, (cuuint64_t)Wa * C * 2, (cuuint64_t)Ha * Wa * C * 2};
    const cuuint32_t box[4] = {(cuuint32_t)C, (cuuint32_t)box_w, (cuuint32_t)box_h, 1};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    return enc(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4,
               const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 3-D view (x * 8 + element, y, frame * 3 + chunk) of the chunk-planar
// s2d tensor (N, 3, H0, W0, 8); a box is 22 pixels x 18 rows x 3 chunks
bool encode_s2d24_map(const void* base, bool bf16, int H0, int W0, int nf, CUtensorMap* m) {
    auto enc = tensor_map_encoder();
    if (!enc || ((uintptr_t)base % 16)) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)W0 * 8, (cuuint64_t)H0, (cuuint64_t)nf * 3};
    const cuuint64_t strides[2] = {(cuuint64_t)W0 * 16, (cuuint64_t)H0 * W0 * 16};
    const cuuint32_t box[3] = {(cuuint32_t)S24_BOXW * 8, (cuuint32_t)E0_IR, 3};
    const cuuint32_t es[3] = {1, 1, 1};
    return enc(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3,
               const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <typename T, int CIN, int C3, int C1, int SRC, int DST, int NB, int NIN, int NMID>
nsm_status launch_level(const LevelArgs& a, int nf, cudaStream_t st, const char* name) {
    using G = LvGeom<CIN, C3, C1, NB, NIN, NMID, SRC == SRC_UP>;
    static_assert(G::SMEM <= 232448, "level kernel exceeds 227 KB of shared memory");
    constexpr int NPW = SRC == SRC_TENSOR ? 1 : 12;
    auto k = level_kernel<T, CIN, C3, C1, SRC, DST, NB, NIN, NMID, NPW>;
    static PerDevice attr;
    if (attr.first()) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
    CUtensorMap tin, tlo;
    memset(&tin, 0, sizeof tin);
    memset(&tlo, 0, sizeof tlo);
    constexpr bool bf = std::is_same<T, __nv_bfloat16>::value;
    bool ok = true;
    if (SRC == SRC_TENSOR) {
        ok = encode_nhwc_map(a.x, bf, CIN, a.H, a.W, nf, G::IC, G::IR, &tin);
    } else {
        ok = encode_nhwc_map4(a.x, bf, CIN, a.H / 2, a.W / 2, nf, G::LC, G::LR, &tlo);
        if (a.skip)
            ok = ok && (G::STAGED ? encode_nhwc_map4(a.skip, bf, CIN, a.H, a.W, nf, G::IC, G::IR, &tin)
                                  : encode_nhwc_map(a.skip, bf, CIN, a.H, a.W, nf, G::ICB, G::IRB, &tin));
    }
    if (!ok) return fail(NSM_ERR_CUDA, "%s: TMA tensor map encoding failed", name);
    const int total = ((a.W + G::TW - 1) / G::TW) * ((a.H + G::TH - 1) / G::TH) * nf;
    const int grid = std::min(total, num_sms());      // TMEM: 512 columns -> one CTA per SM
    const_cast<LevelArgs&>(a).dbg = env_int("NSM_LEVEL_DBG", 0);
    static long long* trace_buf = nullptr;
    bool trace = false;
#ifdef NSM_EXPERIMENTS
    static const char* trace_name = getenv("NSM_LEVEL_TRACE");
    trace = trace_name && !strcmp(trace_name, name);
    if (trace) {
        if (!trace_buf) cudaMalloc(&trace_buf, 1024 * sizeof(long long));
        cudaMemsetAsync(trace_buf, 0, 1024 * sizeof(long long), st);
    }
#endif
    const_cast<LevelArgs&>(a).trace = trace ? trace_buf : nullptr;
    NSM_PROF(name, st);
    launch_pdl(k, dim3(grid), dim3(lv_threads<SRC, NB, NPW>()), G::SMEM, st, a, tin, tlo, total);
    if (trace) {   // experiments only: print CTA 0's timeline (us at 1.965 GHz) and stall the stream
        static long long h[1024];
        cudaMemcpyAsync(h, trace_buf, sizeof h, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        {
            long long s0 = 0, e1 = 0;
            double dsum = 0, dmin = 1e30, dmax = 0;
            int nc = 0;
            for (int c = 0; c < 256; ++c) {
                const long long a0 = h[256 + 2 * c], a1 = h[257 + 2 * c];
                if (!a0 || !a1) continue;
                ++nc;
                if (!s0 || a0 < s0) s0 = a0;
                if (a1 > e1) e1 = a1;
                const double d = (a1 - a0) / 1e3;
                dsum += d, dmin = std::min(dmin, d), dmax = std::max(dmax, d);
            }
            fprintf(stderr, "%s CTAs %d: first start -> last end %.2f us; CTA span min/avg/max %.2f/%.2f/%.2f us\n", name,
                    nc, (e1 - s0) / 1e3, dmin, dsum / std::max(nc, 1), dmax);
        }
        long long t0 = 0;
        for (long long v : h) if (v && (!t0 || v < t0)) t0 = v;
        fprintf(stderr, "%s CTA0 (us): tile prod_start prod_done mma3_issue mma1_issued epi1_start epi1_end epi2_start epi2_end\n", name);
        for (int k = 0; k < 32; ++k) {
            if (!h[k * 8 + 2]) break;
            fprintf(stderr, "%2d", k);
            for (int e = 0; e < 8; ++e) fprintf(stderr, " %7.2f", h[k * 8 + e] ? (h[k * 8 + e] - t0) / 1965.0 : -1.0);
            fprintf(stderr, "\n");
        }
    }
    return NSM_OK;
}

struct Bufs {
    void *p1, *s1, *p2, *s2, *p3, *b3, *d2, *d1;
    __half* y;
    void* x5;        // 5-plane nets: the chunk-planar s2d input (nf, 3, H0, W0, 8)
    int* ctr;        // enc0's dynamic tile counters (2 ints)
    size_t bytes;
};

Bufs carve(void* ws, int nf, int H0, int W0, int es, bool x5 = false) {
    const int H1 = H0 / 2, W1 = W0 / 2, H2 = H1 / 2, W2 = W1 / 2, H3 = H2 / 2, W3 = W2 / 2;
    Bufs b{};
    char* p = (char*)ws;
    auto take = [&](size_t bytes) {
        char* r = p;
        p += (bytes + 255) / 256 * 256;
        return (void*)r;
    };
    b.p1 = take((size_t)nf * H1 * W1 * 16 * es);
    b.s1 = take((size_t)nf * H1 * W1 * 32 * es);
    b.p2 = take((size_t)nf * H2 * W2 * 32 * es);
    b.s2 = take((size_t)nf * H2 * W2 * 64 * es);
    b.p3 = take((size_t)nf * H3 * W3 * 64 * es);
    b.b3 = take((size_t)nf * H3 * W3 * 64 * es);
    b.d2 = take((size_t)nf * H2 * W2 * 32 * es);
    b.d1 = take((size_t)nf * (H1 + 2) * (W1 + 2) * 16 * es);   // replicate-padded, chunk-planar (DST_PADREP)
    b.y = (__half*)take((size_t)nf * H0 * W0 * 8);
    b.x5 = x5 ? take((size_t)nf * 3 * H0 * W0 * 8 * es) : nullptr;
    b.ctr = (int*)take(2 * sizeof(int));
    b.bytes = (size_t)(p - (char*)ws);
    return b;
}

template <typename T>
nsm_status run_levels(const Plan& p, const Bufs& b, int nf, int H0, int W0, cudaStream_t st) {
    const int H1 = H0 / 2, W1 = W0 / 2, H2 = H1 / 2, W2 = W1 / 2, H3 = H2 / 2, W3 = W2 / 2;
    const Level& L1 = p.lev[1];
    const Level& L2 = p.lev[2];
    const Level& L3 = p.lev[3];
    LevelArgs a{};
    // l1 encoder: P1 (16) -> S1 (32) + pool -> P2
    a = LevelArgs{b.p1, nullptr, H1, W1, L1.enc3.wpk, L1.enc3.b32, L1.enc1.wpk, L1.enc1.b32, b.s1, b.p2};
    nsm_status s = launch_level<T, 16, 32, 32, SRC_TENSOR, DST_STORE | DST_POOL, 4, 4, 2>(a, nf, st, "lv1_enc");
    if (s != NSM_OK) return s;
    // l2 encoder: P2 (32) -> S2 (64) + pool -> P3
    a = LevelArgs{b.p2, nullptr, H2, W2, L2.enc3.wpk, L2.enc3.b32, L2.enc1.wpk, L2.enc1.b32, b.s2, b.p3};
    s = launch_level<T, 32, 64, 64, SRC_TENSOR, DST_STORE | DST_POOL, 2, 2, 2>(a, nf, st, "lv2_enc");
    if (s != NSM_OK) return s;
    // l3 bottleneck: P3 (64) -> 128 -> B3 (64)
    a = LevelArgs{b.p3, nullptr, H3, W3, L3.enc3.wpk, L3.enc3.b32, L3.enc1.wpk, L3.enc1.b32, b.b3, nullptr};
    s = launch_level<T, 64, 128, 64, SRC_TENSOR, DST_STORE, 1, 2, 2>(a, nf, st, "lv3_bott");
    if (s != NSM_OK) return s;
    // l2 decoder: up(B3) + S2 -> 64 -> D2 (32)
    a = LevelArgs{b.b3, b.s2, H2, W2, L2.dec3.wpk, L2.dec3.b32, L2.dec1.wpk, L2.dec1.b32, b.d2, nullptr};
    s = launch_level<T, 64, 64, 32, SRC_UP, DST_STORE, 2, 2, 2>(a, nf, st, "lv2_dec");
    if (s != NSM_OK) return s;
    // l1 decoder: up(D2) + S1 -> 32 -> D1 (16)
    a = LevelArgs{b.d2, b.s1, H1, W1, L1.dec3.wpk, L1.dec3.b32, L1.dec1.wpk, L1.dec1.b32, b.d1, nullptr};
    s = launch_level<T, 32, 32, 16, SRC_UP, DST_STORE | DST_PADREP, 4, 2, 2>(a, nf, st, "lv1_dec");
    (void)W3;
    return s;
}

// Tensor maps over the planar fp32 G-buffer of frames [0, nf) of a chunk;
// false when TMA's 16-byte stride / address rules do not hold.
bool encode_gbuf_maps(const GBufK& g, int nf, int h, int w, GbufMaps* m) {
    auto enc = tensor_map_encoder();
    const int64_t fs = g.frame_stride;
    if (!enc || (w * 4) % 16 || (fs * 4) % 16 || ((uintptr_t)g.d | (uintptr_t)g.normal | (uintptr_t)g.position) % 16)
        return false;
    const cuuint32_t box3[3] = {(cuuint32_t)ST_TCOLS, (cuuint32_t)ST_ROWS, 1};
    const cuuint32_t box4[4] = {(cuuint32_t)ST_TCOLS, (cuuint32_t)ST_ROWS, 3, 1};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    const cuuint64_t dim3_[3] = {(cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)nf};
    const cuuint64_t str3[2] = {(cuuint64_t)w * 4, (cuuint64_t)fs * 4};
    const cuuint64_t dim4[4] = {(cuuint64_t)w, (cuuint64_t)h, 3, (cuuint64_t)nf};
    const cuuint64_t str4[3] = {(cuuint64_t)w * 4, (cuuint64_t)h * w * 4, (cuuint64_t)fs * 12};
    CUresult r = enc(&m->d, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(g.d), dim3_, str3, box3, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
    r = enc(&m->n, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(g.normal), dim4, str4, box4, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
    r = enc(&m->p, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(g.position), dim4, str4, box4, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <typename T>
nsm_status run_l0(const Plan& p, const Bufs& b, const Enc0Args& e0, const GbufMaps& tm, int nf, int H0,
                  int W0, int h, int w, void* y, int y_f16, cudaStream_t st, int src) {
    // src: 0 fp32 feature planes, 1 G-buffer (LDG), 2 G-buffer (TMA),
    // 3 the 5-plane s2d tensor b.x5 (enc0_s2d)
    static PerDevice attr;
    if (attr.first()) {
        cudaFuncSetAttribute(enc0_kernel<T, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * E0_SMEM);
        cudaFuncSetAttribute(enc0_kernel<T, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * E0_SMEM);
        cudaFuncSetAttribute(enc0_kernel<T, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, ENC0_SMEM_TMA);
        cudaFuncSetAttribute(enc0_kernel<T, 2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, ENC0_SMEM_TMA);
        cudaFuncSetAttribute(enc0_s2d_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, S24_SMEM);
    }
    // setmaxnreg.inc blocks until .dec released enough of the CTA's launch
    // allocation: refuse to launch a budget that could hang
    static const int launch_regs = [] {
        cudaFuncAttributes fa{}, fb{};
        cudaFuncGetAttributes(&fa, enc0_kernel<T, 2>);
        cudaFuncGetAttributes(&fb, enc0_kernel<T, 2, true>);
        return std::min(fa.numRegs, fb.numRegs);
    }();
    if (kE0Prod * kE0ProdRegs + (kE0Threads - kE0Prod) * kE0MmaRegs > launch_regs * kE0Threads)
        return fail(NSM_ERR_CUDA, "enc0: register budget %d x %d + %d x %d exceeds launch allocation %d x %d",
                    kE0Prod, kE0ProdRegs, kE0Threads - kE0Prod, kE0MmaRegs, kE0Threads, launch_regs);
    const int total = ((W0 + E0_TW - 1) / E0_TW) * ((H0 + E0_TH - 1) / E0_TH) * nf;
    const int pgrid = std::min(total, num_sms());
    {
        NSM_PROF(src == 3 ? "enc0_s2d" : "enc0_fused", st);
        if (src == 3) {
            CUtensorMap xm;
            memset(&xm, 0, sizeof xm);
            if (!encode_s2d24_map(b.x5, std::is_same<T, __nv_bfloat16>::value, H0, W0, nf, &xm))
                return fail(NSM_ERR_CUDA, "enc0_s2d: TMA tensor map encoding failed");
            launch_pdl(enc0_s2d_kernel<T>, dim3(pgrid), dim3(kS24Threads), S24_SMEM, st, e0, xm, total);
        } else if (src == 2 && e0.tidx)
            launch_pdl(enc0_kernel<T, 2, true>, dim3(pgrid), dim3(kE0Threads), ENC0_SMEM_TMA, st, e0, tm, total);
        else if (src == 2) launch_pdl(enc0_kernel<T, 2>, dim3(pgrid), dim3(kE0Threads), ENC0_SMEM_TMA, st, e0, tm, total);
        else if (src == 1) launch_pdl(enc0_kernel<T, 1>, dim3(pgrid), dim3(kL0Threads), 2 * E0_SMEM, st, e0, tm, total);
        else launch_pdl(enc0_kernel<T, 0>, dim3(pgrid), dim3(kL0Threads), 2 * E0_SMEM, st, e0, tm, total);
    }
    nsm_status s = run_levels<T>(p, b, nf, H0, W0, st);
    if (s != NSM_OK) return s;
    const Level& L0 = p.lev[0];
    if (!p.d0p3.present()) return fail(NSM_ERR_UNSUPPORTED, "dec0: polyphase level-0 decoder weights missing");
    {
        // polyphase level-0 decoder on the level-1 grid + the exact outer ring
        const int H1 = H0 / 2, W1 = W0 / 2;
        static PerDevice pattr;
        if (pattr.first()) cudaFuncSetAttribute(dec0p_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, D0P_SMEM);
        CUtensorMap dm;
        memset(&dm, 0, sizeof dm);
        if (!encode_cplanar_map(b.d1, std::is_same<T, __nv_bfloat16>::value, H1 + 2, W1 + 2, nf, D0P_IC, D0P_IR, &dm))
            return fail(NSM_ERR_CUDA, "dec0p: TMA tensor map encoding failed");
        Dec0pArgs dp{p.d0p3.wpk, p.d0p1.wpk, p.d0ph.wpk, L0.dec3.b32, L0.dec1.b32, p.head.b32, b.y, H1, W1, H0, W0, nullptr};
        static long long* d0_trace = nullptr;
#ifdef NSM_EXPERIMENTS
        if (getenv("NSM_DEC0_TRACE")) {
            if (!d0_trace) cudaMalloc(&d0_trace, 64 * 8 * sizeof(long long));
            cudaMemsetAsync(d0_trace, 0, 64 * 8 * sizeof(long long), st);
            dp.trace = d0_trace;
        }
#endif
        const int ptotal = ((W1 + 7) / 8) * ((H1 + 15) / 16) * nf;
        {
            NSM_PROF("dec0_fused", st);
            launch_pdl(dec0p_kernel<T>, dim3(std::min(ptotal, num_sms())), dim3(D0P_THREADS), D0P_SMEM, st, dp, dm, ptotal);
            if (dp.trace) {   // experiments only: CTA 0's dec0p timeline (us at 1.965 GHz), stalls the stream
                static long long hb[64 * 8];
                cudaMemcpyAsync(hb, dp.trace, sizeof hb, cudaMemcpyDeviceToHost, st);
                cudaStreamSynchronize(st);
                long long t0 = 0;
                for (long long v : hb) if (v && (!t0 || v < t0)) t0 = v;
                fprintf(stderr, "dec0p CTA0 (us): tile tma conv3_iss epi1_end dec1_iss epi2_end head_iss epi3_end epi1_start\n");
                for (int k = 0; k < 64; ++k) {
                    if (!hb[k * 8 + 1]) break;
                    fprintf(stderr, "%2d", k);
                    for (int ev = 0; ev < 8; ++ev) fprintf(stderr, " %7.2f", hb[k * 8 + ev] ? (hb[k * 8 + ev] - t0) / 1965.0 : -1.0);
                    fprintf(stderr, "\n");
                }
            }
        }
        static const bool ring = env_int("NSM_DEC0_RING", 1) != 0;   // 0: timing only (experiments)
        if (ring) {
            const int items = 2 * ((W0 + 29) / 30 + (H0 - 2 + 29) / 30) * nf;
            NSM_PROF("dec0_ring", st);
            launch_pdl(dec0_ring_kernel<T>, dim3(std::min((items + 3) / 4, 2 * num_sms())), dim3(128), 0, st, (const T*)b.d1,
                       H1, W1, H0, W0, (const uint2*)L0.dec3.wpk, (const uint2*)L0.dec1.wpk, (const uint2*)p.head.wpk,
                       L0.dec3.b32, L0.dec1.b32, p.head.b32, b.y, nf);
        }
    }
    {
        static_assert(8 % kReconPx == 0, "W0 = round16(w) / 2 is a multiple of 8: float4 rows");
        dim3 g2((W0 / kReconPx + 127) / 128, H0, nf);
        NSM_PROF("recon", st);
        launch_pdl(recon_kernel, g2, dim3(128), 0, st, (const __half*)b.y, H0, W0, h, w, nf, y, y_f16);
    }
    return NSM_OK;
}

int round16(int v) { return (v + 15) / 16 * 16; }

}  // namespace

bool f16_supported(const Plan& p) {
    const nsm_net_config& c = p.cfg;
    return c.layers == 5 && c.base_channels == 16 && (c.in_channels == 4 || c.in_channels == 5) &&
           c.use_space_to_depth && c.channel_cap >= 128;
}

size_t infer_f16_workspace(const Plan& p, int n, int h, int w) {
    const int Hp = round16(h), Wp = round16(w);
    const int nf = std::min(n, chunk_frames());
    return carve(nullptr, nf, Hp / 2, Wp / 2, 2, p.cfg.in_channels == 5).bytes + 1024;
}

nsm_status pack_f16(Plan& p, std::vector<char>& blob, size_t& offset_out) {
    const bool bf = p.act == NSM_BF16;
    if (!f16_supported(p)) {
        // generic layer-by-layer path (net_gen16.cu): every conv as mma.sync
        // B fragments in reference channel order.  Everything is packed
        // before `blob` grows: the fp32 sources (c->w32) point into it
        std::vector<std::pair<ConvW*, std::vector<uint32_t>>> items;
        auto pack = [&](ConvW* c) {
            std::vector<uint32_t> v;
            if (bf) pack_frag<__nv_bfloat16>(c->w32, c->cout, c->cin, c->k, false, v);
            else pack_frag<__half>(c->w32, c->cout, c->cin, c->k, false, v);
            items.emplace_back(c, std::move(v));
        };
        for (int j = 0; j < p.nlev; ++j)
            for (ConvW* c : {&p.lev[j].enc3, &p.lev[j].enc1, &p.lev[j].dec3, &p.lev[j].dec1})
                if (c->present()) pack(c);
        pack(&p.head);
        for (auto& it : items) {
            const size_t off = (blob.size() + 255) / 256 * 256;
            blob.resize(off + it.second.size() * 4);
            memcpy(blob.data() + off, it.second.data(), it.second.size() * 4);
            it.first->wpk = (const void*)(uintptr_t)off;
        }
        offset_out = blob.size();
        return NSM_OK;
    }
    // gather every packed tensor first (the fp32 sources live in `blob`)
    struct Item {
        ConvW* c;
        std::vector<char> bytes;
    };
    std::vector<Item> items;
    auto frag = [&](ConvW& c, bool perm, float scale = 1.f) {
        std::vector<uint32_t> v;
        if (bf) pack_frag<__nv_bfloat16>(c.w32, c.cout, c.cin, c.k, perm, v, scale);
        else pack_frag<__half>(c.w32, c.cout, c.cin, c.k, perm, v, scale);
        Item it{&c, std::vector<char>((char*)v.data(), (char*)v.data() + v.size() * 4)};
        items.push_back(std::move(it));
    };
    auto umma = [&](ConvW& c) {
        std::vector<uint16_t> v;
        if (bf) pack_umma<__nv_bfloat16>(c.w32, c.cout, c.cin, c.k, v);
        else pack_umma<__half>(c.w32, c.cout, c.cin, c.k, v);
        Item it{&c, std::vector<char>((char*)v.data(), (char*)v.data() + v.size() * 2)};
        items.push_back(std::move(it));
    };
    frag(p.lev[0].enc3, true);
    // l0.enc1 feeds only enc0's 2x2 average pool: relu(0.25 x) = 0.25 relu(x),
    // so the 1/4 is folded into the weights (exact: a power of two) and the
    // bias (enc0 loads it scaled) and the pool is a plain sum
    frag(p.lev[0].enc1, false, 0.25f);
    frag(p.lev[0].dec3, false);
    frag(p.lev[0].dec1, false);
    frag(p.head, false);
    for (int j = 1; j < p.nlev; ++j) {
        umma(p.lev[j].enc3);
        umma(p.lev[j].enc1);
        if (p.lev[j].dec3.present()) {
            umma(p.lev[j].dec3);
            umma(p.lev[j].dec1);
        }
    }
    // Polyphase level-0 decoder (dec0p_kernel).  up2 with an edge clamp is
    // up2 of the replicate-padded low-res tensor, so every output phase
    // (a, b) of conv3(up2(x)) is a 3x3 convolution of x whose taps combine
    // the reference's taps with the (1/4, 3/4) bilinear weights; only the
    // outermost level-0 ring (where the conv's zero padding differs from
    // the replicate padding) is recomputed by dec0_ring_kernel.
    std::vector<float> w3p, w1d, whd;
    const ConvW& d3 = p.lev[0].dec3;
    const ConvW& d1 = p.lev[0].dec1;
    if (d3.present() && d3.k == 3 && d3.cin == 16 && d3.cout == 16 && d1.cin == 16 && d1.cout == 16 &&
        p.head.cin == 16 && p.head.cout == 4) {
        auto coef = [](int a, int d, float (&c)[3]) {     // x(i + l - 1) weights in U(2i + a + d - 1)
            c[0] = c[1] = c[2] = 0.f;
            const int r = a + d - 1, m = (r >= 0 ? r / 2 : -1), ph = r - 2 * m;
            if (ph == 0) {
                c[m] += 0.25f;
                c[m + 1] += 0.75f;
            } else {
                c[m + 1] += 0.75f;
                c[m + 2] += 0.25f;
            }
        };
        w3p.assign(64 * 16 * 9, 0.f);
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b)
                for (int dy = 0; dy < 3; ++dy)
                    for (int dx = 0; dx < 3; ++dx) {
                        float cy[3], cx[3];
                        coef(a, dy, cy);
                        coef(b, dx, cx);
                        for (int co = 0; co < 16; ++co)
                            for (int ci = 0; ci < 16; ++ci) {
                                const float w = d3.w32[((size_t)co * 16 + ci) * 9 + dy * 3 + dx];
                                for (int ly = 0; ly < 3; ++ly)
                                    for (int lx = 0; lx < 3; ++lx)
                                        w3p[((size_t)((a * 2 + b) * 16 + co) * 16 + ci) * 9 + ly * 3 + lx] +=
                                            w * cy[ly] * cx[lx];
                            }
                    }
        w1d.assign(64 * 64, 0.f);
        whd.assign(16 * 64, 0.f);
        for (int ph = 0; ph < 4; ++ph) {
            for (int co = 0; co < 16; ++co)
                for (int ci = 0; ci < 16; ++ci) w1d[(size_t)(ph * 16 + co) * 64 + ph * 16 + ci] = d1.w32[co * 16 + ci];
            for (int hc = 0; hc < 4; ++hc)
                for (int ci = 0; ci < 16; ++ci) whd[(size_t)(ph * 4 + hc) * 64 + ph * 16 + ci] = p.head.w32[hc * 16 + ci];
        }
        auto setc = [](ConvW& c, const std::vector<float>& w, int cout, int cin, int k) {
            c.cin = cin;
            c.cout = cout;
            c.k = k;
            c.w32 = w.data();
        };
        setc(p.d0p3, w3p, 64, 16, 3);
        setc(p.d0p1, w1d, 64, 64, 1);
        setc(p.d0ph, whd, 16, 64, 1);
        umma(p.d0p3);
        umma(p.d0p1);
        umma(p.d0ph);
    }
    for (auto& it : items) {
        const size_t off = (blob.size() + 255) / 256 * 256;
        blob.resize(off + it.bytes.size());
        memcpy(blob.data() + off, it.bytes.data(), it.bytes.size());
        it.c->wpk = (const void*)(uintptr_t)off;   // rebased to the device block later
    }
    p.d0p3.w32 = p.d0p1.w32 = p.d0ph.w32 = nullptr;   // host-only sources (packed above)
    offset_out = blob.size();
    return NSM_OK;
}

nsm_status infer_f16(const Plan& p, const nsm_gbuffer* g, const float* sm, int64_t sm_stride,
                     const nsm_frame* frames, int n, int h, int w, void* y, nsm_dtype y_dtype,
                     int64_t* first_bad, int32_t* texel_idx, void* ws, size_t ws_bytes, cudaStream_t st) {
    if (g->dtype != NSM_F32) return fail(NSM_ERR_UNSUPPORTED, "16-bit path reads fp32 G-buffer planes");
    if (g->z_f || g->c_e || g->c_c || g->coverage)
        return fail(NSM_ERR_UNSUPPORTED, "16-bit path derives z_f/c_e/c_c from the planes");
    const int Hp = round16(h), Wp = round16(w), H0 = Hp / 2, W0 = Wp / 2;
    const int nfmax = std::min(n, chunk_frames());
    if (sm_stride * nfmax > INT32_MAX)   // the fused feature pass indexes a chunk's maps in 32 bits
        return fail(NSM_ERR_UNSUPPORTED, "shadow maps of %lld texels x %d frames per pass exceed 2^31",
                    (long long)sm_stride, nfmax);
    const bool five = p.cfg.in_channels == 5;
    Bufs b = carve(ws, nfmax, H0, W0, 2, five);
    if (ws_bytes < b.bytes) return fail(NSM_ERR_ARG, "workspace too small (%zu < %zu)", ws_bytes, b.bytes);
    {
        NSM_PROF("fill_i64", st);
        launch_pdl(fill_first_bad, dim3((n + 127) / 128), dim3(128), 0, st, first_bad, n, b.ctr);
    }
    for (int f0 = 0; f0 < n; f0 += chunk_frames()) {
        const int nf = std::min(chunk_frames(), n - f0);
        Enc0Args e{};
        e.g = GBufK{(const float*)g->d + (int64_t)f0 * g->frame_stride,
                    (const float*)g->normal + (int64_t)f0 * 3 * g->frame_stride,
                    (const float*)g->position + (int64_t)f0 * 3 * g->frame_stride,
                    nullptr, nullptr, nullptr, nullptr, g->frame_stride};
        e.sm = sm + f0 * sm_stride;
        e.sm_stride = sm_stride;
        make_frame_table(frames + f0, nf, e.tab);
        e.h = h;
        e.w = w;
        e.H0 = H0;
        e.W0 = W0;
        e.td = tile_div(H0, W0);
        e.wb3 = (const uint2*)p.lev[0].enc3.wpk;
        e.wb1 = (const uint2*)p.lev[0].enc1.wpk;
        e.b3 = p.lev[0].enc3.b32;
        e.b1 = p.lev[0].enc1.b32;
        e.out = b.p1;
        e.tile_ctr = b.ctr;
        e.first_bad = first_bad + f0;
        e.tidx = texel_idx ? texel_idx + (int64_t)f0 * 2 * h * w : nullptr;
        e.dbg = env_int("NSM_ENC0_DBG", 0);
        e.trace = nullptr;
#ifdef NSM_EXPERIMENTS
        static long long* e0_trace = nullptr;
        if (getenv("NSM_ENC0_TRACE")) {
            if (!e0_trace) cudaMalloc(&e0_trace, 2048 * sizeof(long long));
            cudaMemsetAsync(e0_trace, 0, 2048 * sizeof(long long), st);
            e.trace = e0_trace;
        }
#endif
        void* yo = (char*)y + (size_t)f0 * h * w * (y_dtype == NSM_F16 ? 2 : 4);
        GbufMaps tm;
        memset(&tm, 0, sizeof tm);
        int src;
        if (five) {
            // 5-plane net: features + blocker search -> b.x5, then enc0_s2d
            nsm_gbuffer gc = *g;
            gc.d = e.g.d;
            gc.normal = e.g.normal;
            gc.position = e.g.position;
            nsm_status s5 = launch_feat5(&gc, e.sm, sm_stride, frames + f0, nf, h, w, H0, W0, b.x5,
                                         p.act == NSM_BF16 ? 1 : 0, first_bad + f0, e.tidx, st);
            if (s5 != NSM_OK) return s5;
            src = 3;
        } else {
            src = encode_gbuf_maps(e.g, nf, h, w, &tm) ? 2 : 1;
        }
        nsm_status s = p.act == NSM_BF16
                           ? run_l0<__nv_bfloat16>(p, b, e, tm, nf, H0, W0, h, w, yo, y_dtype == NSM_F16, st, src)
                           : run_l0<__half>(p, b, e, tm, nf, H0, W0, h, w, yo, y_dtype == NSM_F16, st, src);
        if (s != NSM_OK) return s;
#ifdef NSM_EXPERIMENTS
        if (e.trace) {   // experiments only: per-CTA spans of enc0 (globaltimer), stalls the stream
            static long long hb[2048];
            cudaMemcpyAsync(hb, e.trace, sizeof hb, cudaMemcpyDeviceToHost, st);
            cudaStreamSynchronize(st);
            long long s0 = 0, e1 = 0;
            int nc = 0;
            double dsum = 0, dmax = 0, dmin = 1e30;
            for (int c = 0; c < 512; ++c) {
                const long long a0 = hb[2 * c], a1 = hb[2 * c + 1];
                if (!a0 || !a1) continue;
                ++nc;
                if (!s0 || a0 < s0) s0 = a0;
                if (a1 > e1) e1 = a1;
                const double d = (a1 - a0) / 1e3;
                dsum += d, dmax = std::max(dmax, d), dmin = std::min(dmin, d);
            }
            fprintf(stderr, "enc0 CTAs %d: first start -> last end %.2f us; CTA span min/avg/max %.2f/%.2f/%.2f us\n", nc,
                    (e1 - s0) / 1e3, dmin, dsum / std::max(nc, 1), dmax);
            if (getenv("NSM_ENC0_TRACE_ALL")) {
                fprintf(stderr, "enc0 per-CTA span (us):");
                for (int c = 0; c < nc; ++c) fprintf(stderr, " %.1f/%lld", (hb[2 * c + 1] - hb[2 * c]) / 1e3, hb[1024 + c]);
                fprintf(stderr, "\n");
            }
        }
#endif
    }
    NSM_CUDA_TRY(cudaGetLastError());
    return NSM_OK;
}

nsm_status forward_f16(const Plan& p, const float* x, int n, int h, int w, float* out, void* ws,
                       size_t ws_bytes, cudaStream_t st) {
    if (!f16_supported(p)) return fail(NSM_ERR_UNSUPPORTED, "no 16-bit kernels for this NetworkConfig");
    const int H0 = h / 2, W0 = w / 2;
    const int nfmax = std::min(n, chunk_frames());
    const bool five = p.cfg.in_channels == 5;
    Bufs b = carve(ws, nfmax, H0, W0, 2, five);
    if (ws_bytes < b.bytes) return fail(NSM_ERR_ARG, "workspace too small");
    for (int f0 = 0; f0 < n; f0 += chunk_frames()) {
        const int nf = std::min(chunk_frames(), n - f0);
        Enc0Args e{};
        e.x = x + (int64_t)f0 * p.cfg.in_channels * h * w;
        e.h = h;
        e.w = w;
        e.H0 = H0;
        e.W0 = W0;
        e.td = tile_div(H0, W0);
        e.wb3 = (const uint2*)p.lev[0].enc3.wpk;
        e.wb1 = (const uint2*)p.lev[0].enc1.wpk;
        e.b3 = p.lev[0].enc3.b32;
        e.b1 = p.lev[0].enc1.b32;
        e.out = b.p1;
        e.first_bad = nullptr;
        float* yo = out + (size_t)f0 * h * w;
        GbufMaps tm;
        memset(&tm, 0, sizeof tm);
        if (five) {
            const int64_t items = (int64_t)nf * H0 * W0;
            const int grid = (int)((items + 255) / 256);
            NSM_PROF("pack_s2d24", st);
            if (p.act == NSM_BF16)
                pack_s2d24_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(e.x, h, w, nf, (__nv_bfloat16*)b.x5);
            else
                pack_s2d24_kernel<__half><<<grid, 256, 0, st>>>(e.x, h, w, nf, (__half*)b.x5);
        }
        const int src = five ? 3 : 0;
        nsm_status s = p.act == NSM_BF16
                           ? run_l0<__nv_bfloat16>(p, b, e, tm, nf, H0, W0, h, w, yo, 0, st, src)
                           : run_l0<__half>(p, b, e, tm, nf, H0, W0, h, w, yo, 0, st, src);
        if (s != NSM_OK) return s;
    }
    NSM_CUDA_TRY(cudaGetLastError());
    return NSM_OK;
}

}  // namespace nsm
