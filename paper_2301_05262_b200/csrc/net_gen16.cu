// Generic 16-bit tensor-core path: network.forward (network.py:165-209) for
// every NetworkConfig the reference accepts (layers 2-8, any base / input
// channel count, plain or space-to-depth input, any channel cap) on plans
// that the level-fused kernels of net_f16.cu do not cover (those are built
// for the default layers=5 / base 16 / s2d net with 4 or 5 input planes).
//
// Layer by layer, NHWC 16-bit activations with the channel count padded to a
// multiple of 16 (the padding channels are zero): every conv is an implicit
// GEMM on mma.sync m16n8k16 with fp32 accumulation -- a CTA stages the K
// input rows of a 64-pixel output segment (all channels) in shared memory
// and its 4 warps compute 16 pixels x 64 output channels each, 9 (or 1) taps
// x Cin/16 K-steps of ldmatrix A fragments against B fragments packed by the
// plan ([tap][k16][n8][lane], pack_frag).  Bias and ReLU run in the epilogue;
// pooling, bilinear upsampling + skip, the head reconstruction and the
// sigmoid are small fp32-math kernels between the convs.
#include <algorithm>
#include <atomic>
#include <type_traits>

#include "common.cuh"
#include "net.cuh"
#include "prof.cuh"
#include "tc.cuh"

namespace nsm {

namespace {

constexpr int G_PX = 64, G_CO = 64, G_THREADS = 128;

__host__ __device__ inline int pad16(int c) { return (c + 15) / 16 * 16; }

// fp32 planes (n, cin, h, w) -> NHWC 16-bit (n, hl, wl, cp), space_to_depth
// (autodiff.py:290-308: channel 4c + 2dy + dx) when s2d; padding channels 0.
template <typename T>
__global__ void g16_pack_input(const float* __restrict__ x, int n, int cin, int h, int w, int s2d, int cp,
                               T* __restrict__ y) {
    const int hl = s2d ? h / 2 : h, wl = s2d ? w / 2 : w;
    const int64_t total = (int64_t)n * hl * wl * cp;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i % cp);
        const int64_t pix = i / cp;
        const int X = (int)(pix % wl), Y = (int)((pix / wl) % hl), f = (int)(pix / ((int64_t)wl * hl));
        float v = 0.f;
        if (s2d) {
            if (c < 4 * cin) {
                const int cc = c >> 2, dy = (c >> 1) & 1, dx = c & 1;
                v = x[(((int64_t)f * cin + cc) * h + 2 * Y + dy) * w + 2 * X + dx];
            }
        } else if (c < cin) {
            v = x[(((int64_t)f * cin + c) * h + Y) * w + X];
        }
        y[i] = (T)v;
    }
}

template <typename T>
__device__ __forceinline__ float to_f(T v) {
    if constexpr (std::is_same<T, __half>::value) return __half2float(v);
    else return __bfloat162float(v);
}

// Implicit-GEMM conv k in {1, 3}, zero padding, + bias, optional ReLU.
// x: (n, h, w, cinp) 16-bit; y: (n, h, w, coutp) 16-bit, or fp32 when F32OUT.
template <typename T, int K, bool F32OUT>
__global__ void __launch_bounds__(G_THREADS) g16_conv(const T* __restrict__ x, int h, int w, int cinp,
                                                     const uint2* __restrict__ wb, const float* __restrict__ bias,
                                                     int cout, int coutp, int relu, void* __restrict__ yv) {
    extern __shared__ __align__(16) uint8_t gsm[];
    constexpr int P = (K - 1) / 2, IC = G_PX + K - 1;
    const int pxb = cinp * 2 + 16;                        // padded pixel stride (bank spread)
    const int nchunk = (coutp + G_CO - 1) / G_CO;
    const int f = blockIdx.z / nchunk, co0 = (blockIdx.z % nchunk) * G_CO;
    const int y0 = blockIdx.y, x0 = blockIdx.x * G_PX;
    const int c8 = cinp / 8;
    // stage rows y0-P .. y0+P, columns x0-P .. x0+63+P, all channels
    for (int i = threadIdx.x; i < K * IC * c8; i += G_THREADS) {
        const int c = i % c8, q = (i / c8) % IC, r = i / (c8 * IC);
        const int gy = y0 + r - P, gx = x0 + q - P;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (gy >= 0 && gy < h && gx >= 0 && gx < w)
            v = __ldg(reinterpret_cast<const uint4*>(x + (((int64_t)f * h + gy) * w + gx) * cinp) + c);
        *reinterpret_cast<uint4*>(gsm + (r * IC + q) * pxb + c * 16) = v;
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3, lm = lane >> 3, li = lane & 7;
    const int KK = cinp / 16, NT = (cout + 7) / 8;
    float acc[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[j][e] = 0.f;
    const uint32_t sbase = smem_u32(gsm);
    for (int tap = 0; tap < K * K; ++tap) {
        const int ky = tap / K, kx = tap % K;
        const uint32_t rowa = sbase + (ky * IC + warp * 16 + (lm & 1) * 8 + li + kx) * pxb + (lm >> 1) * 16;
        for (int kk = 0; kk < KK; ++kk) {
            uint32_t a[4];
            ldsm_x4(rowa + kk * 32, a);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int nt = co0 / 8 + j;
                if (nt < NT) {
                    const uint2 b = __ldg(wb + (((int64_t)tap * KK + kk) * NT + nt) * 32 + lane);
                    mma16816<T>(acc[j], a, b.x, b.y);
                }
            }
        }
    }
    // epilogue: rows g, g + 8 of the warp's 16 pixels; channels 2t, 2t + 1
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int co = co0 + j * 8 + 2 * t;
        if (co >= coutp) continue;
        const float b0 = co < cout ? __ldg(bias + co) : 0.f, b1 = co + 1 < cout ? __ldg(bias + co + 1) : 0.f;
#pragma unroll
        for (int hr = 0; hr < 2; ++hr) {
            const int px = x0 + warp * 16 + g + hr * 8;
            if (px >= w) continue;
            float v0 = acc[j][2 * hr] + b0, v1 = acc[j][2 * hr + 1] + b1;
            if (relu) {
                v0 = fmaxf(v0, 0.f);
                v1 = fmaxf(v1, 0.f);
            }
            if (co >= cout) v0 = 0.f;
            if (co + 1 >= cout) v1 = 0.f;
            const int64_t o = (((int64_t)f * h + y0) * w + px) * coutp + co;
            if constexpr (F32OUT)
                *reinterpret_cast<float2*>(reinterpret_cast<float*>(yv) + o) = make_float2(v0, v1);
            else
                *reinterpret_cast<uint32_t*>(reinterpret_cast<T*>(yv) + o) = Elem<T>::pack(v0, v1);
        }
    }
}

// avg_pool2 (autodiff.py:241-247) on NHWC.
template <typename T>
__global__ void g16_pool(const T* __restrict__ x, int n, int h, int w, int cp, T* __restrict__ y) {
    const int ho = h / 2, wo = w / 2;
    const int64_t total = (int64_t)n * ho * wo * cp;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i % cp);
        const int64_t pix = i / cp;
        const int X = (int)(pix % wo), Y = (int)((pix / wo) % ho), f = (int)(pix / ((int64_t)wo * ho));
        const T* s = x + (((int64_t)f * h + 2 * Y) * w + 2 * X) * cp + c;
        const float v = ((to_f(s[0]) + to_f(s[cp])) + (to_f(s[(int64_t)w * cp]) + to_f(s[(int64_t)w * cp + cp]))) * 0.25f;
        y[i] = (T)v;
    }
}

// _upsample_taps (autodiff.py:258-264)
__device__ __forceinline__ void g_tap(int i, int n, int& i0, int& i1, float& wt) {
    float s = fminf(fmaxf((i + 0.5f) * 0.5f - 0.5f, 0.f), (float)(n - 1));
    i0 = (int)s;
    i1 = min(i0 + 1, n - 1);
    wt = s - i0;
}

// bilinear_upsample2 (autodiff.py:267-274, rows then columns) + optional
// skip (network.py:191-192), NHWC.
template <typename T>
__global__ void g16_up2_add(const T* __restrict__ x, int n, int h, int w, int cp, const T* __restrict__ skip,
                            T* __restrict__ y) {
    const int ho = 2 * h, wo = 2 * w;
    const int64_t total = (int64_t)n * ho * wo * cp;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i % cp);
        const int64_t pix = i / cp;
        const int X = (int)(pix % wo), Y = (int)((pix / wo) % ho), f = (int)(pix / ((int64_t)wo * ho));
        int r0, r1, c0, c1;
        float rw, cw;
        g_tap(Y, h, r0, r1, rw);
        g_tap(X, w, c0, c1, cw);
        const T* b = x + (int64_t)f * h * w * cp + c;
        auto at = [&](int r, int q) { return to_f(b[((int64_t)r * w + q) * cp]); };
        const float a0 = at(r0, c0) * (1.f - rw) + at(r1, c0) * rw;
        const float a1 = at(r0, c1) * (1.f - rw) + at(r1, c1) * rw;
        float v = a0 * (1.f - cw) + a1 * cw;
        if (skip) v += to_f(skip[i]);
        y[i] = (T)v;
    }
}

__device__ __forceinline__ float g_sigmoid(float v) {
    const float e = expf(-fabsf(v));
    return v >= 0.f ? 1.f / (1.f + e) : e / (1.f + e);
}

// Head reconstruction (network.py:199-209) from the fp32 NHWC head output
// (n, hl, wl, hp): s2d: sigmoid(up2(y0) + d2s(y with channel 0 zeroed)),
// plain: sigmoid(y0); out (n, 1, h, w) fp32.
__global__ void g16_recon(const float* __restrict__ yh, int n, int hl, int wl, int hp, int s2d,
                          float* __restrict__ out) {
    const int h = s2d ? 2 * hl : hl, w = s2d ? 2 * wl : wl;
    const int64_t total = (int64_t)n * h * w;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int X = (int)(i % w), Y = (int)((i / w) % h), f = (int)(i / ((int64_t)w * h));
        const float* b = yh + (int64_t)f * hl * wl * hp;
        float v;
        if (s2d) {
            int r0, r1, c0, c1;
            float rw, cw;
            g_tap(Y, hl, r0, r1, rw);
            g_tap(X, wl, c0, c1, cw);
            auto at = [&](int r, int q) { return b[((int64_t)r * wl + q) * hp]; };
            const float a0 = at(r0, c0) * (1.f - rw) + at(r1, c0) * rw;
            const float a1 = at(r0, c1) * (1.f - rw) + at(r1, c1) * rw;
            v = a0 * (1.f - cw) + a1 * cw;
            const int k = 2 * (Y & 1) + (X & 1);
            if (k) v += b[((int64_t)(Y >> 1) * wl + (X >> 1)) * hp + k];
        } else {
            v = b[((int64_t)Y * wl + X) * hp];
        }
        out[i] = g_sigmoid(v);
    }
}

int g_grid(int64_t total) { return (int)std::min<int64_t>((total + 255) / 256, 148 * 32); }

template <typename T>
nsm_status g16_conv_launch(const T* x, int n, int h, int w, int cinp, const ConvW& c, int relu, void* y,
                           bool f32out, cudaStream_t st) {
    const int coutp = pad16(c.cout);
    const int K = c.k;
    const int smem = K * (G_PX + K - 1) * (cinp * 2 + 16);
    if (smem > 227 * 1024) return fail(NSM_ERR_UNSUPPORTED, "generic conv: %d input channels exceed shared memory", cinp);
    dim3 grid((w + G_PX - 1) / G_PX, h, n * ((coutp + G_CO - 1) / G_CO));
    const uint2* wb = (const uint2*)c.wpk;
    // the opt-in shared-memory size is per-device state: set it once per
    // (device, instantiation) for the largest tile this process has used
    auto opt_in = [&](const void* k) {
        static std::atomic<int> set_bytes[64][3];
        int dev = 0;
        cudaGetDevice(&dev);
        const int slot = (K == 3 ? 0 : f32out ? 2 : 1);
        std::atomic<int>& cur = set_bytes[dev & 63][slot];
        if (smem > cur.load()) {
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
            cur.store(227 * 1024);
        }
    };
    NSM_PROF("g16_conv", st);
    if (K == 3 && !f32out) {
        opt_in((const void*)g16_conv<T, 3, false>);
        g16_conv<T, 3, false><<<grid, G_THREADS, smem, st>>>(x, h, w, cinp, wb, c.b32, c.cout, coutp, relu, y);
    } else if (K == 1 && !f32out) {
        opt_in((const void*)g16_conv<T, 1, false>);
        g16_conv<T, 1, false><<<grid, G_THREADS, smem, st>>>(x, h, w, cinp, wb, c.b32, c.cout, coutp, relu, y);
    } else if (K == 1) {
        opt_in((const void*)g16_conv<T, 1, true>);
        g16_conv<T, 1, true><<<grid, G_THREADS, smem, st>>>(x, h, w, cinp, wb, c.b32, c.cout, coutp, relu, y);
    } else {
        return fail(NSM_ERR_UNSUPPORTED, "generic conv: k=%d head", K);
    }
    return NSM_OK;
}

struct GenBufs {
    void *a, *b, *head;
    void* skip[kMaxLevels];
    size_t bytes;
};

GenBufs gen_carve(const Plan& p, void* ws, int n, int h, int w) {
    const int s = p.cfg.use_space_to_depth ? 1 : 0;
    const int64_t hw0 = (int64_t)(h >> s) * (w >> s);
    int cmax = pad16(p.first_in);
    for (int j = 0; j < p.nlev; ++j) cmax = std::max(cmax, pad16(p.chans[j]));
    char* q = (char*)ws;
    auto take = [&](size_t bytes) {
        char* r = q;
        q += (bytes + 255) / 256 * 256;
        return (void*)r;
    };
    GenBufs g{};
    g.a = take((size_t)n * cmax * hw0 * 2);
    g.b = take((size_t)n * cmax * hw0 * 2);
    for (int j = 0; j < p.nlev - 1; ++j) g.skip[j] = take((size_t)n * pad16(p.chans[j]) * (hw0 >> (2 * j)) * 2);
    g.head = take((size_t)n * pad16(p.out_ch) * hw0 * 4);
    g.bytes = (size_t)(q - (char*)ws);
    return g;
}

template <typename T>
nsm_status forward_gen16_t(const Plan& p, const float* x, int n, int h, int w, float* out, void* ws,
                           size_t ws_bytes, cudaStream_t st) {
    GenBufs g = gen_carve(p, ws, n, h, w);
    if (ws_bytes < g.bytes) return fail(NSM_ERR_ARG, "workspace too small (%zu < %zu bytes)", ws_bytes, g.bytes);
    const int s = p.cfg.use_space_to_depth ? 1 : 0;
    int hl = h >> s, wl = w >> s;
    T* A = (T*)g.a;
    T* B = (T*)g.b;
    int cp = pad16(p.first_in);
    {
        NSM_PROF("g16_pack_input", st);
        g16_pack_input<T><<<g_grid((int64_t)n * hl * wl * cp), 256, 0, st>>>(x, n, p.cfg.in_channels, h, w, s, cp, A);
    }
    T* in = A;
    T* tmp = B;
    nsm_status e;
    for (int j = 0; j < p.nlev - 1; ++j) {
        const Level& L = p.lev[j];
        if ((e = g16_conv_launch<T>(in, n, hl, wl, cp, L.enc3, 1, tmp, false, st))) return e;
        T* sk = (T*)g.skip[j];
        if ((e = g16_conv_launch<T>(tmp, n, hl, wl, pad16(L.enc3.cout), L.enc1, 1, sk, false, st))) return e;
        cp = pad16(L.enc1.cout);
        {
            NSM_PROF("g16_pool", st);
            g16_pool<T><<<g_grid((int64_t)n * hl * wl * cp / 4), 256, 0, st>>>(sk, n, hl, wl, cp, in);
        }
        hl /= 2;
        wl /= 2;
    }
    {
        const Level& L = p.lev[p.nlev - 1];
        if ((e = g16_conv_launch<T>(in, n, hl, wl, cp, L.enc3, 1, tmp, false, st))) return e;
        if ((e = g16_conv_launch<T>(tmp, n, hl, wl, pad16(L.enc3.cout), L.enc1, 1, in, false, st))) return e;
        cp = pad16(L.enc1.cout);
    }
    for (int j = p.nlev - 2; j >= 0; --j) {
        const Level& L = p.lev[j];
        {
            NSM_PROF("g16_up2_add", st);
            g16_up2_add<T><<<g_grid((int64_t)n * hl * wl * 4 * cp), 256, 0, st>>>(
                in, n, hl, wl, cp, j > 0 ? (const T*)g.skip[j] : nullptr, tmp);
        }
        hl *= 2;
        wl *= 2;
        if ((e = g16_conv_launch<T>(tmp, n, hl, wl, cp, L.dec3, 1, in, false, st))) return e;
        if ((e = g16_conv_launch<T>(in, n, hl, wl, pad16(L.dec3.cout), L.dec1, 1, tmp, false, st))) return e;
        cp = pad16(L.dec1.cout);
        std::swap(in, tmp);
    }
    if ((e = g16_conv_launch<T>(in, n, hl, wl, cp, p.head, 0, g.head, true, st))) return e;
    {
        NSM_PROF("g16_recon", st);
        g16_recon<<<g_grid((int64_t)n * h * w), 256, 0, st>>>((const float*)g.head, n, hl, wl, pad16(p.out_ch), s, out);
    }
    NSM_CUDA_TRY(cudaGetLastError());
    return NSM_OK;
}

}  // namespace

size_t forward_gen16_workspace(const Plan& p, int n, int h, int w) { return gen_carve(p, nullptr, n, h, w).bytes + 1024; }

nsm_status forward_gen16(const Plan& p, const float* x, int n, int h, int w, float* out, void* ws, size_t ws_bytes,
                         cudaStream_t st) {
    return p.act == NSM_BF16 ? forward_gen16_t<__nv_bfloat16>(p, x, n, h, w, out, ws, ws_bytes, st)
                             : forward_gen16_t<__half>(p, x, n, h, w, out, ws, ws_bytes, st);
}

}  // namespace nsm
