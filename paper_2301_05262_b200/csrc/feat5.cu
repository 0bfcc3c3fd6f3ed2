// Stage 1 of the 5-plane network (BASELINE configs 3/4, "soft shadows" with
// the 16x16 blocker search): the 4 reference feature planes
// (raster.assemble_features, raster.py:266-278) plus the blocker-search
// penumbra plane (nsm.h nsm_blocker_plane; analysis.py:240-269, 319-320), in
// one pass over the G-buffer.
//
// Layout: one CTA per 16 x 16 level-0 tile (32 x 32 frame pixels: square,
// so the staged map region has the least halo; 8 x 32 measured 1.5 %
// slower), one thread per level-0 pixel (its 2 x 2 frame pixels).  The texel windows of the
// tile's covered pixels are bounded by their texel bounding box; that map
// region is staged in shared memory (rows of the map, coalesced), and the
// sliding 4 x 4 min / max of every staged position is built from it, so a
// pixel's 16 x 16 window is 16 sub-blocks:
//   zmin = min of the 16 block minima (the window minimum: a blocker exists
//          iff it is below the threshold, and then it is the blocker minimum)
//   block max < thr        -> every texel is a blocker: zmax candidate = max
//   block min >= thr       -> no blocker in the block
//   otherwise (straddling) -> its 16 texels are scanned
// Depths are positive floats (or +inf), so they are compared as int32; the
// threshold test and the blocker maximum fold into one DPX instruction per
// texel: min_u32((thr - 1) - t) over the block is (thr - 1) - (max blocker).
// The shadow map is read from HBM about once per tile; the window traffic is
// shared-memory traffic (the roofline that bounds this kernel).
//
// Outputs: the hot path's level-0 input tensor, 16-bit, chunk-planar
// (N, 3, H0, W0, 8): chunks 0-1 the space_to_depth of the 4 planes in the
// permuted order l0.enc3's packing expects (k' = (2dy + dx) * 4 + c), chunk 2
// the 4 blocker values of the pixel's 2 x 2 (s2d channels 16-19) and zeros;
// or (parity / drop-in mode) fp32 planes (N, 5, h, w).
#include <algorithm>
#include <atomic>
#include <cfloat>

#include "common.cuh"
#include "net.cuh"
#include "prof.cuh"
#include "tc.cuh"

namespace nsm {

namespace {

constexpr int F5_TY = 16, F5_TX = 16, F5_THREADS = F5_TY * F5_TX;
constexpr int F5_R = 8;                      // window rows ri-8 .. ri+7 (16 x 16)
constexpr int F5_MAX_TEX = 4096;             // staged texels per CTA (both regions)
constexpr int F5_SMEM = 3 * F5_MAX_TEX * 4;   // texels + sliding 4x4 blocks (int2): 48 KB; 3 CTAs per SM (registers)
// leave L1 to the global-memory window scans (8 x 32 tiles: 6144 texels per
// CTA 481 us, 3584: 458, 3072: 463, 2048: 482; 16 x 16 tiles: 3072-5120 all
// within 440-446 us)
constexpr int kInfBits = 0x7f800000;

struct Feat5Args {
    GBufK g;
    const float* sm;
    int64_t sm_stride;
    FrameTable tab;
    int h, w;          // frame pixels present
    int H0, W0;        // level-0 grid (padded frame / 2)
    void* out;         // 16-bit (N, 3, H0, W0, 8) or fp32 (N, 5, h, w)
    int64_t* first_bad;
    int32_t* tidx;     // parity hook (nullable): (N, 2, h, w)
    int32_t* dbg;      // debugging (nullable): (N, h, w, 4) zmin, zmax, thr, path bits
};

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// analysis.penumbra_extents (analysis.py:240-269) -> screen width
// (x_a + x_b) * focal_px / d (analysis.py:319-320) in units of the focal
// length, (x_a + x_b) / d, fp32 (the plane is rounded to 16 bits right
// after); 0 where the model's preconditions fail.
// The reference's angles are theta = atan(T), T = (bq + r_e) / z_f, and
// theta_d = asin(s), s = r_s / hyp, so tan(theta -/+ theta_d) follow from
// the tangent addition formula with tan(theta_d) = s / sqrt(1 - s^2) -- no
// transcendental calls -- and theta + theta_d < pi / 2 is 1 - T tan(theta_d) > 0.
__device__ __forceinline__ float penumbra_width_f(float zmin, float zmax, float zf, float izf, float re,
                                                  float d) {
    const float zm = 0.5f * (zmax + zmin), rs = 0.5f * (zmax - zmin);
    const float hyp2 = zm * zm + re * re;
    if (!(zmin > 0.f && zmax >= zmin && zf > zmax && zm > 0.f && rs * rs <= hyp2 && re > 0.f)) return 0.f;
    // MUFU reciprocals / square roots (the plane is rounded to 16 bits)
    const float sn = fminf(rs * rsqrtf(hyp2), 1.f);
    const float u = sn * rsqrtf(fmaxf(1.f - sn * sn, 0.f));    // tan(theta_d); inf at s = 1
    const float bq = re * (zf - zm) * rcp_approx(zm);
    const float T = (bq + re) * izf;                           // tan(theta)
    const float den_p = 1.f - T * u;                           // cos(theta + theta_d) sign
    if (!(den_p > 0.f)) return 0.f;
    const float ta = __fdividef(T - u, 1.f + T * u), tb = __fdividef(T + u, den_p);
    const float xa = zf * ta - re, xb = zf * tb - re;
    return __fdividef(xa + xb, d);
}

// A staged map region: rows R0 .. R0+RH-1, cols C0 .. C0+RW-1 as depth
// bits (+inf off the map) and its sliding 4 x 4 (min, max) map.
struct Region {
    int R0, C0, RH, RW;
    bool on;
    int* tex;
    int2* blk;
};

// 16-B chunk variant: C0 and RW are multiples of 4, map rows a multiple of 4
// texels (a chunk is wholly on or off the map); asynchronous copies, waited
// for before the barrier that ends staging.
__device__ __forceinline__ void stage_region16(const Region& g, const float* smf, const FrameK& F, int tid) {
    if (!g.on) return;
    const int RQ = g.RW >> 2;
    for (int rr = tid >> 5; rr < g.RH; rr += F5_THREADS / 32) {
        const int r = g.R0 + rr;
        const bool rin = r >= 0 && r < F.hs;
        const float* src = smf + (int64_t)r * F.ws;
        int* dst = g.tex + rr * g.RW;
        for (int q = tid & 31; q < RQ; q += 32) {
            const int c = g.C0 + 4 * q;
            if (rin && c >= 0 && c < F.ws) {
                const unsigned d = (unsigned)__cvta_generic_to_shared(dst + 4 * q);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + c) : "memory");
            } else {
                *reinterpret_cast<int4*>(dst + 4 * q) = make_int4(kInfBits, kInfBits, kInfBits, kInfBits);
            }
        }
    }
}

__device__ __forceinline__ void stage_region(const Region& g, const float* smf, const FrameK& F, int tid) {
    if (!g.on) return;
    // one warp per map row, lanes along it (coalesced, no index division)
    for (int rr = tid >> 5; rr < g.RH; rr += F5_THREADS / 32) {
        const int r = g.R0 + rr;
        const bool rin = r >= 0 && r < F.hs;
        const float* src = smf + (int64_t)r * F.ws;
        int* dst = g.tex + rr * g.RW;
        for (int cc = tid & 31; cc < g.RW; cc += 32) {
            const int c = g.C0 + cc;
            dst[cc] = rin && c >= 0 && c < F.ws ? __float_as_int(__ldg(src + c)) : kInfBits;
        }
    }
}

__device__ __forceinline__ void build_blocks(const Region& g, int tid) {
    if (!g.on) return;
    const int BW = g.RW - 3, BH = g.RH - 3;
    for (int r = tid >> 5; r < BH; r += F5_THREADS / 32)
        for (int c = tid & 31; c < BW; c += 32) {
            int mn[4], mx[4];
#pragma unroll
            for (int dy = 0; dy < 4; ++dy) {
                const int* row = g.tex + (r + dy) * g.RW + c;
                mn[dy] = min(__vimin3_s32(row[0], row[1], row[2]), row[3]);
                mx[dy] = max(__vimax3_s32(row[0], row[1], row[2]), row[3]);
            }
            g.blk[r * BW + c] = make_int2(min(__vimin3_s32(mn[0], mn[1], mn[2]), mn[3]),
                                          max(__vimax3_s32(mx[0], mx[1], mx[2]), mx[3]));
        }
}

__device__ __forceinline__ int region_texels(const int (&b)[4]) {
    return (b[1] - b[0] + 2 * F5_R) * (b[3] - b[2] + 2 * F5_R);
}

// Texel bounding box (row lo, hi, col lo, hi) of the CTA's covered pixels
// of cluster k into bb[k] (warp reduction, then shared atomics).  Ends with
// a barrier; bb[k] must not be read by anyone before the call.
__device__ __forceinline__ void block_bbox(const int (&ri)[4], const int (&ci)[4], const bool (&cov)[4],
                                           const int (&cl)[4], int k, int (*bb)[4], int tid) {
    if (tid == 0) {
        bb[k][0] = INT32_MAX;
        bb[k][1] = INT32_MIN;
        bb[k][2] = INT32_MAX;
        bb[k][3] = INT32_MIN;
    }
    int rlo = INT32_MAX, rhi = INT32_MIN, clo = INT32_MAX, chi = INT32_MIN;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        if (!cov[e] || cl[e] != k) continue;
        rlo = min(rlo, ri[e]);
        rhi = max(rhi, ri[e]);
        clo = min(clo, ci[e]);
        chi = max(chi, ci[e]);
    }
    rlo = __reduce_min_sync(0xffffffffu, rlo);
    rhi = __reduce_max_sync(0xffffffffu, rhi);
    clo = __reduce_min_sync(0xffffffffu, clo);
    chi = __reduce_max_sync(0xffffffffu, chi);
    __syncthreads();
    if ((tid & 31) == 0 && rlo <= rhi) {
        atomicMin(&bb[k][0], rlo);
        atomicMax(&bb[k][1], rhi);
        atomicMin(&bb[k][2], clo);
        atomicMax(&bb[k][3], chi);
    }
    __syncthreads();
}

template <typename T, bool kF32>
__global__ void __launch_bounds__(F5_THREADS, 3) feat5_kernel(const __grid_constant__ Feat5Args a) {
    extern __shared__ __align__(16) int smem5[];
    __shared__ int bb[2][4];
    const int f = blockIdx.z;
    const int tid = threadIdx.x;
    const int X = blockIdx.x * F5_TX + (tid % F5_TX), Y = blockIdx.y * F5_TY + (tid / F5_TX);
    const FrameK& F = a.tab.f[f];
    if (tid == 0) bb[1][0] = INT32_MAX, bb[1][1] = INT32_MIN;   // cluster 1 empty unless split
    const int64_t hw = (int64_t)a.h * a.w;
    const int64_t base = (int64_t)f * a.g.frame_stride;
    const float* gd = reinterpret_cast<const float*>(a.g.d) + base;
    const float* gp = reinterpret_cast<const float*>(a.g.position) + 3 * base;
    const float* gn = reinterpret_cast<const float*>(a.g.normal) + 3 * base;
    // the 2 x 2 frame pixels of this level-0 pixel, e = 2 dy + dx
    float dv[4], pxv[4], pyv[4], pzv[4], nxv[4], nyv[4], nzv[4];
    int ri[4], ci[4];
    bool cov[4];
    // rows 2Y and 2Y+1, columns 2X and 2X+1: 8-byte loads when w is even
    const bool pairs = (a.w & 1) == 0 && 2 * X + 1 < a.w;
#pragma unroll
    for (int dy = 0; dy < 2; ++dy) {
        const int y = 2 * Y + dy, x = 2 * X;
        const int e0 = 2 * dy, e1 = e0 + 1;
        const int64_t p = (int64_t)y * a.w + x;
        if (y < a.h && pairs) {
            const float2 dd = __ldg(reinterpret_cast<const float2*>(gd + p));
            dv[e0] = dd.x;
            dv[e1] = dd.y;
        } else {
            dv[e0] = y < a.h && x < a.w ? __ldg(gd + p) : 0.f;
            dv[e1] = y < a.h && x + 1 < a.w ? __ldg(gd + p + 1) : 0.f;
        }
        cov[e0] = dv[e0] > 0.f;
        cov[e1] = dv[e1] > 0.f;
        pxv[e0] = pyv[e0] = pzv[e0] = nxv[e0] = nyv[e0] = nzv[e0] = 0.f;
        pxv[e1] = pyv[e1] = pzv[e1] = nxv[e1] = nyv[e1] = nzv[e1] = 0.f;
        ri[e0] = ci[e0] = ri[e1] = ci[e1] = 0;
        if (pairs && (cov[e0] || cov[e1])) {
            auto ld2 = [&](const float* b, float& u, float& v) {
                const float2 t = __ldg(reinterpret_cast<const float2*>(b + p));
                u = t.x;
                v = t.y;
            };
            ld2(gp, pxv[e0], pxv[e1]);
            ld2(gp + hw, pyv[e0], pyv[e1]);
            ld2(gp + 2 * hw, pzv[e0], pzv[e1]);
            ld2(gn, nxv[e0], nxv[e1]);
            ld2(gn + hw, nyv[e0], nyv[e1]);
            ld2(gn + 2 * hw, nzv[e0], nzv[e1]);
        } else {
#pragma unroll
            for (int e = e0; e <= e1; ++e) {
                if (!cov[e]) continue;
                const int64_t q = p + (e - e0);
                pxv[e] = __ldg(gp + q);
                pyv[e] = __ldg(gp + hw + q);
                pzv[e] = __ldg(gp + 2 * hw + q);
                nxv[e] = __ldg(gn + q);
                nyv[e] = __ldg(gn + hw + q);
                nzv[e] = __ldg(gn + 2 * hw + q);
            }
        }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        if (!cov[e]) continue;
        const bool ok = texel_fused(F, pxv[e], pyv[e], pzv[e], ri[e], ci[e]);
        const int y = 2 * Y + (e >> 1), x = 2 * X + (e & 1);
        if (!ok) atomic_min_i64(a.first_bad + f, (int64_t)y * a.w + x);
        if (a.tidx) {
            int32_t* ti = a.tidx + (int64_t)f * 2 * hw + (int64_t)y * a.w + x;
            ti[0] = ri[e];
            ti[hw] = ci[e];
        }
    }
    // Texel bounding box of the tile; when its window region does not fit
    // the shared-memory budget (a tile across an occluder edge maps to two
    // separate map areas), the covered pixels are split in two clusters at
    // the middle of the longer bbox side, each with its own region.
    int cl[4] = {0, 0, 0, 0};
    block_bbox(ri, ci, cov, cl, 0, bb, tid);
    const bool any = bb[0][0] <= bb[0][1];
    int nreg = 0;
    if (any && region_texels(bb[0]) > F5_MAX_TEX) {
        const bool by_rows = bb[0][1] - bb[0][0] >= bb[0][3] - bb[0][2];
        const int sv = by_rows ? (bb[0][0] + bb[0][1]) >> 1 : (bb[0][2] + bb[0][3]) >> 1;
#pragma unroll
        for (int e = 0; e < 4; ++e) cl[e] = ((by_rows ? ri[e] : ci[e]) > sv) ? 1 : 0;
        __syncthreads();            // every thread has read bb[0]
        block_bbox(ri, ci, cov, cl, 0, bb, tid);
        block_bbox(ri, ci, cov, cl, 1, bb, tid);
        nreg = 2;
    } else if (any) {
        nreg = 1;
    }
    // regions: A = cluster 0 (or all), B = cluster 1; staged if they fit
    const float* smf = a.sm + (int64_t)f * a.sm_stride;
    int* regs = smem5;                                           // depth bits
    int2* blks = reinterpret_cast<int2*>(smem5 + F5_MAX_TEX);     // sliding 4x4 (min, max)
    // 16-B staging when map rows are 16-B aligned: region columns widened
    // to whole chunks
    const bool vec4 = (F.ws & 3) == 0 && (reinterpret_cast<uintptr_t>(smf) & 15) == 0;
    const int cmask = vec4 ? ~3 : ~0;
    Region RA, RB;
    RA.R0 = bb[0][0] - F5_R;
    RA.C0 = (bb[0][2] - F5_R) & cmask;
    RA.RH = bb[0][1] - bb[0][0] + 2 * F5_R;
    RA.RW = ((bb[0][3] + F5_R - RA.C0) + ~cmask) & cmask;
    RA.on = nreg >= 1 && bb[0][0] <= bb[0][1] && RA.RH * RA.RW <= F5_MAX_TEX;
    RA.tex = regs;
    RA.blk = blks;
    const int usedA = RA.on ? RA.RH * RA.RW : 0, busedA = RA.on ? (RA.RH - 3) * (RA.RW - 3) : 0;
    RB.R0 = bb[1][0] - F5_R;
    RB.C0 = (bb[1][2] - F5_R) & cmask;
    RB.RH = bb[1][1] - bb[1][0] + 2 * F5_R;
    RB.RW = ((bb[1][3] + F5_R - RB.C0) + ~cmask) & cmask;
    RB.on = nreg == 2 && bb[1][0] <= bb[1][1] && usedA + RB.RH * RB.RW <= F5_MAX_TEX;
    RB.tex = regs + usedA;
    RB.blk = blks + busedA;
    if (vec4) {
        stage_region16(RA, smf, F, tid);
        stage_region16(RB, smf, F, tid);
        asm volatile("cp.async.wait_all;" ::: "memory");
    } else {
        stage_region(RA, smf, F, tid);
        stage_region(RB, smf, F, tid);
    }
    __syncthreads();
    build_blocks(RA, tid);
    build_blocks(RB, tid);

    // phase A, per pixel: the 4 reference planes (fp32 math as the fused
    // 4-plane producer), the exact blocker threshold, the window key
    float feat[4][5];
    float zfv[4];
    int thrv[4], key[4];
    const double bias = F.bias;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
#pragma unroll
        for (int k = 0; k < 5; ++k) feat[e][k] = 0.f;
        zfv[e] = 1.f;
        thrv[e] = 0;
        key[e] = -2;                                    // -2 uncovered, -1 window not staged
        if (!cov[e]) continue;
        // z_f in fp64 as render_gbuffer (raster.py:228): the blocker test
        // t < z_f - b must classify exactly like the fp64 oracle
        const double tx = F.ec[0] - (double)pxv[e], ty = F.ec[1] - (double)pyv[e], tz = F.ec[2] - (double)pzv[e];
        const double zf64 = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(tx, tx), __dmul_rn(ty, ty)), __dmul_rn(tz, tz)));
        const float zf = (float)zf64;
        zfv[e] = zf;
        thrv[e] = __float_as_int(__double2float_ru(zf64 - bias));   // t < thr64 <=> t < thr (fp32 t)
        const float izf = rcp_approx(zf);
        const float ftx = (float)tx, fty = (float)ty, ftz = (float)tz;
        const float ce = __saturatef((nxv[e] * ftx + nyv[e] * fty + nzv[e] * ftz) * izf);
        const float dx = F.fcp[0] - pxv[e], dy = F.fcp[1] - pyv[e], dz = F.fcp[2] - pzv[e];
        const float cc = __saturatef((nxv[e] * dx + nyv[e] * dy + nzv[e] * dz) * rsqrtf(dx * dx + dy * dy + dz * dz));
        const int tr = ri[e], tc = ci[e];
        const bool k1 = cl[e] != 0;
        const bool st = k1 ? RB.on : RA.on;
        const int W_ = k1 ? RB.RW : RA.RW;
        const int loc = (tr - (k1 ? RB.R0 : RA.R0)) * W_ + (tc - (k1 ? RB.C0 : RA.C0));
        const float look = st ? __int_as_float((k1 ? RB.tex : RA.tex)[loc]) : __ldg(smf + (int64_t)tr * F.ws + tc);
        if (st) key[e] = (k1 ? usedA : 0) + loc;
        else key[e] = -1;
        float ch0 = 0.f, ch1 = 1.f;
        if (look < INFINITY) {                                       // raster.py:262
            const float m = fminf(look, zf);
            ch0 = (m - zf) + F.fbias;
            ch1 = (m + F.fbias) * izf;
        }
        feat[e][0] = ch0;
        feat[e][1] = ch1;
        feat[e][2] = ce + F.fsize;
        feat[e][3] = cc * rcp_approx(dv[e]);
    }
    __syncthreads();   // block maps built
    // phase 3, per pixel: combine the window summary with its own threshold
    const float re = (float)(F.size_index * (0.5 / 2.0 / 4.0));       // scene.emitter_radius
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        if (key[e] == -2) continue;
        const int thr = thrv[e];
        const unsigned thr1 = (unsigned)thr - 1u;
        const int tr = ri[e], tc = ci[e];
        int zmin = kInfBits, zmx = -1;
        {
            // the pixel's scan: over the staged blocks, or straight from global
            // memory (window outside the staged regions)
            unsigned um = 0xffffffffu;
            zmin = kInfBits;
            const bool k1 = cl[e] != 0;
            const bool st = k1 ? RB.on : RA.on;
            if (st) {
                const int W_ = k1 ? RB.RW : RA.RW, BW = W_ - 3;
                const int r0 = tr - F5_R - (k1 ? RB.R0 : RA.R0), c0 = tc - F5_R - (k1 ? RB.C0 : RA.C0);
                const int2* blk = k1 ? RB.blk : RA.blk;
                const int* reg = k1 ? RB.tex : RA.tex;
                unsigned strad = 0;
                int zq[4] = {kInfBits, kInfBits, kInfBits, kInfBits};
                unsigned ub[4] = {um, um, um, um};
#pragma unroll
                for (int b = 0; b < 16; ++b) {
                    const int2 mm = blk[(r0 + 4 * (b >> 2)) * BW + c0 + 4 * (b & 3)];
                    zq[b & 3] = min(zq[b & 3], mm.x);
                    if (mm.y < thr) ub[b & 3] = min(ub[b & 3], thr1 - (unsigned)mm.y);
                    else if (mm.x < thr) strad |= 1u << b;
                }
                zmin = min(min(zq[0], zq[1]), min(zq[2], zq[3]));
                um = min(min(ub[0], ub[1]), min(ub[2], ub[3]));
                // one accumulator per block row: four independent DPX chains
                unsigned uq[4] = {um, 0xffffffffu, 0xffffffffu, 0xffffffffu};
                while (strad) {
                    const int b = __ffs(strad) - 1;
                    strad &= strad - 1;
                    const int* p = reg + (r0 + 4 * (b >> 2)) * W_ + c0 + 4 * (b & 3);
#pragma unroll
                    for (int dy = 0; dy < 4; ++dy)
#pragma unroll
                        for (int dxx = 0; dxx < 4; ++dxx)
                            uq[dy] = __viaddmin_u32(thr1, (unsigned)(-p[dy * W_ + dxx]), uq[dy]);
                }
                um = min(min(uq[0], uq[1]), min(uq[2], uq[3]));
            } else if (vec4 && tr >= F5_R && tr + F5_R <= F.hs && tc >= F5_R && tc + F5_R <= F.ws) {
                // 16 texel rows from global memory (L1 / L2) as the aligned
                // 16-B blocks covering each window row (4 or 5 per row; map
                // rows are a multiple of 4 texels, so no block crosses a row),
                // the compiler keeps two rows in flight; texels outside the
                // window are masked to +inf (neutral for both scans)
                const int cs = tc - F5_R, m = cs & 3;
                const float4* rowp = reinterpret_cast<const float4*>(smf + (int64_t)(tr - F5_R) * F.ws + (cs - m));
                const int rq = F.ws >> 2;
                int zq[4] = {kInfBits, kInfBits, kInfBits, kInfBits};
                unsigned uq[4] = {um, um, um, um};
#pragma unroll 2
                for (int r = 0; r < 2 * F5_R; ++r, rowp += rq) {
                    float4 v[5];
#pragma unroll
                    for (int b = 0; b < 4; ++b) v[b] = __ldg(rowp + b);
                    v[4] = m ? __ldg(rowp + 4) : make_float4(INFINITY, INFINITY, INFINITY, INFINITY);
                    int t[20];
#pragma unroll
                    for (int b = 0; b < 5; ++b) {
                        t[4 * b] = __float_as_int(v[b].x);
                        t[4 * b + 1] = __float_as_int(v[b].y);
                        t[4 * b + 2] = __float_as_int(v[b].z);
                        t[4 * b + 3] = __float_as_int(v[b].w);
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (j < m) t[j] = kInfBits;             // left of the window
                        if (j >= m) t[16 + j] = kInfBits;       // right of it
                    }
#pragma unroll
                    for (int c = 0; c < 20; c += 2) {
                        const int q = (c >> 1) & 3;
                        zq[q] = __vimin3_s32(t[c], t[c + 1], zq[q]);
                        uq[q] = __viaddmin_u32(thr1, (unsigned)(-t[c]), uq[q]);
                        uq[q] = __viaddmin_u32(thr1, (unsigned)(-t[c + 1]), uq[q]);
                    }
                }
                zmin = min(min(zq[0], zq[1]), min(zq[2], zq[3]));
                um = min(min(uq[0], uq[1]), min(uq[2], uq[3]));
            } else if (tr >= F5_R && tr + F5_R <= F.hs && tc >= F5_R && tc + F5_R <= F.ws) {
                // 16 texel rows from global memory (L1 / L2), two rows (32
                // loads) in flight per round trip
                const float* rowp = smf + (int64_t)(tr - F5_R) * F.ws + (tc - F5_R);
                int zq[4] = {kInfBits, kInfBits, kInfBits, kInfBits};
                unsigned uq[4] = {um, um, um, um};
                for (int r = 0; r < 2 * F5_R; r += 2, rowp += 2 * F.ws) {
                    int t[32];
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        t[c] = __float_as_int(__ldg(rowp + c));
                        t[16 + c] = __float_as_int(__ldg(rowp + F.ws + c));
                    }
#pragma unroll
                    for (int c = 0; c < 32; c += 2) {
                        zq[(c >> 1) & 3] = __vimin3_s32(t[c], t[c + 1], zq[(c >> 1) & 3]);
                        uq[(c >> 1) & 3] = __viaddmin_u32(thr1, (unsigned)(-t[c]), uq[(c >> 1) & 3]);
                        uq[(c >> 1) & 3] = __viaddmin_u32(thr1, (unsigned)(-t[c + 1]), uq[(c >> 1) & 3]);
                    }
                }
                zmin = min(min(zq[0], zq[1]), min(zq[2], zq[3]));
                um = min(min(uq[0], uq[1]), min(uq[2], uq[3]));
            } else {
                // window clipped by the map border (rare): bounds-checked scan
                for (int r = tr - F5_R; r < tr + F5_R; ++r) {
                    if (r < 0 || r >= F.hs) continue;
                    for (int c = tc - F5_R; c < tc + F5_R; ++c) {
                        if (c < 0 || c >= F.ws) continue;
                        const int t = __float_as_int(__ldg(smf + (int64_t)r * F.ws + c));
                        zmin = min(zmin, t);
                        um = __viaddmin_u32(thr1, (unsigned)(-t), um);
                    }
                }
            }
            zmx = (int)(thr1 - um);
        }
        if (a.dbg) {
            const int y = 2 * Y + (e >> 1), x = 2 * X + (e & 1);
            int32_t* d4 = a.dbg + (((int64_t)f * a.h + y) * a.w + x) * 4;
            d4[0] = zmin;
            d4[1] = zmx;
            d4[2] = thr;
            d4[3] = (key[e] < 0 ? 1 : 0) | (cl[e] << 3);
        }
        if (zmin < thr)                                            // blockers exist
            feat[e][4] = penumbra_width_f(__int_as_float(zmin), __int_as_float(zmx), zfv[e], rcp_approx(zfv[e]), re,
                                           dv[e]);
    }

    if constexpr (kF32) {
        float* o = reinterpret_cast<float*>(a.out) + (int64_t)f * 5 * hw;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int y = 2 * Y + (e >> 1), x = 2 * X + (e & 1);
            if (y >= a.h || x >= a.w) continue;
            const int64_t p = (int64_t)y * a.w + x;
#pragma unroll
            for (int k = 0; k < 5; ++k) o[k * hw + p] = feat[e][k];
        }
    } else {
    if (Y >= a.H0 || X >= a.W0) return;
    T* o = reinterpret_cast<T*>(a.out);
    const int64_t plane = (int64_t)a.H0 * a.W0 * 8;
    const int64_t at = ((int64_t)f * 3 * a.H0 * a.W0 + (int64_t)Y * a.W0 + X) * 8;
    uint4 c0, c1, c2;
    c0.x = Elem<T>::pack(feat[0][0], feat[0][1]);
    c0.y = Elem<T>::pack(feat[0][2], feat[0][3]);
    c0.z = Elem<T>::pack(feat[1][0], feat[1][1]);
    c0.w = Elem<T>::pack(feat[1][2], feat[1][3]);
    c1.x = Elem<T>::pack(feat[2][0], feat[2][1]);
    c1.y = Elem<T>::pack(feat[2][2], feat[2][3]);
    c1.z = Elem<T>::pack(feat[3][0], feat[3][1]);
    c1.w = Elem<T>::pack(feat[3][2], feat[3][3]);
    // 16-bit range: a degenerate penumbra (theta + theta_d -> pi/2) saturates
    auto sat = [](float v) { return fminf(fmaxf(v, -60000.f), 60000.f); };
    c2.x = Elem<T>::pack(sat(feat[0][4]), sat(feat[1][4]));
    c2.y = Elem<T>::pack(sat(feat[2][4]), sat(feat[3][4]));
    c2.z = 0u;
    c2.w = 0u;
    *reinterpret_cast<uint4*>(o + at) = c0;
    *reinterpret_cast<uint4*>(o + at + plane) = c1;
    *reinterpret_cast<uint4*>(o + at + 2 * plane) = c2;
    }
}

}  // namespace

// 16-bit mode: x5 = (nf, 3, H0, W0, 8) of the chunk's frames (fp16 / bf16);
// fp32 mode: planes (nf, 5, h, w).  first_bad must be pre-filled.
nsm_status launch_feat5(const nsm_gbuffer* g, const float* sm, int64_t sm_stride, const nsm_frame* frames,
                        int nf, int h, int w, int H0, int W0, void* out, int out_kind, int64_t* first_bad,
                        int32_t* tidx, cudaStream_t st, int32_t* dbg) {
    if (g->dtype != NSM_F32 || g->z_f || g->c_e || g->c_c || g->coverage)
        return fail(NSM_ERR_UNSUPPORTED, "the 5-plane feature pass reads fp32 d / normal / position planes");
    if (nf > NSM_MAX_FRAMES_PER_LAUNCH) return fail(NSM_ERR_ARG, "launch_feat5: too many frames");
    Feat5Args a{};
    a.g = GBufK{g->d, g->normal, g->position, nullptr, nullptr, nullptr, nullptr, g->frame_stride};
    a.sm = sm;
    a.sm_stride = sm_stride;
    make_frame_table(frames, nf, a.tab);
    a.h = h;
    a.w = w;
    a.H0 = H0;
    a.W0 = W0;
    a.out = out;
    a.first_bad = first_bad;
    a.tidx = tidx;
    a.dbg = dbg;
    // 16-bit: every level-0 pixel of the padded grid; fp32: the frame's pixels
    const int LX = out_kind == 2 ? (w + 1) / 2 : W0, LY = out_kind == 2 ? (h + 1) / 2 : H0;
    dim3 grid((LX + F5_TX - 1) / F5_TX, (LY + F5_TY - 1) / F5_TY, nf);
    static std::atomic<uint64_t> attr[3];           // per device: the attribute is per-device state
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr[out_kind].fetch_or(1ull << (dev & 63)) & (1ull << (dev & 63)))) {
        cudaFuncSetAttribute(out_kind == 0 ? (const void*)feat5_kernel<__half, false>
                             : out_kind == 1 ? (const void*)feat5_kernel<__nv_bfloat16, false>
                                             : (const void*)feat5_kernel<float, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, F5_SMEM);
    }
    NSM_PROF("feat5_blocker", st);
    switch (out_kind) {
        case 0:
            feat5_kernel<__half, false><<<grid, F5_THREADS, F5_SMEM, st>>>(a);
            break;
        case 1:
            feat5_kernel<__nv_bfloat16, false><<<grid, F5_THREADS, F5_SMEM, st>>>(a);
            break;
        default:
            feat5_kernel<float, true><<<grid, F5_THREADS, F5_SMEM, st>>>(a);
            break;
    }
    return NSM_OK;
}

}  // namespace nsm
