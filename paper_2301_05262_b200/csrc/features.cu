// Stage 1 standalone: raster.assemble_features (raster.py:266-278) on the GPU.
//
// One thread per camera pixel, grid.z = frame.  Reads the planar G-buffer
// (coalesced along x), projects the world position into the emitter frustum
// in fp64 (bit-exact np.rint texel indices), gathers the shadow map, and
// writes the 4 fp32 planes.  This is the drop-in for the numpy entry point and
// the stage-1 parity kernel; the fp16 hot path fuses the same per-pixel math
// into the level-0 encoder (net_f16.cu) and never writes these planes.
#include "common.cuh"
#include "prof.cuh"

namespace nsm {

// Derived planes of render_gbuffer (raster.py:227-232) from depth/normal/pos.
struct Derived {
    double z_f, c_e, c_c;
};

__device__ __forceinline__ Derived derive(const FrameK& f, int y, int x, double nx, double ny,
                                          double nz, double px, double py, double pz) {
    Derived r;
    double tx = f.ec[0] - px, ty = f.ec[1] - py, tz = f.ec[2] - pz;
    r.z_f = sqrt(tx * tx + ty * ty + tz * tz);
    double ce = (nx * (tx / r.z_f) + ny * (ty / r.z_f) + nz * (tz / r.z_f));
    r.c_e = fmin(fmax(ce, 0.0), 1.0);
    double ray[3];
    camera_ray(f, y, x, ray);
    double cc = -(nx * ray[0] + ny * ray[1] + nz * ray[2]);
    r.c_c = fmin(fmax(cc, 0.0), 1.0);
    return r;
}

template <typename T, bool kGiven>
__global__ void __launch_bounds__(256) features_kernel(GBufK g, const float* __restrict__ sm,
                                                       int64_t sm_stride, FrameTable tab, int h,
                                                       int w, int ho, int wo, float* __restrict__ out,
                                                       int32_t* __restrict__ tidx,
                                                       int64_t* __restrict__ first_bad) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    const int fr = blockIdx.z;
    if (x >= wo || y >= ho) return;
    const FrameK& f = tab.f[fr];
    // output planes may be padded past the frame (rows/cols >= h/w are
    // uncovered, zero features); texel indices use the output geometry too
    const int64_t ohw = (int64_t)ho * wo;
    const int64_t opix = (int64_t)y * wo + x;
    float* o = out + (int64_t)fr * 4 * ohw + opix;
    const int64_t hw = (int64_t)h * w;
    const int64_t pix = (int64_t)y * w + x;
    const int64_t base = (int64_t)fr * g.frame_stride;

    const bool inside = x < w && y < h;
    const double d = inside ? ldd<T>(g.d, base + pix) : 0.0;
    const bool cov = inside && (g.coverage ? (g.coverage[base + pix] != 0) : (d > 0.0));
    if (!cov) {
        o[0] = 0.f;
        o[ohw] = 0.f;
        o[2 * ohw] = 0.f;
        o[3 * ohw] = 0.f;
        if (tidx) {
            tidx[(int64_t)fr * 2 * ohw + opix] = -1;
            tidx[(int64_t)fr * 2 * ohw + ohw + opix] = -1;
        }
        return;
    }
    const int64_t pb = 3 * base;
    const double px = ldd<T>(g.position, pb + pix);
    const double py = ldd<T>(g.position, pb + hw + pix);
    const double pz = ldd<T>(g.position, pb + 2 * hw + pix);
    Derived dv;
    if (kGiven) {
        dv.z_f = ldd<T>(g.z_f, base + pix);
        dv.c_e = ldd<T>(g.c_e, base + pix);
        dv.c_c = ldd<T>(g.c_c, base + pix);
    } else {
        const double nx = ldd<T>(g.normal, pb + pix);
        const double ny = ldd<T>(g.normal, pb + hw + pix);
        const double nz = ldd<T>(g.normal, pb + 2 * hw + pix);
        dv = derive(f, y, x, nx, ny, nz, px, py, pz);
    }
    int ri, ci;
    if (!texel_of(f, px, py, pz, ri, ci)) atomic_min_i64(first_bad + fr, pix);
    if (tidx) {
        tidx[(int64_t)fr * 2 * ohw + opix] = ri;
        tidx[(int64_t)fr * 2 * ohw + ohw + opix] = ci;
    }
    const double look = (double)__ldg(sm + fr * sm_stride + (int64_t)ri * f.ws + ci);
    // _shadow_lookup (raster.py:262): misses clamp to z_f, beyond-receiver
    // occluders clamp to the receiver, then the acne bias.
    const double z = isfinite(look) ? fmin(look, dv.z_f) + f.bias : dv.z_f;
    o[0] = (float)(z - dv.z_f);
    o[ohw] = (float)(z / dv.z_f);
    o[2 * ohw] = (float)(dv.c_e + f.size_index);
    o[3 * ohw] = (float)(dv.c_c / d);
}

__global__ void fill_i64(int64_t* p, int n, int64_t v) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

void launch_fill_i64(int64_t* p, int n, int64_t v, cudaStream_t st) {
    NSM_PROF("fill_i64", st);
    fill_i64<<<(n + 127) / 128, 128, 0, st>>>(p, n, v);
}

nsm_status launch_features(const nsm_gbuffer* g, const float* sm, int64_t sm_stride,
                           const nsm_frame* frames, int32_t n, int32_t h, int32_t w,
                           int32_t ho, int32_t wo, float* out, int32_t* tidx,
                           int64_t* first_bad, cudaStream_t st) {
    GBufK gk{g->d, g->normal, g->position, g->z_f, g->c_e, g->c_c, g->coverage, g->frame_stride};
    const bool given = g->z_f && g->c_e && g->c_c;
    {
        NSM_PROF("fill_i64", st);
        fill_i64<<<(n + 127) / 128, 128, 0, st>>>(first_bad, n, INT64_MAX);
    }
    for (int32_t f0 = 0; f0 < n; f0 += NSM_MAX_FRAMES_PER_LAUNCH) {
        const int nf = min(n - f0, NSM_MAX_FRAMES_PER_LAUNCH);
        FrameTable tab;
        make_frame_table(frames + f0, nf, tab);
        GBufK gf = gk;
        const int64_t es = g->dtype == NSM_F64 ? 8 : 4;
        auto adv = [&](const void* p, int64_t planes) -> const void* {
            return p ? (const void*)((const char*)p + es * planes * f0 * g->frame_stride) : nullptr;
        };
        gf.d = adv(g->d, 1);
        gf.normal = adv(g->normal, 3);
        gf.position = adv(g->position, 3);
        gf.z_f = adv(g->z_f, 1);
        gf.c_e = adv(g->c_e, 1);
        gf.c_c = adv(g->c_c, 1);
        gf.coverage = g->coverage ? g->coverage + f0 * g->frame_stride : nullptr;
        const float* smf = sm + f0 * sm_stride;
        float* of = out + (int64_t)f0 * 4 * ho * wo;
        int32_t* tf = tidx ? tidx + (int64_t)f0 * 2 * ho * wo : nullptr;
        dim3 blk(32, 8), grd((wo + 31) / 32, (ho + 7) / 8, nf);
        if (g->dtype == NSM_F64) {
            if (given)
                {
                    NSM_PROF("features_kernel", st);
                    features_kernel<double, true><<<grd, blk, 0, st>>>(gf, smf, sm_stride, tab, h, w, ho, wo, of, tf, first_bad + f0);
                }
            else
                {
                    NSM_PROF("features_kernel", st);
                    features_kernel<double, false><<<grd, blk, 0, st>>>(gf, smf, sm_stride, tab, h, w, ho, wo, of, tf, first_bad + f0);
                }
        } else {
            if (given)
                {
                    NSM_PROF("features_kernel", st);
                    features_kernel<float, true><<<grd, blk, 0, st>>>(gf, smf, sm_stride, tab, h, w, ho, wo, of, tf, first_bad + f0);
                }
            else
                {
                    NSM_PROF("features_kernel", st);
                    features_kernel<float, false><<<grd, blk, 0, st>>>(gf, smf, sm_stride, tab, h, w, ho, wo, of, tf, first_bad + f0);
                }
        }
    }
    NSM_CUDA_TRY(cudaGetLastError());
    return NSM_OK;
}

}  // namespace nsm

// ---------------------------------------------------------------------------
// Blocker-search penumbra plane (BASELINE configs 3/4 extension; no reference
// implementation -- parity is against oracle/blocker.py).  Per covered pixel:
// the nearest texel exactly as _shadow_lookup, a (2R)x(2R) texel window,
// blockers = finite depths < z_f - b, (z_min, z_max) -> the bounding-sphere
// penumbra model of analysis.penumbra_extents (analysis.py:240-269) with the
// emitter radius, and the screen-space width (x_a + x_b) * focal_px / d
// (analysis.py:319-320) in units of the focal length, i.e. (x_a + x_b) / d
// (resolution independent, O(0.1): see oracle/blocker.py for why not pixels).
// 0 where uncovered / no blockers / invalid geometry.
namespace nsm {

__device__ double penumbra_width(double zmin, double zmax, double zf, double re, double d) {
    const double zm = (zmax + zmin) / 2.0, rs = (zmax - zmin) / 2.0;
    const double hyp = sqrt(zm * zm + re * re);
    if (!(zmin > 0.0 && zmax >= zmin && zf > zmax && zm > 0.0 && rs <= hyp && re > 0.0)) return 0.0;
    const double td = asin(rs / hyp);
    const double bq = re * (zf - zm) / zm;
    const double th = atan((bq + re) / zf);
    if (!(th + td < 1.5707963267948966)) return 0.0;
    const double xa = zf * tan(th - td) - re, xb = zf * tan(th + td) - re;
    return (xa + xb) / d;
}

template <typename T>
__global__ void __launch_bounds__(256) blocker_kernel(GBufK g, const float* __restrict__ sm, int64_t sm_stride,
                                                      FrameTable tab, int h, int w, int radius,
                                                      float* __restrict__ out, int64_t* __restrict__ first_bad) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    const int fr = blockIdx.z;
    if (x >= w || y >= h) return;
    const FrameK& f = tab.f[fr];
    const int64_t hw = (int64_t)h * w, pix = (int64_t)y * w + x, base = (int64_t)fr * g.frame_stride;
    float* o = out + (int64_t)fr * hw + pix;
    const double d = ldd<T>(g.d, base + pix);
    if (!(d > 0.0)) {
        *o = 0.f;
        return;
    }
    const int64_t pb = 3 * base;
    const double px = ldd<T>(g.position, pb + pix), py = ldd<T>(g.position, pb + hw + pix),
                 pz = ldd<T>(g.position, pb + 2 * hw + pix);
    const double tx = f.ec[0] - px, ty = f.ec[1] - py, tz = f.ec[2] - pz;
    const double zf = sqrt(tx * tx + ty * ty + tz * tz);
    int ri, ci;
    if (!texel_of(f, px, py, pz, ri, ci)) atomic_min_i64(first_bad + fr, pix);
    const double thr = zf - f.bias;
    const float* smf = sm + fr * sm_stride;
    float zmin = INFINITY, zmax = -INFINITY;
    const int r0 = max(ri - radius, 0), r1 = min(ri + radius, f.hs);
    const int c0 = max(ci - radius, 0), c1 = min(ci + radius, f.ws);
    for (int r = r0; r < r1; ++r) {
        const float* row = smf + (int64_t)r * f.ws;
        for (int c = c0; c < c1; ++c) {
            const float t = __ldg(row + c);
            if ((double)t < thr) {          // +inf misses never pass
                zmin = fminf(zmin, t);
                zmax = fmaxf(zmax, t);
            }
        }
    }
    double wv = 0.0;
    if (zmin <= zmax) {
        const double re = f.size_index * (0.5 / 2.0 / 4.0);          // scene.emitter_radius
        wv = penumbra_width(zmin, zmax, zf, re, d);
    }
    *o = (float)wv;
}

nsm_status launch_blocker(const nsm_gbuffer* g, const float* sm, int64_t sm_stride, const nsm_frame* frames,
                          int32_t n, int32_t h, int32_t w, int32_t radius, float* out, int64_t* first_bad,
                          cudaStream_t st) {
    GBufK gk{g->d, g->normal, g->position, nullptr, nullptr, nullptr, nullptr, g->frame_stride};
    launch_fill_i64(first_bad, n, INT64_MAX, st);
    for (int32_t f0 = 0; f0 < n; f0 += NSM_MAX_FRAMES_PER_LAUNCH) {
        const int nf = min(n - f0, NSM_MAX_FRAMES_PER_LAUNCH);
        FrameTable tab;
        make_frame_table(frames + f0, nf, tab);
        GBufK gf = gk;
        const int64_t es = g->dtype == NSM_F64 ? 8 : 4;
        gf.d = (const char*)g->d + es * f0 * g->frame_stride;
        gf.position = (const char*)g->position + es * 3 * f0 * g->frame_stride;
        dim3 blk(32, 8), grd((w + 31) / 32, (h + 7) / 8, nf);
        NSM_PROF("blocker_kernel", st);
        if (g->dtype == NSM_F64)
            blocker_kernel<double><<<grd, blk, 0, st>>>(gf, sm + f0 * sm_stride, sm_stride, tab, h, w, radius,
                                                        out + (int64_t)f0 * h * w, first_bad + f0);
        else
            blocker_kernel<float><<<grd, blk, 0, st>>>(gf, sm + f0 * sm_stride, sm_stride, tab, h, w, radius,
                                                       out + (int64_t)f0 * h * w, first_bad + f0);
    }
    NSM_CUDA_TRY(cudaGetLastError());
    return NSM_OK;
}

}  // namespace nsm
