// Input producers: the ray-cast G-buffer and shadow-map passes that feed the
// hot path (raster.render_gbuffer raster.py:217-242, raster.render_shadowmap
// raster.py:206-214).  Untimed supporting kernels: one thread per pixel/texel,
// fp64 like the reference, nearest hit over an analytic primitive table with
// the first object winning ties (Scene.intersect, scene.py:430-441).
#include <math_constants.h>

#include "common.cuh"
#include "prof.cuh"

namespace nsm {

namespace {

constexpr int kRow = 16;  // doubles per primitive row (scenes.primitive_table)

// Plane.intersect (scene.py:218-231): finite rectangle, normal as stored.
__device__ double hit_plane(const double* r, const double o[3], const double d[3], double n[3]) {
    const double den = d[0] * r[4] + d[1] * r[5] + d[2] * r[6];
    const double t = ((r[1] - o[0]) * r[4] + (r[2] - o[1]) * r[5] + (r[3] - o[2]) * r[6]) / den;
    if (!(fabs(den) > 1e-12 && t > 0.0)) return CUDART_INF;
    double hx = o[0] + t * d[0] - r[1], hy = o[1] + t * d[1] - r[2], hz = o[2] + t * d[2] - r[3];
    const double lu = hx * r[7] + hy * r[8] + hz * r[9];
    const double lv = hx * r[10] + hy * r[11] + hz * r[12];
    if (!(fabs(lu) <= r[13] && fabs(lv) <= r[14])) return CUDART_INF;
    n[0] = r[4];
    n[1] = r[5];
    n[2] = r[6];
    return t;
}

// Sphere.intersect (scene.py:260-272).
__device__ double hit_sphere(const double* r, const double o[3], const double d[3], double n[3]) {
    const double ox = o[0] - r[1], oy = o[1] - r[2], oz = o[2] - r[3];
    const double b = ox * d[0] + oy * d[1] + oz * d[2];
    const double c = (ox * ox + oy * oy + oz * oz) - r[4] * r[4];
    const double disc = b * b - c;
    if (!(disc >= 0.0)) return CUDART_INF;
    const double s = sqrt(disc);
    double t = -b - s;
    if (!(t > 1e-12)) {
        t = -b + s;
        if (!(t > 1e-12)) return CUDART_INF;
    }
    n[0] = (o[0] + t * d[0] - r[1]) / r[4];
    n[1] = (o[1] + t * d[1] - r[2]) / r[4];
    n[2] = (o[2] + t * d[2] - r[3]) / r[4];
    return t;
}

// Box.intersect (scene.py:301-326): slabs, degenerate axes, argmax-|local|
// face normal with sign(0) -> +1.
__device__ double hit_box(const double* r, const double o[3], const double d[3], double n[3]) {
    double tn = -CUDART_INF, tf = CUDART_INF;
    for (int a = 0; a < 3; ++a) {
        const double lo = r[1 + a], hi = r[4 + a];
        double t0, t1;
        if (fabs(d[a]) < 1e-15) {
            const bool in = (o[a] >= lo) && (o[a] <= hi);
            t0 = in ? -CUDART_INF : CUDART_INF;
            t1 = in ? CUDART_INF : -CUDART_INF;
        } else {
            const double inv = 1.0 / d[a];
            const double u = (lo - o[a]) * inv, v = (hi - o[a]) * inv;
            t0 = fmin(u, v);
            t1 = fmax(u, v);
        }
        tn = fmax(tn, t0);
        tf = fmin(tf, t1);
    }
    const double t = tn > 1e-12 ? tn : tf;
    if (!(tf >= tn && t > 1e-12)) return CUDART_INF;
    int best = 0;
    double bv = -1.0, loc[3];
    for (int a = 0; a < 3; ++a) {
        const double c = (r[1 + a] + r[4 + a]) / 2.0, hw = (r[4 + a] - r[1 + a]) / 2.0;
        loc[a] = (o[a] + t * d[a] - c) / hw;
        if (fabs(loc[a]) > bv) {  // np.argmax: first maximum wins
            bv = fabs(loc[a]);
            best = a;
        }
    }
    n[0] = n[1] = n[2] = 0.0;
    n[best] = loc[best] > 0.0 ? 1.0 : (loc[best] < 0.0 ? -1.0 : 1.0);
    return t;
}

__device__ double nearest(const double* __restrict__ prims, int np_, const double o[3],
                          const double d[3], double n[3]) {
    double best = CUDART_INF;
    n[0] = n[1] = n[2] = 0.0;
    for (int k = 0; k < np_; ++k) {
        const double* r = prims + (int64_t)k * kRow;
        double nk[3];
        const int kind = (int)r[0];
        const double t = kind == 0 ? hit_plane(r, o, d, nk)
                         : kind == 1 ? hit_sphere(r, o, d, nk)
                                     : hit_box(r, o, d, nk);
        if (t < best) {
            best = t;
            n[0] = nk[0];
            n[1] = nk[1];
            n[2] = nk[2];
        }
    }
    return best;
}

__global__ void gbuffer_kernel(const double* __restrict__ prims, int np_, nsm_camera cam,
                               double half_h, double half_w, float* __restrict__ dout,
                               float* __restrict__ nout, float* __restrict__ pout) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    const int h = cam.height, w = cam.width;
    if (x >= w || y >= h) return;
    FrameK f;
    for (int a = 0; a < 3; ++a) {
        f.cf[a] = cam.forward[a];
        f.cu[a] = cam.up[a];
    }
    f.cr[0] = cam.forward[1] * cam.up[2] - cam.forward[2] * cam.up[1];
    f.cr[1] = cam.forward[2] * cam.up[0] - cam.forward[0] * cam.up[2];
    f.cr[2] = cam.forward[0] * cam.up[1] - cam.forward[1] * cam.up[0];
    f.half_h = half_h;
    f.half_w = half_w;
    f.ch = h;
    f.cw = w;
    double d[3], n[3];
    camera_ray(f, y, x, d);
    const double t = nearest(prims, np_, cam.position, d, n);
    const int64_t hw = (int64_t)h * w, p = (int64_t)y * w + x;
    if (isfinite(t)) {
        dout[p] = (float)(t * (d[0] * cam.forward[0] + d[1] * cam.forward[1] + d[2] * cam.forward[2]));
        for (int a = 0; a < 3; ++a) {
            nout[a * hw + p] = (float)n[a];
            pout[a * hw + p] = (float)(cam.position[a] + t * d[a]);
        }
    } else {
        dout[p] = 0.f;
        for (int a = 0; a < 3; ++a) {
            nout[a * hw + p] = 0.f;
            pout[a * hw + p] = 0.f;
        }
    }
}

// EmitterView.texel_rays (raster.py:75-82) + radial depth.
__global__ void shadowmap_kernel(const double* __restrict__ prims, int np_, nsm_emitter_view v,
                                 float* __restrict__ out) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y * blockDim.y + threadIdx.y;
    if (x >= v.width || y >= v.height) return;
    const double u = ((x + 0.5) / v.width * 2.0 - 1.0) * v.tan_half;
    const double s = (1.0 - (y + 0.5) / v.height * 2.0) * v.tan_half;
    double d[3], n[3];
    for (int a = 0; a < 3; ++a) d[a] = v.forward[a] + u * v.right[a] + s * v.up[a];
    const double inv = 1.0 / sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    for (int a = 0; a < 3; ++a) d[a] *= inv;
    const double t = nearest(prims, np_, v.position, d, n);
    out[(int64_t)y * v.width + x] = (float)t;  // +inf stays +inf
}

}  // namespace

nsm_status launch_render_gbuffer(const double* prims, int32_t n_prims, const nsm_camera* cam,
                                 float* d, float* normal, float* position, cudaStream_t st) {
    const double half_h = tan(cam->fov_y / 2.0);
    const double half_w = half_h * ((double)cam->width / cam->height);
    dim3 blk(32, 8), grd((cam->width + 31) / 32, (cam->height + 7) / 8);
    {
        NSM_PROF("gbuffer_kernel", st);
        gbuffer_kernel<<<grd, blk, 0, st>>>(prims, n_prims, *cam, half_h, half_w, d, normal, position);
    }
    NSM_CUDA_TRY(cudaGetLastError());
    return NSM_OK;
}

nsm_status launch_render_shadowmap(const double* prims, int32_t n_prims,
                                   const nsm_emitter_view* view, float* depth, cudaStream_t st) {
    dim3 blk(32, 8), grd((view->width + 31) / 32, (view->height + 7) / 8);
    {
        NSM_PROF("shadowmap_kernel", st);
        shadowmap_kernel<<<grd, blk, 0, st>>>(prims, n_prims, *view, depth);
    }
    NSM_CUDA_TRY(cudaGetLastError());
    return NSM_OK;
}

}  // namespace nsm
