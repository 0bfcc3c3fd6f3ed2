// Shared device-side definitions for the nsm kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/nsm.h"

namespace nsm {

// Per-frame constants as the kernels read them (kernel parameter, no HBM).
struct FrameK {
    double vp[3], vf[3], vu[3], vr[3];   // emitter view frame (raster.py:64-73)
    double tan_half;
    double cp[3], cf[3], cu[3], cr[3];   // camera frame (scene.py:102-145)
    double half_h, half_w;               // tan(fov/2), tan(fov/2) * w/h
    double ec[3];                        // emitter centre
    double size_index, bias;
    int hs, ws;                          // shadow-map resolution
    int ch, cw;                          // camera resolution (rays)
    // fused-path constants, precomputed on the host (abi.cu make_frame_table)
    double pa, pb, qa, qb;               // col = xr/zc * pa + pb ; row = qb - yr/zc * qa
    double kx[4], ky[4], kz[4];          // pa*xr = kx.p + kx[3], -qa*yr = ky.p + ky[3], zc = kz.p + kz[3]
    float fcp[3];                        // camera position
    float fec[3], fcf[3], fcr[3], fcu[3];
    float fu1, fu0, fw1, fw0;            // u = fx * fu1 + fu0 ; w = fy * fw1 + fw0
    float fbias, fsize;
};

struct FrameTable {
    FrameK f[NSM_MAX_FRAMES_PER_LAUNCH];
};

struct GBufK {
    const void* d;
    const void* normal;
    const void* position;
    const void* z_f;
    const void* c_e;
    const void* c_c;
    const uint8_t* coverage;
    int64_t frame_stride;
};

template <typename T>
__device__ __forceinline__ double ldd(const void* p, int64_t i) {
    return (double)__ldg(reinterpret_cast<const T*>(p) + i);
}

// Unit camera ray through pixel (y, x) centre -- CameraPose.pixel_rays
// (scene.py:153-163); fp64 like the reference.
__device__ __forceinline__ void camera_ray(const FrameK& f, int y, int x, double r[3]) {
    double u = ((x + 0.5) / f.cw * 2.0 - 1.0) * f.half_w;
    double v = (1.0 - (y + 0.5) / f.ch * 2.0) * f.half_h;
    double a = f.cf[0] + u * f.cr[0] + v * f.cu[0];
    double b = f.cf[1] + u * f.cr[1] + v * f.cu[1];
    double c = f.cf[2] + u * f.cr[2] + v * f.cu[2];
    double inv = 1.0 / sqrt(a * a + b * b + c * c);
    r[0] = a * inv;
    r[1] = b * inv;
    r[2] = c * inv;
}

// Nearest shadow-map texel of world point p: EmitterView.project
// (raster.py:84-94) + np.rint (raster.py:249-250, round half to even).
// fp64 throughout: an fp32 projection flips ~1e-4 of the indices.
// Returns false when the point is outside the frustum (raster.py:251).
__device__ __forceinline__ bool texel_of(const FrameK& f, double px, double py, double pz,
                                         int& ri, int& ci) {
    double rx = px - f.vp[0], ry = py - f.vp[1], rz = pz - f.vp[2];
    double zc = rx * f.vf[0] + ry * f.vf[1] + rz * f.vf[2];
    double xr = rx * f.vr[0] + ry * f.vr[1] + rz * f.vr[2];
    double yr = rx * f.vu[0] + ry * f.vu[1] + rz * f.vu[2];
    double den = zc * f.tan_half;
    double xn = xr / den;
    double yn = yr / den;
    double col = (xn + 1.0) / 2.0 * f.ws - 0.5;
    double row = (1.0 - yn) / 2.0 * f.hs - 0.5;
    long long r = __double2ll_rn(row);
    long long c = __double2ll_rn(col);
    bool ok = (zc > 0.0) && r >= 0 && r < f.hs && c >= 0 && c < f.ws;
    ri = (int)min(max(r, 0LL), (long long)f.hs - 1);
    ci = (int)min(max(c, 0LL), (long long)f.ws - 1);
    return ok;
}

// Same texel as texel_of with the affine map folded (one fp64 division):
// col = (xr / zc) * ws / (2 tan) + ws / 2 - 0.5.  Differs from the
// reference's rounding sequence by a few fp64 ulps, i.e. only for values
// within ~1e-12 texel of a half-integer tie.
__device__ __forceinline__ bool texel_fast(const FrameK& f, double px, double py, double pz, int& ri,
                                           int& ci) {
    const double rx = px - f.vp[0], ry = py - f.vp[1], rz = pz - f.vp[2];
    const double zc = rx * f.vf[0] + ry * f.vf[1] + rz * f.vf[2];
    const double xr = rx * f.vr[0] + ry * f.vr[1] + rz * f.vr[2];
    const double yr = rx * f.vu[0] + ry * f.vu[1] + rz * f.vu[2];
    const double inv = 1.0 / zc;
    const double col = fma(xr * inv, f.pa, f.pb);
    const double row = fma(-yr * inv, f.qa, f.qb);
    const long long r = __double2ll_rn(row);
    const long long c = __double2ll_rn(col);
    const bool ok = (zc > 0.0) && r >= 0 && r < f.hs && c >= 0 && c < f.ws;
    ri = (int)min(max(r, 0LL), (long long)f.hs - 1);
    ci = (int)min(max(c, 0LL), (long long)f.ws - 1);
    return ok;
}

// Fused-path texel: the frustum projection as three affine forms of the fp32
// world position evaluated in fp64 (k = scaled view axes, constants folded on
// the host), a Newton-refined fp64 reciprocal of the depth, and int32
// round-half-even conversion.  Agrees with the reference's np.rint index
// except within a few fp64 ulps of a half-texel tie (never observed).
__device__ __forceinline__ bool texel_fused(const FrameK& f, float px, float py, float pz, int& ri,
                                            int& ci) {
    // fp32 -> fp64 without the .ftz flush fast-math would add (G-buffer
    // values are normal or zero)
    double x, y, z;
    asm("cvt.f64.f32 %0, %1;" : "=d"(x) : "f"(px));
    asm("cvt.f64.f32 %0, %1;" : "=d"(y) : "f"(py));
    asm("cvt.f64.f32 %0, %1;" : "=d"(z) : "f"(pz));
    // one constant per DFMA (the second operand comes from a uniform
    // register): the affine offsets k[3] are added last
    const double zc = fma(f.kz[0], x, fma(f.kz[1], y, f.kz[2] * z)) + f.kz[3];
    const double xs = fma(f.kx[0], x, fma(f.kx[1], y, f.kx[2] * z)) + f.kx[3];
    const double ys = fma(f.ky[0], x, fma(f.ky[1], y, f.ky[2] * z)) + f.ky[3];
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(zc));
    double e = fma(-zc, r, 1.0);
    r = fma(r, e, r);
    e = fma(-zc, r, 1.0);
    r = fma(r, e, r);
    const int c = __double2int_rn(fma(xs, r, f.pb));
    const int rr = __double2int_rn(fma(ys, r, f.qb));
    const bool ok = (zc > 0.0) && (unsigned)rr < (unsigned)f.hs && (unsigned)c < (unsigned)f.ws;
    ri = min(max(rr, 0), f.hs - 1);
    ci = min(max(c, 0), f.ws - 1);
    return ok;
}

__device__ __forceinline__ void atomic_min_i64(int64_t* addr, int64_t v) {
    atomicMin(reinterpret_cast<long long*>(addr), (long long)v);
}

}  // namespace nsm

#define NSM_CUDA_TRY(expr)                                                    \
    do {                                                                      \
        cudaError_t _e = (expr);                                              \
        if (_e != cudaSuccess) {                                              \
            return nsm::fail(NSM_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(_e)); \
        }                                                                     \
    } while (0)

namespace nsm {
nsm_status fail(nsm_status code, const char* fmt, ...);
void clear_error();
void make_frame_table(const nsm_frame* frames, int32_t n, FrameTable& tab);
}  // namespace nsm
