// Temporal consumers of the path's output:
//   motion_kernel      raster.motion_vectors      (raster.py:330-358)
//   instability_kernel analysis.temporal_instability (analysis.py:350-377)
// Both are HBM-bound gathers (one reprojected tap per pixel); fp64 where the
// reference computes in fp64 so vectors, masks and the rounded reprojection
// indices agree with it.  Built without --use_fast_math (build.py).
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "net.cuh"
#include "prof.cuh"

namespace nsm {
namespace {

struct CamK {
    double p[3], f[3], r[3], u[3];
    double half_h, half_w;
    int h, w;
};

CamK make_cam(const nsm_camera& c) {
    CamK k;
    for (int a = 0; a < 3; ++a) {
        k.p[a] = c.position[a];
        k.f[a] = c.forward[a];
        k.u[a] = c.up[a];
    }
    // CameraPose.right = forward x up (scene.py:143-145)
    k.r[0] = c.forward[1] * c.up[2] - c.forward[2] * c.up[1];
    k.r[1] = c.forward[2] * c.up[0] - c.forward[0] * c.up[2];
    k.r[2] = c.forward[0] * c.up[1] - c.forward[1] * c.up[0];
    k.half_h = std::tan(c.fov_y / 2.0);
    k.half_w = k.half_h * ((double)c.width / c.height);
    k.h = c.height;
    k.w = c.width;
    return k;
}

struct CamTable {
    CamK c[NSM_MAX_FRAMES_PER_LAUNCH];
};

__device__ __forceinline__ double dot3(const double a[3], double x, double y, double z) {
    // rel @ axis, left to right without contraction
    return __dadd_rn(__dadd_rn(__dmul_rn(x, a[0]), __dmul_rn(y, a[1])), __dmul_rn(z, a[2]));
}

template <typename T>
__device__ __forceinline__ bool covered(const GBufK& g, int64_t i) {
    return g.coverage ? g.coverage[i] != 0 : ldd<T>(g.d, i) > 0.0;
}

// One pair (t-1, t) per blockIdx.y: frame t's points reprojected with
// camera t-1 (CameraPose.project, scene.py:165-183).
template <typename T>
__global__ void motion_kernel(GBufK g, CamTable cams, int f0, int h, int w, double* __restrict__ vec,
                              uint8_t* __restrict__ valid) {
    const int pair = blockIdx.y;            // output pair index within this launch
    const int t = f0 + pair + 1;
    const CamK& c = cams.c[pair];
    const int64_t hw = (int64_t)h * w;
    const int64_t bt = (int64_t)t * g.frame_stride, bp = (int64_t)(t - 1) * g.frame_stride;
    double* v = vec + (int64_t)(f0 + pair) * 2 * hw;
    uint8_t* ok = valid + (int64_t)(f0 + pair) * hw;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hw;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int y = (int)(i / w), x = (int)(i % w);
        const double px = ldd<T>(g.position, bt * 3 + i), py = ldd<T>(g.position, bt * 3 + hw + i),
                     pz = ldd<T>(g.position, bt * 3 + 2 * hw + i);
        const double rx = px - c.p[0], ry = py - c.p[1], rz = pz - c.p[2];
        const double zc = dot3(c.f, rx, ry, rz);
        const double xc = dot3(c.r, rx, ry, rz);
        const double yc = dot3(c.u, rx, ry, rz);
        const double xn = xc / (zc * c.half_w);
        const double yn = yc / (zc * c.half_h);
        const double col = __dsub_rn(__dmul_rn(__dmul_rn(xn + 1.0, 0.5), (double)w), 0.5);
        const double row = __dsub_rn(__dmul_rn(__dmul_rn(1.0 - yn, 0.5), (double)h), 0.5);
        const bool cov = covered<T>(g, bt + i);
        v[i] = cov ? row - y : 0.0;
        v[hw + i] = cov ? col - x : 0.0;
        // np.rint + bounds + depth > 0 (raster.py:346-350); NaN/inf -> out of bounds
        bool inb = zc > 0.0 && row > -1.0 && row < (double)h && col > -1.0 && col < (double)w;
        int ri = 0, ci = 0;
        if (inb) {
            ri = (int)__double2ll_rn(row);
            ci = (int)__double2ll_rn(col);
            inb = ri >= 0 && ri < h && ci >= 0 && ci < w;
        }
        bool good = false;
        if (cov && inb) {
            const int64_t j = (int64_t)ri * w + ci;
            if (covered<T>(g, bp + j)) {
                const double pd = ldd<T>(g.d, bp + j);
                const double rel = fabs(pd - zc) / fmax(zc, 1e-12);
                // n_t . n_prev in the planes' precision, summed c0, c1, c2
                bool nok;
                if (sizeof(T) == 4) {
                    const float* nt = reinterpret_cast<const float*>(g.normal);
                    const float a0 = __fmul_rn(nt[bt * 3 + i], nt[bp * 3 + j]);
                    const float a1 = __fmul_rn(nt[bt * 3 + hw + i], nt[bp * 3 + hw + j]);
                    const float a2 = __fmul_rn(nt[bt * 3 + 2 * hw + i], nt[bp * 3 + 2 * hw + j]);
                    // float32 array >= Python float compares in float32 (NEP 50)
                    nok = __fadd_rn(__fadd_rn(a0, a1), a2) >= 0.9f;
                } else {
                    const double* nt = reinterpret_cast<const double*>(g.normal);
                    nok = __dadd_rn(__dadd_rn(__dmul_rn(nt[bt * 3 + i], nt[bp * 3 + j]),
                                             __dmul_rn(nt[bt * 3 + hw + i], nt[bp * 3 + hw + j])),
                                   __dmul_rn(nt[bt * 3 + 2 * hw + i], nt[bp * 3 + 2 * hw + j])) >= 0.9;
                }
                good = rel <= 0.01 && nok;
            }
        }
        ok[i] = good;
    }
}

// Per pair: sum of expm1(alpha |cur - prev[reprojected]|) over valid pixels
// and their count, accumulated into acc[pair] (fp64) / cnt[pair].
__global__ void instability_kernel(const float* __restrict__ vis, const double* __restrict__ vec,
                                   const uint8_t* __restrict__ valid, int h, int w, double alpha,
                                   double* __restrict__ acc, unsigned long long* __restrict__ cnt) {
    const int pair = blockIdx.y;
    const int64_t hw = (int64_t)h * w;
    const float* cur = vis + (int64_t)(pair + 1) * hw;
    const float* prev = vis + (int64_t)pair * hw;
    const double* v = vec + (int64_t)pair * 2 * hw;
    const uint8_t* ok = valid + (int64_t)pair * hw;
    double s = 0.0;
    unsigned int n = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hw;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (!ok[i]) continue;
        const int y = (int)(i / w), x = (int)(i % w);
        // np.clip(np.rint(ys + v), 0, h - 1) (analysis.py:366-367)
        const double ry = rint((double)y + v[i]), rx = rint((double)x + v[hw + i]);
        const int ri = (int)fmin(fmax(ry, 0.0), (double)(h - 1));
        const int ci = (int)fmin(fmax(rx, 0.0), (double)(w - 1));
        const double d = fabs((double)cur[i] - (double)prev[(int64_t)ri * w + ci]);
        s += expm1(alpha * d);
        ++n;
    }
    for (int o = 16; o; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        n += __shfl_xor_sync(0xffffffffu, n, o);
    }
    __shared__ double ss[32];
    __shared__ unsigned int sn[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
        ss[wid] = s;
        sn[wid] = n;
    }
    __syncthreads();
    if (wid == 0) {
        s = lane < (int)(blockDim.x >> 5) ? ss[lane] : 0.0;
        n = lane < (int)(blockDim.x >> 5) ? sn[lane] : 0u;
        for (int o = 16; o; o >>= 1) {
            s += __shfl_xor_sync(0xffffffffu, s, o);
            n += __shfl_xor_sync(0xffffffffu, n, o);
        }
        if (lane == 0 && n) {
            atomicAdd(acc + pair, s);
            atomicAdd(cnt + pair, (unsigned long long)n);
        }
    }
}

}  // namespace

nsm_status launch_motion(const nsm_gbuffer* g, const nsm_camera* cams, int t_frames, int h, int w,
                         double* vec, uint8_t* valid, cudaStream_t st) {
    GBufK gk{g->d, g->normal, g->position, nullptr, nullptr, nullptr, g->coverage, g->frame_stride};
    const int64_t hw = (int64_t)h * w;
    const int gx = (int)std::min<int64_t>((hw + 255) / 256, 148 * 8);
    for (int f0 = 0; f0 < t_frames - 1; f0 += NSM_MAX_FRAMES_PER_LAUNCH) {
        const int np = std::min(NSM_MAX_FRAMES_PER_LAUNCH, t_frames - 1 - f0);
        CamTable tab;
        for (int k = 0; k < np; ++k) tab.c[k] = make_cam(cams[f0 + k]);
        NSM_PROF("motion_kernel", st);
        if (g->dtype == NSM_F64)
            motion_kernel<double><<<dim3(gx, np), 256, 0, st>>>(gk, tab, f0, h, w, vec, valid);
        else
            motion_kernel<float><<<dim3(gx, np), 256, 0, st>>>(gk, tab, f0, h, w, vec, valid);
    }
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? NSM_OK : fail(NSM_ERR_CUDA, "motion_kernel: %s", cudaGetErrorString(e));
}

nsm_status launch_instability(const float* vis, const double* vec, const uint8_t* valid, int t_frames,
                              int h, int w, double alpha, double* acc, unsigned long long* cnt,
                              cudaStream_t st) {
    const int pairs = t_frames - 1;
    cudaMemsetAsync(acc, 0, sizeof(double) * pairs, st);
    cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * pairs, st);
    const int64_t hw = (int64_t)h * w;
    const int gx = (int)std::min<int64_t>((hw + 255) / 256, std::max(1, 148 * 4 / pairs));
    for (int p0 = 0; p0 < pairs; p0 += 65535) {
        const int np = std::min(65535, pairs - p0);
        NSM_PROF("instability_kernel", st);
        instability_kernel<<<dim3(gx, np), 256, 0, st>>>(vis + (int64_t)p0 * hw, vec + (int64_t)p0 * 2 * hw,
                                                         valid + (int64_t)p0 * hw, h, w, alpha, acc + p0,
                                                         cnt + p0);
    }
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? NSM_OK : fail(NSM_ERR_CUDA, "instability_kernel: %s", cudaGetErrorString(e));
}

}  // namespace nsm
