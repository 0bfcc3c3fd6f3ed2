// Stage 2, fp32 reference-precision path: network.forward (network.py:165-209)
// as unfused NCHW fp32 kernels on CUDA cores.  This is the parity anchor for
// the fp32 mode (<= 1e-4 max-abs vs the oracle) and the drop-in for
// `network.forward` on fp32 plans; the fp16/bf16 plans run the fused
// tensor-core level kernels of net_f16.cu instead.
#include <algorithm>

#include "common.cuh"
#include "prof.cuh"
#include "net.cuh"

namespace nsm {

namespace {

constexpr int kTX = 32, kTY = 16;   // output pixels per CTA (x, y): 2 per thread, x and x + 16
constexpr int kThr = 256;
constexpr int kCo = 16;             // output channels per CTA
constexpr int kCi = 8;              // input channels staged per step

// autodiff.conv2d (autodiff.py:146-166): zero-padded cross-correlation,
// k in {1, 3}, stride 1, + bias, optional ReLU (autodiff.py:190-191).
// Register-blocked: each thread accumulates 2 pixels x 16 output channels;
// per (input channel, tap) it reads 2 staged inputs and the 16 weights as 4
// broadcast 16-B loads, i.e. 32 FMAs per 6 shared loads.
template <int K>
__global__ void __launch_bounds__(kThr) conv_f32_kernel(
    const float* __restrict__ x, int cin, int h, int w, const float* __restrict__ wt,
    const float* __restrict__ bias, int cout, int relu, float* __restrict__ y,
    int64_t x_nstride, int64_t y_nstride) {
    constexpr int P = (K - 1) / 2;
    constexpr int TY = kTY + 2 * P, TX = kTX + 2 * P;
    __shared__ float sx[kCi][TY][TX + 1];
    __shared__ __align__(16) float sw[kCi][K * K][kCo];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int ox = blockIdx.x * kTX + tx, oy = blockIdx.y * kTY + ty;
    const int ngrp = (cout + kCo - 1) / kCo;
    const int n = blockIdx.z / ngrp, co0 = (blockIdx.z % ngrp) * kCo;
    const float* xn = x + n * x_nstride;
    float acc[2][kCo];
#pragma unroll
    for (int o = 0; o < kCo; ++o) acc[0][o] = acc[1][o] = 0.f;
    for (int ci0 = 0; ci0 < cin; ci0 += kCi) {
        __syncthreads();
        for (int i = threadIdx.x; i < kCi * TY * TX; i += kThr) {
            const int c = i / (TY * TX), r = (i / TX) % TY, q = i % TX;
            const int gy = blockIdx.y * kTY + r - P, gx = blockIdx.x * kTX + q - P;
            float v = 0.f;
            if (ci0 + c < cin && gy >= 0 && gy < h && gx >= 0 && gx < w)
                v = xn[(int64_t)(ci0 + c) * h * w + (int64_t)gy * w + gx];
            sx[c][r][q] = v;
        }
        for (int i = threadIdx.x; i < kCi * K * K * kCo; i += kThr) {
            const int o = i % kCo, t = (i / kCo) % (K * K), c = i / (kCo * K * K);
            float v = 0.f;
            if (co0 + o < cout && ci0 + c < cin)
                v = wt[((int64_t)(co0 + o) * cin + ci0 + c) * K * K + t];
            sw[c][t][o] = v;
        }
        __syncthreads();
        const int cn = min(kCi, cin - ci0);
        for (int c = 0; c < cn; ++c) {
#pragma unroll
            for (int t = 0; t < K * K; ++t) {
                const float v0 = sx[c][ty + t / K][tx + t % K];
                const float v1 = sx[c][ty + t / K][tx + 16 + t % K];
                const float4* wq = reinterpret_cast<const float4*>(sw[c][t]);
#pragma unroll
                for (int q = 0; q < kCo / 4; ++q) {
                    const float4 ww = wq[q];
                    acc[0][4 * q + 0] = fmaf(ww.x, v0, acc[0][4 * q + 0]);
                    acc[0][4 * q + 1] = fmaf(ww.y, v0, acc[0][4 * q + 1]);
                    acc[0][4 * q + 2] = fmaf(ww.z, v0, acc[0][4 * q + 2]);
                    acc[0][4 * q + 3] = fmaf(ww.w, v0, acc[0][4 * q + 3]);
                    acc[1][4 * q + 0] = fmaf(ww.x, v1, acc[1][4 * q + 0]);
                    acc[1][4 * q + 1] = fmaf(ww.y, v1, acc[1][4 * q + 1]);
                    acc[1][4 * q + 2] = fmaf(ww.z, v1, acc[1][4 * q + 2]);
                    acc[1][4 * q + 3] = fmaf(ww.w, v1, acc[1][4 * q + 3]);
                }
            }
        }
    }
    if (oy >= h) return;
    float* yn = y + n * y_nstride;
#pragma unroll
    for (int hx = 0; hx < 2; ++hx) {
        const int px = ox + 16 * hx;
        if (px >= w) continue;
#pragma unroll
        for (int o = 0; o < kCo; ++o) {
            if (co0 + o >= cout) break;
            float v = acc[hx][o] + bias[co0 + o];
            if (relu) v = fmaxf(v, 0.f);
            yn[(int64_t)(co0 + o) * h * w + (int64_t)oy * w + px] = v;
        }
    }
}

// space_to_depth (autodiff.py:290-308): out[4c + 2dy + dx][Y][X] = x[c][2Y+dy][2X+dx].
__global__ void s2d_kernel(const float* __restrict__ x, int c, int h, int w,
                           float* __restrict__ y, int n) {
    const int64_t total = (int64_t)n * c * h * w;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int xx = i % w, yy = (i / w) % h;
        const int64_t nc = i / ((int64_t)h * w);
        const int cc = nc % c, nn = nc / c;
        const int dy = yy & 1, dx = xx & 1;
        y[(((int64_t)nn * 4 * c + 4 * cc + 2 * dy + dx) * (h / 2) + yy / 2) * (w / 2) + xx / 2] = x[i];
    }
}

// avg_pool2 (autodiff.py:241-247).
__global__ void pool_kernel(const float* __restrict__ x, int planes, int h, int w,
                            float* __restrict__ y) {
    const int ho = h / 2, wo = w / 2;
    const int64_t total = (int64_t)planes * ho * wo;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int xo = i % wo, yo = (i / wo) % ho;
        const int64_t p = i / ((int64_t)ho * wo);
        const float* s = x + p * h * w + (int64_t)(2 * yo) * w + 2 * xo;
        y[i] = ((s[0] + s[1]) + (s[w] + s[w + 1])) * 0.25f;
    }
}

// _upsample_taps (autodiff.py:258-264): centres (i + 0.5)/2 - 0.5 clamped.
__device__ __forceinline__ void up_tap(int i, int n, int& i0, int& i1, float& wt) {
    double s = (i + 0.5) / 2.0 - 0.5;
    s = fmin(fmax(s, 0.0), n - 1.0);
    i0 = (int)floor(s);
    i1 = min(i0 + 1, n - 1);
    wt = (float)(s - i0);
}

// bilinear_upsample2 (autodiff.py:267-274), rows then columns, products and
// sums rounded separately like the numpy expression; + optional skip
// (network.py:191-192).
__device__ __forceinline__ float up2_at(const float* __restrict__ s, int h, int w, int oy, int ox) {
    int r0, r1, c0, c1;
    float rw, cw;
    up_tap(oy, h, r0, r1, rw);
    up_tap(ox, w, c0, c1, cw);
    const float rw0 = __fsub_rn(1.f, rw), cw0 = __fsub_rn(1.f, cw);
    const float a = __fadd_rn(__fmul_rn(s[r0 * w + c0], rw0), __fmul_rn(s[r1 * w + c0], rw));
    const float b = __fadd_rn(__fmul_rn(s[r0 * w + c1], rw0), __fmul_rn(s[r1 * w + c1], rw));
    return __fadd_rn(__fmul_rn(a, cw0), __fmul_rn(b, cw));
}

__global__ void up2_add_kernel(const float* __restrict__ x, int planes, int h, int w,
                               const float* __restrict__ skip, float* __restrict__ y) {
    const int ho = 2 * h, wo = 2 * w;
    const int64_t total = (int64_t)planes * ho * wo;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int xo = i % wo, yo = (i / wo) % ho;
        const int64_t p = i / ((int64_t)ho * wo);
        float v = up2_at(x + p * h * w, h, w, yo, xo);
        if (skip) v = __fadd_rn(v, skip[i]);
        y[i] = v;
    }
}

}  // namespace

// sigmoid (autodiff.py:200-203), the two-branch stable form.
__device__ __forceinline__ float stable_sigmoid(float v) {
    const float e = expf(-fabsf(v));
    return v >= 0.f ? 1.f / (1.f + e) : e / (1.f + e);
}

namespace {

// Head reconstruction (network.py:199-209): out = sigmoid(up2(y0) + d2s(y
// with channel 0 zeroed)); y is (4, h, w) half resolution.
__global__ void head_s2d_kernel(const float* __restrict__ yh, int h, int w, float* __restrict__ out,
                                int n, int64_t out_nstride) {
    const int ho = 2 * h, wo = 2 * w;
    const int64_t total = (int64_t)n * ho * wo;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int xo = i % wo, yo = (i / wo) % ho;
        const int nn = i / ((int64_t)ho * wo);
        const float* y = yh + (int64_t)nn * 4 * h * w;
        float v = up2_at(y, h, w, yo, xo);
        const int k = 2 * (yo & 1) + (xo & 1);
        if (k) v = __fadd_rn(v, y[(int64_t)k * h * w + (yo >> 1) * w + (xo >> 1)]);
        out[nn * out_nstride + (int64_t)yo * wo + xo] = stable_sigmoid(v);
    }
}

__global__ void sigmoid_kernel(const float* __restrict__ x, int64_t total, float* __restrict__ y) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x)
        y[i] = stable_sigmoid(x[i]);
}

int grid_for(int64_t total) {
    return (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
}

void conv_f32(const float* x, int n, int cin, int h, int w, const ConvW& c, int relu, float* y,
              cudaStream_t st) {
    dim3 grd((w + kTX - 1) / kTX, (h + kTY - 1) / kTY, n * ((c.cout + kCo - 1) / kCo));
    const int64_t xs = (int64_t)cin * h * w, ys = (int64_t)c.cout * h * w;
    if (c.k == 3)
        {
            NSM_PROF("conv_f32_kernel", st);
            conv_f32_kernel<3><<<grd, kThr, 0, st>>>(x, cin, h, w, c.w32, c.b32, c.cout, relu, y, xs, ys);
        }
    else
        {
            NSM_PROF("conv_f32_kernel", st);
            conv_f32_kernel<1><<<grd, kThr, 0, st>>>(x, cin, h, w, c.w32, c.b32, c.cout, relu, y, xs, ys);
        }
}

}  // namespace

size_t forward_f32_workspace(const Plan& p, int n, int h, int w) {
    // per level: skip (C_j, h_j, w_j) + two ping-pong buffers of the widest
    // channel count at the finest processed resolution + the s2d input
    const int s = p.cfg.use_space_to_depth ? 1 : 0;
    const int64_t hw0 = (int64_t)(h >> s) * (w >> s);
    int cmax = p.first_in;
    for (int j = 0; j < p.nlev; ++j) cmax = max(cmax, p.chans[j]);
    size_t bytes = 0;
    bytes += 2 * (size_t)n * cmax * hw0 * 4;                  // ping-pong
    for (int j = 0; j < p.nlev - 1; ++j)
        bytes += (size_t)n * p.chans[j] * (hw0 >> (2 * j)) * 4;  // skips
    bytes += (size_t)n * 4 * hw0 * 4;                            // head output
    return bytes + 1024;
}

nsm_status forward_f32(const Plan& p, const float* x, int n, int h, int w, float* out, void* ws,
                       size_t ws_bytes, cudaStream_t st) {
    if (ws_bytes < forward_f32_workspace(p, n, h, w))
        return fail(NSM_ERR_ARG, "workspace too small (%zu < %zu bytes)", ws_bytes,
                    forward_f32_workspace(p, n, h, w));
    const int s = p.cfg.use_space_to_depth ? 1 : 0;
    int hl = h >> s, wl = w >> s;
    const int64_t hw0 = (int64_t)hl * wl;
    int cmax = p.first_in;
    for (int j = 0; j < p.nlev; ++j) cmax = max(cmax, p.chans[j]);
    float* A = (float*)ws;
    float* B = A + (size_t)n * cmax * hw0;
    float* skips[kMaxLevels];
    float* cur = B + (size_t)n * cmax * hw0;
    for (int j = 0; j < p.nlev - 1; ++j) {
        skips[j] = cur;
        cur += (size_t)n * p.chans[j] * (hw0 >> (2 * j));
    }
    float* head = cur;

    // NCHW batched convs: each kernel handles n frames through blockIdx.z.
    const float* in = x;
    int cin = p.cfg.in_channels;
    if (s) {
        const int64_t tot = (int64_t)n * cin * h * w;
        {
            NSM_PROF("s2d_kernel", st);
            s2d_kernel<<<grid_for(tot), 256, 0, st>>>(x, cin, h, w, A, n);
        }
        in = A;
        cin *= 4;
    }
    float* tmp = (in == A) ? B : A;
    for (int j = 0; j < p.nlev - 1; ++j) {
        const Level& L = p.lev[j];
        conv_f32(in, n, cin, hl, wl, L.enc3, 1, tmp, st);
        conv_f32(tmp, n, L.enc3.cout, hl, wl, L.enc1, 1, skips[j], st);
        cin = L.enc1.cout;
        float* dst = (tmp == A) ? B : A;
        {
            NSM_PROF("pool_kernel", st);
            pool_kernel<<<grid_for((int64_t)n * cin * hl * wl / 4), 256, 0, st>>>(skips[j], n * cin, hl, wl, dst);
        }
        hl /= 2;
        wl /= 2;
        in = dst;
        tmp = (dst == A) ? B : A;
    }
    {
        const Level& L = p.lev[p.nlev - 1];
        conv_f32(in, n, cin, hl, wl, L.enc3, 1, tmp, st);
        float* dst = (tmp == A) ? B : A;
        conv_f32(tmp, n, L.enc3.cout, hl, wl, L.enc1, 1, dst, st);
        cin = L.enc1.cout;
        in = dst;
        tmp = (dst == A) ? B : A;
    }
    for (int j = p.nlev - 2; j >= 0; --j) {
        const Level& L = p.lev[j];
        {
            NSM_PROF("up2_add_kernel", st);
            up2_add_kernel<<<grid_for((int64_t)n * cin * hl * wl * 4), 256, 0, st>>>(
                in, n * cin, hl, wl, j > 0 ? skips[j] : nullptr, tmp);
        }
        hl *= 2;
        wl *= 2;
        float* dst = (tmp == A) ? B : A;
        conv_f32(tmp, n, cin, hl, wl, L.dec3, 1, dst, st);
        conv_f32(dst, n, L.dec3.cout, hl, wl, L.dec1, 1, tmp, st);
        cin = L.dec1.cout;
        in = tmp;
        tmp = dst;
    }
    conv_f32(in, n, cin, hl, wl, p.head, 0, head, st);
    if (s) {
        {
            NSM_PROF("head_s2d_kernel", st);
            head_s2d_kernel<<<grid_for((int64_t)n * hl * wl * 4), 256, 0, st>>>(head, hl, wl, out, n,
                                                                                 (int64_t)h * w);
        }
    } else {
        {
            NSM_PROF("sigmoid_kernel", st);
            sigmoid_kernel<<<grid_for((int64_t)n * h * w), 256, 0, st>>>(head, (int64_t)n * h * w, out);
        }
    }
    NSM_CUDA_TRY(cudaGetLastError());
    return NSM_OK;
}

}  // namespace nsm
