// TMA probe: 3D / 4D fp32 tensor-map tile loads with negative (out-of-bounds)
// start coordinates into a 128-B aligned SMEM stage, checked against the
// host.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tma_probe tma_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe2d(const __grid_constant__ CUtensorMap m2, float* out, int x, int y, int bytes) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     :: "r"(su32(smem)), "l"(reinterpret_cast<uint64_t>(&m2)), "r"(x), "r"(y), "r"(su32(&bar)) : "memory");
    }
    asm volatile("{\n\t.reg .pred P1;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}\n"
                 :: "r"(su32(&bar)), "r"(0) : "memory");
    for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x) out[i] = reinterpret_cast<float*>(smem)[i];
}

template <int MODE>
__global__ void probe(const __grid_constant__ CUtensorMap m3, const __grid_constant__ CUtensorMap m4, float* out,
                      int x, int y, int z) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar;
    constexpr int BOX = 132 * 18;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t bytes = MODE == 0 ? BOX * 4 : BOX * 4 * 3;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(bytes) : "memory");
        if (MODE == 0)
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         :: "r"(su32(smem)), "l"(reinterpret_cast<uint64_t>(&m3)), "r"(x), "r"(y), "r"(z), "r"(su32(&bar)) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                         :: "r"(su32(smem)), "l"(reinterpret_cast<uint64_t>(&m4)), "r"(x), "r"(y), "r"(0), "r"(z), "r"(su32(&bar)) : "memory");
    }
    asm volatile("{\n\t.reg .pred P1;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}\n"
                 :: "r"(su32(&bar)), "r"(0) : "memory");
    const int n = MODE == 0 ? BOX : 3 * BOX;
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = reinterpret_cast<float*>(smem)[i];
}

int main(int argc, char** argv) {
    const int sel = argc > 1 ? atoi(argv[1]) : -1;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
    const int W = 256, H = 256, N = 2;
    std::vector<float> h3(W * H * N), h4(W * H * 3 * N);
    for (size_t i = 0; i < h3.size(); ++i) h3[i] = (float)i;
    for (size_t i = 0; i < h4.size(); ++i) h4[i] = (float)i;
    float *d3, *d4, *out;
    CK(cudaMalloc(&d3, h3.size() * 4)); CK(cudaMalloc(&d4, h4.size() * 4)); CK(cudaMalloc(&out, 3 * 132 * 18 * 4));
    CK(cudaMemcpy(d3, h3.data(), h3.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d4, h4.data(), h4.size() * 4, cudaMemcpyHostToDevice));
    CUtensorMap m3, m4;
    const cuuint64_t dim3_[3] = {W, H, N}, str3[2] = {W * 4, (cuuint64_t)W * H * 4};
    const cuuint64_t dim4[4] = {W, H, 3, N}, str4[3] = {W * 4, (cuuint64_t)W * H * 4, (cuuint64_t)W * H * 12};
    const cuuint32_t box3[3] = {132, 18, 1}, box4[4] = {132, 18, 3, 1}, es[4] = {1, 1, 1, 1};
    CUresult r = enc(&m3, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d3, dim3_, str3, box3, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode 3d: %d\n", (int)r);
    r = enc(&m4, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d4, dim4, str4, box4, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode 4d: %d\n", (int)r);
    if (sel >= 10) {
        // 2D modes: 10 = box 32x8 at (0,0); 11 = box 132x18 at (0,0); 12 = 132x18 at (-2,240); 13 = box 128x16 at (-2, 240)
        const cuuint32_t bw = sel == 10 ? 32 : sel == 13 ? 128 : sel == 14 ? 136 : 132, bh = sel == 10 ? 8 : sel == 13 ? 16 : 18;
        const int x = sel == 14 ? -4 : sel == 15 ? 4 : sel >= 12 ? -2 : 0, y = sel >= 12 ? 240 : 0;
        CUtensorMap m2;
        const cuuint64_t dim2[2] = {W, (cuuint64_t)H * N}, str2[1] = {W * 4};
        const cuuint32_t box2[2] = {bw, bh};
        r = enc(&m2, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d3, dim2, str2, box2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("encode 2d: %d\n", (int)r);
        CK(cudaFuncSetAttribute(probe2d, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000));
        probe2d<<<1, 128, 40000>>>(m2, out, x, y, bw * bh * 4);
        CK(cudaDeviceSynchronize());
        std::vector<float> o(bw * bh);
        CK(cudaMemcpy(o.data(), out, o.size() * 4, cudaMemcpyDeviceToHost));
        int bad = 0;
        for (int r2 = 0; r2 < (int)bh; ++r2)
            for (int cc = 0; cc < (int)bw; ++cc) {
                const int gx = x + cc, gy = y + r2;
                const float want = (gx >= 0 && gx < W && gy >= 0 && gy < H * N) ? h3[(size_t)gy * W + gx] : 0.f;
                if (o[r2 * bw + cc] != want) ++bad;
            }
        printf("2d mode %d: %d mismatches\n", sel, bad);
        return 0;
    }
    CK(cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000));
    CK(cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000));
    for (int mode = 0; mode < 2; ++mode) {
        const int x = -2, y = 240, z = 1;
        if (mode == 0) probe<0><<<1, 128, 40000>>>(m3, m4, out, x, y, z);
        else probe<1><<<1, 128, 40000>>>(m3, m4, out, x, y, z);
        CK(cudaDeviceSynchronize());
        std::vector<float> o(3 * 132 * 18);
        CK(cudaMemcpy(o.data(), out, o.size() * 4, cudaMemcpyDeviceToHost));
        int bad = 0;
        for (int c = 0; c < (mode ? 3 : 1); ++c)
            for (int r2 = 0; r2 < 18; ++r2)
                for (int cc = 0; cc < 132; ++cc) {
                    const int gx = x + cc, gy = y + r2;
                    float want = 0.f;
                    if (gx >= 0 && gx < W && gy >= 0 && gy < H)
                        want = mode == 0 ? h3[((size_t)z * H + gy) * W + gx] : h4[(((size_t)z * 3 + c) * H + gy) * W + gx];
                    if (o[(c * 18 + r2) * 132 + cc] != want) ++bad;
                }
        printf("mode %dd: %d mismatches\n", mode ? 4 : 3, bad);
    }
    return 0;
}
