// TMA cost of a level-kernel input tile (18 x 34 pixels x 16 channels, fp16)
// loaded as 16-B box rows (pixel-major NHWC through a 5-D chunk view: 1224
// rows) against 512-B box rows (chunk-planar tensor, 32 px: 36 rows).  Each CTA
// streams `iters` tiles through 4 stages; cycles per tile at grid = 148.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_rows_probe tools/tma_rows_probe.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(32, 1) k(const __grid_constant__ CUtensorMap m, int mode, int iters, int W, int H,
                                           long long* cyc) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ uint64_t bar[4];
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    if (threadIdx.x != 0) return;
    const int tiles_x = W / 32, tiles_y = H / 16;
    const long long t0 = clock64();
    for (int i = 0; i < iters + 4; ++i) {
        if (i >= 4) {   // wait for tile i - 4
            const int s = (i - 4) & 3;
            const uint32_t par = ((i - 4) >> 2) & 1;
            asm volatile("{\n\t.reg .pred P;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W;\n\t}" ::"r"(smem_u32(&bar[s])), "r"(par));
        }
        if (i < iters) {
            const int s = i & 3;
            const int t = blockIdx.x + i * gridDim.x;
            const int x0 = (t % tiles_x) * 32 - 1, y0 = ((t / tiles_x) % tiles_y) * 16 - 1, f = (t / (tiles_x * tiles_y)) & 7;
            const uint32_t dst = smem_u32(sm + s * 20480), b = smem_u32(&bar[s]);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(mode ? 18 * 32 * 32 : 18 * 34 * 32));
            if (mode == 0)
                asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                             ::"r"(dst), "l"(&m), "r"(0), "r"(x0), "r"(y0), "r"(0), "r"(f), "r"(b) : "memory");
            else
                asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                             ::"r"(dst), "l"(&m), "r"(8 * (x0 + 1)), "r"(y0 + 1), "r"(2 * f), "r"(b) : "memory");
        }
    }
    cyc[blockIdx.x] = clock64() - t0;
}

int main() {
    const int W = 480, H = 272, N = 8, C = 16;
    void* buf;
    cudaMalloc(&buf, (size_t)N * (H + 2) * (W + 2) * C * 2);
    cudaMemset(buf, 0, (size_t)N * (H + 2) * (W + 2) * C * 2);
    long long* d;
    cudaMalloc(&d, 8 * 148);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    for (int mode = 0; mode < 2; ++mode) {
        CUtensorMap m;
        if (mode == 0) {   // NHWC through the 5-D chunk view (encode_nhwc_map)
            const cuuint64_t dims[5] = {8, (cuuint64_t)W, (cuuint64_t)H, 2, (cuuint64_t)N};
            const cuuint64_t str[4] = {32, (cuuint64_t)W * 32, 16, (cuuint64_t)H * W * 32};
            const cuuint32_t box[5] = {8, 34, 18, 2, 1}, es[5] = {1, 1, 1, 1, 1};
            enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 5, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {           // chunk-planar (N, 2, H + 2, W + 2, 8), padded
            const cuuint64_t dims[3] = {(cuuint64_t)(W + 2) * 8, (cuuint64_t)H + 2, 2 * N};
            const cuuint64_t str[2] = {(cuuint64_t)(W + 2) * 16, (cuuint64_t)(H + 2) * (W + 2) * 16};
            const cuuint32_t box[3] = {32 * 8, 18, 2}, es[3] = {1, 1, 1};   // boxDim <= 256
            enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 20480);
        const int iters = 64;
        for (int rep = 0; rep < 2; ++rep) k<<<148, 32, 4 * 20480>>>(m, mode, iters, W, H, d);
        cudaDeviceSynchronize();
        long long h[148];
        cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (long long v : h) mx = v > mx ? v : mx;
        printf("%s: %.0f cycles per tile (max CTA), %s\n", mode ? "chunk-planar 512-B rows" : "NHWC 16-B rows",
               (double)mx / iters, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
