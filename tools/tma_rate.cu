// TMA throughput probe for the level-kernel input tiles: a 5-D box
// (8 elems, x, y, chunk, n) that writes chunk-planar tiles (16-B inner rows)
// vs a 4-D pixel-major box (C elems, x, y, n) of the same bytes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tma_rate tma_rate.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int RANK>
__global__ void rate(const __grid_constant__ CUtensorMap m, int bytes, int iters, int W, int H, long long* cyc) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar[2];
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar[0])), "r"(1));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar[1])), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        const int s = i & 1;
        if (i >= 2) {
            const uint32_t ph = ((i - 2) >> 1) & 1;
            asm volatile("{\n\t.reg .pred P1;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}\n"
                         :: "r"(su32(&bar[s])), "r"(ph) : "memory");
        }
        const int x = ((blockIdx.x * 7 + i * 13) % (W / 32)) * 32, y = ((blockIdx.x * 3 + i * 5) % (H / 16)) * 16;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(bytes) : "memory");
        const uint32_t dst = su32(smem + s * 65536);
        if (RANK == 5)
            asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                         :: "r"(dst), "l"(reinterpret_cast<uint64_t>(&m)), "r"(0), "r"(x - 1), "r"(y - 1), "r"(0), "r"(0), "r"(su32(&bar[s])) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                         :: "r"(dst), "l"(reinterpret_cast<uint64_t>(&m)), "r"(0), "r"(x - 1), "r"(y - 1), "r"(0), "r"(su32(&bar[s])) : "memory");
    }
    for (int s = 0; s < 2 && s < iters; ++s) {
        const int i = iters - 1 - ((iters - 1 - s) & 1 ? 1 : 0);
        (void)i;
    }
    // drain
    for (int i = iters - 2; i < iters; ++i) {
        if (i < 0) continue;
        const int s = i & 1;
        const uint32_t ph = (i >> 1) & 1;
        asm volatile("{\n\t.reg .pred P1;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}\n"
                     :: "r"(su32(&bar[s])), "r"(ph) : "memory");
    }
    cyc[blockIdx.x] = clock64() - t0;
}

int main() {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long* cyc; CK(cudaMalloc(&cyc, sms * 8));
    for (int C : {16, 32, 64}) {
        const int W = 480, H = 272, N = 1, BW = 34, BH = 18;
        __half* d; CK(cudaMalloc(&d, (size_t)W * H * C * 2 * N)); CK(cudaMemset(d, 0, (size_t)W * H * C * 2 * N));
        CUtensorMap m5, m4;
        const cuuint64_t dims5[5] = {8, W, H, (cuuint64_t)C / 8, N};
        const cuuint64_t str5[4] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, 16, (cuuint64_t)H * W * C * 2};
        const cuuint32_t box5[5] = {8, BW, BH, (cuuint32_t)C / 8, 1}, es[5] = {1, 1, 1, 1, 1};
        CUresult r = enc(&m5, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 5, d, dims5, str5, box5, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const cuuint64_t dims4[4] = {(cuuint64_t)C, W, H, N};
        const cuuint64_t str4[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
        const cuuint32_t box4[4] = {(cuuint32_t)C, BW, BH, 1};
        CUresult r4 = enc(&m4, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, d, dims4, str4, box4, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const int bytes = BW * BH * C * 2, iters = 200;
        CK(cudaFuncSetAttribute(rate<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000));
        CK(cudaFuncSetAttribute(rate<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000));
        for (int rank : {5, 4}) {
            if ((rank == 5 ? r : r4) != CUDA_SUCCESS) { printf("encode failed rank %d\n", rank); continue; }
            for (int rep = 0; rep < 2; ++rep) {
                if (rank == 5) rate<5><<<sms, 32, 140000>>>(m5, bytes, iters, W, H, cyc);
                else rate<4><<<sms, 32, 140000>>>(m4, bytes, iters, W, H, cyc);
                CK(cudaDeviceSynchronize());
            }
            std::vector<long long> c(sms);
            CK(cudaMemcpy(c.data(), cyc, sms * 8, cudaMemcpyDeviceToHost));
            double avg = 0; for (auto v : c) avg += v; avg /= sms;
            printf("C=%3d rank %d box %dx%dx%d: %.0f cycles/box (%.1f B/clk/SM), %d B\n", C, rank, BW, BH, C, avg / iters,
                   bytes / (avg / iters), bytes);
        }
        cudaFree(d);
    }
    return 0;
}
