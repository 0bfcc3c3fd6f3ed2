// Throughput of tcgen05.mma kind::f16 (M=128, K=16, SS) against the A-operand
// layout of the implicit-GEMM convolutions: 16 core matrices (8 rows x 16 B)
// spaced SBO bytes apart, starting `shift` bytes past a 1024-B boundary.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_layout_probe tools/umma_layout_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
    return (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d), "l"(da), "l"(db),
                 "r"(idesc), "r"(acc));
}

template <int N>
__global__ void __launch_bounds__(128, 1) k(long long* cyc, int iters, int sbo, int shift, int lbo, int ntaps) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tb;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tb)), "r"(N < 32 ? 32 : N));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = smem_u32(sm);
    const uint32_t bb = base + 160 * 1024;
    const uint32_t idesc = make_idesc(128, N);
    if (threadIdx.x == 0) {
        long long t0 = clock64();
        const uint64_t da0 = make_desc(base + shift, lbo, sbo), db0 = make_desc(bb, N * 16, 128);
        if (ntaps == 0) {            // loop-invariant descriptors
            for (int i = 0; i < iters; ++i) mma_f16(tb, da0, db0, idesc, i > 0);
        } else if (ntaps < 0) {      // 9 taps, descriptor = base + precomputed 16-B-unit offsets
#pragma unroll 1
            for (int i = 0; i < iters; i += 9) {
#pragma unroll
                for (int tap = 0; tap < 9; ++tap)
                    mma_f16(tb, da0 + (uint64_t)(((tap / 3) * sbo + (tap % 3) * 16) >> 4), db0 + tap * 2, idesc, 1);
            }
        } else {
            for (int i = 0; i < iters; ++i) {
                const int tap = i % ntaps;
                const uint32_t a = base + shift + (tap / 3) * sbo + (tap % 3) * 16;
                mma_f16(tb, make_desc(a, lbo, sbo), make_desc(bb, N * 16, 128), idesc, i > 0);
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
        asm volatile("{\n\t.reg .pred P;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra W;\n\t}" ::"r"(smem_u32(&bar)));
        cyc[blockIdx.x] = clock64() - t0;
    }
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(N < 32 ? 32 : N));
}

template <int N>
void run(int sbo, int shift, int lbo, int ntaps) {
    long long* d;
    cudaMalloc(&d, 8 * 148);
    const int iters = 4096;
    cudaFuncSetAttribute(k<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    k<N><<<148, 128, 200 * 1024>>>(d, iters, sbo, shift, lbo, ntaps);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("N=%3d sbo=%4d shift=%3d lbo=%6d taps=%d: %.1f cycles/mma  err=%s\n", N, sbo, shift, lbo, ntaps,
           (double)h / iters, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    for (int n : {32, 64}) {
        auto R = [&](int sbo, int shift, int lbo, int taps) { if (n == 32) run<32>(sbo, shift, lbo, taps); else run<64>(sbo, shift, lbo, taps); };
        R(128, 0, 2048, 0);      // loop-invariant descriptors
        R(544, 0, 16384, 0);
        R(544, 16, 16384, 0);
        R(544, 0, 16384, -1);    // 9 taps, unrolled, descriptor + offset
        R(128, 0, 2048, 1);      // contiguous core matrices (the probe's layout)
        R(512, 0, 16384, 1);     // 128-B aligned rows, pitch 512
        R(544, 0, 16384, 1);     // pitch 544 (34 px), aligned start
        R(544, 16, 16384, 1);    // one pixel shifted
        R(544, 0, 16384, 9);     // 9 taps (dy, dx) like the conv
        R(512, 0, 16384, 9);
        R(1024, 0, 16384, 9);
        R(576, 0, 16384, 9);
    }
    return 0;
}
