// Throughput of tcgen05.mma kind::f16 (M=128, K=16, SS) against the A-operand
// layout of the implicit-GEMM convolutions: 16 core matrices (8 rows x 16 B)
// spaced SBO bytes apart, starting `shift` bytes past a 1024-B boundary.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_layout_probe tools/umma_layout_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

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

__device__ int g_sink;

template <int N>
__global__ void __launch_bounds__(256, 1) k(long long* cyc, int iters, int sbo, int shift, int lbo, int ntaps, int noise) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tb;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tb)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (noise == 3) {   // fill the operands with pseudo-random fp16 values (not zeros)
        for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) {
            uint32_t h = i * 2654435761u;
            h ^= h >> 13;
            const float f0 = ((h & 0xffff) / 65536.f - 0.5f), f1 = (((h >> 16) & 0xffff) / 65536.f - 0.5f);
            __half2 v = __floats2half2_rn(f0, f1);
            reinterpret_cast<uint32_t*>(sm)[i] = *reinterpret_cast<uint32_t*>(&v);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
    }
    const uint32_t base = smem_u32(sm);
    const uint32_t bb = base + 160 * 1024;
    const uint32_t idesc = make_idesc(128, N);
    if (threadIdx.x == 0) {
        long long t0 = clock64();
        const uint64_t da0 = make_desc(base + shift, lbo, sbo), db0 = make_desc(bb, N * 16, 128);
        if (ntaps == 0) {            // loop-invariant descriptors
            for (int i = 0; i < iters; ++i) mma_f16(tb, da0, db0, idesc, i > 0);
        } else if (ntaps == -2) {    // 9 taps x 4 accumulators (M-blocks), like the level kernels
#pragma unroll 1
            for (int i = 0; i < iters; i += 36) {
#pragma unroll 1
                for (int tap = 0; tap < 9; ++tap) {
                    const uint64_t dat = da0 + (uint64_t)(((tap / 3) * sbo + (tap % 3) * 16) >> 4);
#pragma unroll
                    for (int b = 0; b < 4; ++b)
                        mma_f16(tb + b * N, dat + b * 8, db0 + tap * 2, idesc, tap > 0);
                }
            }
        } else if (ntaps == -3) {    // fully unrolled 9 taps x 4 accumulators
#pragma unroll 1
            for (int i = 0; i < iters; i += 36) {
#pragma unroll
                for (int tap = 0; tap < 9; ++tap)
#pragma unroll
                    for (int b = 0; b < 4; ++b)
                        mma_f16(tb + b * N, da0 + (uint64_t)((((tap / 3) * sbo + (tap % 3) * 16) >> 4) + b * 8),
                                db0 + tap * 2, idesc, tap > 0);
            }
        } else if (ntaps == -4) {    // block-outer: 9 consecutive taps per accumulator
#pragma unroll 1
            for (int i = 0; i < iters; i += 36) {
#pragma unroll
                for (int b = 0; b < 4; ++b)
#pragma unroll
                    for (int tap = 0; tap < 9; ++tap)
                        mma_f16(tb + b * N, da0 + (uint64_t)((((tap / 3) * sbo + (tap % 3) * 16) >> 4) + b * 8),
                                db0 + tap * 2, idesc, tap > 0);
            }
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
        atomicExch(&g_sink, 1);
    }
    if (threadIdx.x >= 128 && (noise == 1 || noise == 2)) {   // contention: TMEM loads (1) or SMEM loads (2) until the MMA loop ends
        const int w = (threadIdx.x >> 5) & 3;
        uint32_t acc = 0;
        for (int it = 0; it < 200000 && !*(volatile int*)&g_sink; ++it) {
            if (noise == 1) {
                uint32_t r[16];
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                             : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                               "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                             : "r"(tb + ((uint32_t)(w * 32) << 16) + 256 + (it & 15) * 16));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                acc += r[0] ^ r[15];
            } else {
                const uint4 v = *reinterpret_cast<const uint4*>(sm + 100 * 1024 + ((threadIdx.x * 16 + it * 2048) & 32767));
                acc += v.x ^ v.w;
            }
        }
        if (acc == 0x12345) g_sink = 2;
    }
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
}

template <int N>
void run(int sbo, int shift, int lbo, int ntaps, int noise = 0) {
    long long* d;
    cudaMalloc(&d, 8 * 148);
    const int iters = 4096;
    cudaFuncSetAttribute(k<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    int z = 0;
    cudaMemcpyToSymbol(g_sink, &z, sizeof z);
    k<N><<<148, 256, 200 * 1024>>>(d, iters, sbo, shift, lbo, ntaps, noise);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("N=%3d sbo=%4d shift=%3d lbo=%6d taps=%d noise=%d: %.1f cycles/mma  err=%s\n", N, sbo, shift, lbo, ntaps, noise,
           (double)h / iters, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    for (int n : {32, 64}) {
        auto R = [&](int sbo, int shift, int lbo, int taps, int noise) {
            if (n == 32) run<32>(sbo, shift, lbo, taps, noise); else run<64>(sbo, shift, lbo, taps, noise);
        };
        R(544, 0, 9792, -2, 0);    // four accumulators, per-tap loop, zero operands
        R(544, 0, 9792, -2, 3);    // ... random operands
        R(544, 0, 9792, -3, 3);    // fully unrolled, random operands
    }
    return 0;
}
