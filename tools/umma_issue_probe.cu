// Is tcgen05.mma (kind::f16, M=128, K=16, SS) limited per issuing thread or
// per SM?  1, 2 or 4 warps (on different SM sub-partitions) each issue
// `iters` UMMAs into their own accumulator, loop-invariant descriptors; the
// time until all commits land gives the aggregate cycles per UMMA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/umma_issue_probe tools/umma_issue_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
    return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d), "l"(da), "l"(db),
                 "r"(idesc), "r"(acc));
}

template <int N>
__global__ void __launch_bounds__(128, 1) k(long long* cyc, int iters, int nwarps) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar[4];
    __shared__ uint32_t tb;
    __shared__ long long t0s;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tb)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0)
        for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u * (i & 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int w = threadIdx.x >> 5;
    if (threadIdx.x == 0) t0s = clock64();
    __syncthreads();
    if (w < nwarps && (threadIdx.x & 31) == 0) {
        const uint32_t base = smem_u32(sm);
        const uint64_t da = make_desc(base + w * 8192, 2880, 160), db = make_desc(base + 40960, N * 16, 128);
        const uint32_t idesc = make_idesc(128, N);
        for (int i = 0; i < iters; ++i) mma_f16(tb + w * 128, da, db, idesc, i > 0);
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[w])));
        asm volatile("{\n\t.reg .pred P;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra W;\n\t}" ::"r"(smem_u32(&bar[w])));
    }
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0s;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
}

template <int N>
void run(int nwarps) {
    long long* d;
    cudaMalloc(&d, 8 * 148);
    const int iters = 4096;
    cudaFuncSetAttribute(k<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    k<N><<<148, 128, 64 * 1024>>>(d, iters, nwarps);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("N=%3d issuers=%d: %.1f cycles per UMMA (aggregate), %.1f per issuer  err=%s\n", N, nwarps,
           (double)h / (iters * nwarps), (double)h / iters, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    for (int nw : {1, 2, 4}) {
        run<32>(nw);
        run<64>(nw);
        run<128>(nw);
    }
    return 0;
}
