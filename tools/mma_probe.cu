// Microbenchmarks that decide the conv engine design on B200 (sm_100a):
//   1. legacy mma.sync m16n8k16 f16->f32 throughput per SM
//   2. tcgen05.mma kind::f16 (A and B from SMEM, no swizzle, K-major)
//      throughput for M=128, N in {16,32,64,128,256}, and a correctness
//      check of the descriptor / TMEM layout including a 16-byte (one pixel)
//      shifted A start address -- the implicit-GEMM conv trick.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_probe mma_probe.cu
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cmath>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

// ---------------------------------------------------------------- mma.sync
__global__ void hmma_loop(float* out, int iters) {
    uint32_t a[4] = {0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u};
    uint32_t b[2] = {0x3c003c00u, 0x3c003c00u};
    float c[8][4] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                         : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                         : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
        }
    }
    float s = 0;
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
    if (s == 123.f) out[0] = s;
}

// ---------------------------------------------------------------- tcgen05
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// SWIZZLE_NONE K-major descriptor: start, LBO (K direction core-matrix
// stride), SBO (M/N direction core-matrix stride), version 1.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
    return (1u << 4)            // D = F32
         | (0u << 7)            // A = F16
         | (0u << 10)           // B = F16
         | ((uint32_t)(N >> 3) << 17)
         | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                        uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
                 :: "r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 :: "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, int cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(cnt));
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile("{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                 "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}\n"
                 :: "r"(smem_u32(bar)), "r"(phase) : "memory");
}

template <int N>
__global__ void __launch_bounds__(128, 1) umma_loop(long long* cycles, float* out, int iters,
                                                     int check, const __half* ga, const __half* gb) {
    // A: 128 x 16 (+ 8 rows slack for the shifted check), B: N x 16 -- chunk-planar
    // layout: chunk c (8 halves) of row r at c * PLANE + r * 16 bytes.
    constexpr int MA = 136;
    __shared__ __align__(1024) uint8_t sa[2 * MA * 16];
    __shared__ __align__(1024) uint8_t sb[2 * N * 16];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid / 32;
    // fill: A[r][k] = ga[r*16+k], B[n][k] = gb[n*16+k]
    for (int i = tid; i < MA * 16; i += 128) {
        int r = i / 16, k = i % 16;
        __half v = check ? ga[i] : __float2half(0.f);
        *(__half*)(sa + (k / 8) * MA * 16 + r * 16 + (k % 8) * 2) = v;
    }
    for (int i = tid; i < N * 16; i += 128) {
        int n = i / 16, k = i % 16;
        __half v = check ? gb[i] : __float2half(0.f);
        *(__half*)(sb + (k / 8) * N * 16 + n * 16 + (k % 8) * 2) = v;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        constexpr int cols = N < 32 ? 32 : N;
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"(smem_u32(&tbase)), "r"(cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tbase;
    const uint32_t idesc = make_idesc(128, N);
    const int shift = check == 2 ? 1 : 0;   // shifted A start: rows 1..128
    const uint64_t da = make_desc(smem_u32(sa) + shift * 16, MA * 16, 128);
    const uint64_t db = make_desc(smem_u32(sb), N * 16, 128);
    long long t0 = 0, t1 = 0;
    if (tid == 0) {
        t0 = clock64();
        for (int i = 0; i < iters; ++i) mma_f16(tmem, da, db, idesc, i > 0);
        commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    if (tid == 0) {
        t1 = clock64();
        cycles[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (check) {
        // each warp reads its 32 lanes, 16 columns at a time
        for (int c0 = 0; c0 < N; c0 += 16) {
            uint32_t r[16];
            const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                           "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                         : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            for (int j = 0; j < 16; ++j) out[(warp * 32 + (tid % 32)) * N + c0 + j] = __uint_as_float(r[j]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) {
        constexpr int cols = N < 32 ? 32 : N;
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(cols));
    }
}

template <int N>
void run_umma(int sms) {
    // correctness: D = A(128x16) * B(Nx16)^T, and shifted-A variant
    std::vector<__half> ha(136 * 16), hb(N * 16);
    std::vector<float> fa(136 * 16), fb(N * 16);
    srand(1);
    for (int i = 0; i < 136 * 16; ++i) { fa[i] = (rand() % 17 - 8) / 8.f; ha[i] = __float2half(fa[i]); }
    for (int i = 0; i < N * 16; ++i) { fb[i] = (rand() % 17 - 8) / 8.f; hb[i] = __float2half(fb[i]); }
    __half *ga, *gb; float* gout; long long* gcyc;
    CK(cudaMalloc(&ga, ha.size() * 2)); CK(cudaMalloc(&gb, hb.size() * 2));
    CK(cudaMalloc(&gout, 128 * N * 4)); CK(cudaMalloc(&gcyc, sms * 8));
    CK(cudaMemcpy(ga, ha.data(), ha.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(gb, hb.data(), hb.size() * 2, cudaMemcpyHostToDevice));
    for (int shift = 0; shift <= 1; ++shift) {
        umma_loop<N><<<1, 128>>>(gcyc, gout, 1, 1 + shift, ga, gb);
        CK(cudaDeviceSynchronize());
        std::vector<float> o(128 * N);
        CK(cudaMemcpy(o.data(), gout, o.size() * 4, cudaMemcpyDeviceToHost));
        double err = 0;
        for (int m = 0; m < 128; ++m)
            for (int n = 0; n < N; ++n) {
                double s = 0;
                for (int k = 0; k < 16; ++k) s += fa[(m + shift) * 16 + k] * fb[n * 16 + k];
                err = fmax(err, fabs(s - o[m * N + n]));
            }
        printf("umma N=%3d shift=%d correctness max err %.3g\n", N, shift, err);
    }
    const int iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    umma_loop<N><<<sms, 128>>>(gcyc, gout, iters, 0, ga, gb);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    umma_loop<N><<<sms, 128>>>(gcyc, gout, iters, 0, ga, gb);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    std::vector<long long> cyc(sms);
    CK(cudaMemcpy(cyc.data(), gcyc, sms * 8, cudaMemcpyDeviceToHost));
    double macs = 128.0 * N * 16 * iters * sms;
    printf("umma M=128 N=%3d K=16 SS: %.1f cycles/mma (SM 0), chip %.1f TFLOPS\n", N,
           (double)cyc[0] / iters, 2 * macs / (ms * 1e-3) / 1e12);
    cudaFree(ga); cudaFree(gb); cudaFree(gout); cudaFree(gcyc);
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* d; CK(cudaMalloc(&d, 4));
    for (int warps : {4, 8, 16}) {
        int iters = 4096;
        hmma_loop<<<sms, 32 * warps>>>(d, 16);
        CK(cudaDeviceSynchronize());
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        hmma_loop<<<sms, 32 * warps>>>(d, iters);
        cudaEventRecord(e1);
        CK(cudaDeviceSynchronize());
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double macs = 16.0 * 8 * 16 * 8 * iters * warps * sms;
        printf("mma.sync m16n8k16 f32acc: %d warps/SM -> %.1f TFLOPS\n", warps, 2 * macs / (ms * 1e-3) / 1e12);
    }
    run_umma<16>(sms);
    run_umma<32>(sms);
    run_umma<64>(sms);
    run_umma<128>(sms);
    run_umma<256>(sms);
    return 0;
}
