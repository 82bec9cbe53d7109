// umma_rate_bench.cu -- developer microbenchmark: aggregate tcgen05.mma throughput per SM
// with W concurrent issuing warps (each with its own accumulator), for N in {16,32,64,128,256},
// A from TMEM (TS) or shared memory (SS).  kind::f16, M = 128, K = 16, dependent chain of
// `nmma` MMAs per warp (accumulate), then commit + wait.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_rate_bench umma_rate_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                 ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
                 ::"r"(smem_u32(b)), "r"(phase) : "memory");
}

template <bool TS>
__global__ void bench(long long* out, int reps, int nmma, int N, int nwarps) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* A = sm;                 // 128 x 16 bf16 = 4 KB
    uint8_t* B = sm + 4096;          // up to 256 x 16 bf16 = 8 KB
    __shared__ uint64_t bar[16];
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 12288; i += blockDim.x) sm[i] = 0;
    if (tid < 16) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[tid])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
    // accumulators: warp w uses columns [w*N, w*N+N) when it fits, A (TS) lives at column 448
    // accumulator columns must stay inside [0, 448): warps share columns when they do not fit
    // (the results are garbage but the timing is what we measure)
    const uint32_t d = tbase + (uint32_t)(N <= 448 / 14 ? warp * N : (warp * N) % (448 - N + 1));
    const uint32_t a_t = tbase + 448;
    const uint64_t a_s = sdesc(smem_u32(A), 128, 256);
    const uint64_t b_s = sdesc(smem_u32(B), 128, 256);
    uint32_t phase = 0;
    __syncthreads();
    const long long t0 = clock64();
    if (warp < nwarps && (tid & 31) == 0) {
        for (int r = 0; r < reps; ++r) {
            for (int k = 0; k < nmma; ++k) {
                if (TS) umma_ts(d, a_t, b_s, idesc, k > 0);
                else umma_ss(d, a_s, b_s, idesc, k > 0);
            }
            commit(&bar[warp]);
            mbar_wait(&bar[warp], phase);
            phase ^= 1;
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    if (tid == 0) out[0] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

int main() {
    long long* d_out;
    cudaMalloc(&d_out, 64);
    long long h;
    const int reps = 50, nmma = 8;
    cudaFuncSetAttribute(bench<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
    cudaFuncSetAttribute(bench<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
    for (int ts = 1; ts >= 0; --ts)
        for (int N : {16, 32, 64, 128, 256})
            for (int w : {1, 2, 4, 8, 14}) {
                if (ts) bench<true><<<1, 512, 16384>>>(d_out, reps, nmma, N, w);
                else bench<false><<<1, 512, 16384>>>(d_out, reps, nmma, N, w);
                cudaError_t e = cudaDeviceSynchronize();
                cudaMemcpy(&h, d_out, 8, cudaMemcpyDeviceToHost);
                const double per = (double)h / (reps * nmma * w);
                printf("%s N=%3d warps=%2d: %6.1f cyc per MMA (aggregate), %6.0f MAC/cyc  [%s]\n", ts ? "TS" : "SS", N, w,
                       per, 128.0 * N * 16 / per, cudaGetErrorString(e));
            }
    return 0;
}
