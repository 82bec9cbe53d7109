// umma_issue_bench.cu -- developer microbenchmark: cost of issuing tcgen05.mma (kind::f16,
// M=128, N=32, K=16, A from TMEM) from one thread, with operands in per-thread registers
// (R2UR per MMA) vs. warp-uniform values, and the cost of commit + mbarrier wait.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_issue_bench umma_issue_bench.cu
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
__device__ __forceinline__ void commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
                 ::"r"(smem_u32(b)), "r"(phase) : "memory");
}

template <int MODE>
__global__ void bench(long long* out, int reps, int nmma, int pad, int nacc) {
    __shared__ __align__(1024) uint8_t B[8192];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x;
    for (int i = tid; i < 8192; i += blockDim.x) B[i] = 0;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
    uint32_t phase = 0;
    long long t_issue = 0, t_commit = 0, t_wait = 0;
    // MODE 0: addresses derived from tid (non-uniform registers); MODE 1: from blockIdx/pad (uniform)
    const uint32_t d = MODE == 0 ? tbase + (uint32_t)(tid & 0) : tbase;
    const uint32_t a = d + 256 + (MODE == 0 ? (uint32_t)(tid >> 7) * 40 : (uint32_t)pad);
    if (tid == 0) {
        for (int r = 0; r < reps; ++r) {
            const long long c0 = clock64();
            for (int k = 0; k < nmma; ++k)
                umma_ts(d + 32 * (k % nacc), a + 8 * (k & 3), sdesc(smem_u32(B) + 256 * (k & 1), 128, 768), idesc,
                        k >= nacc);
            const long long c1 = clock64();
            commit(&bar);
            const long long c2 = clock64();
            mbar_wait(&bar, phase);
            phase ^= 1;
            const long long c3 = clock64();
            t_issue += c1 - c0; t_commit += c2 - c1; t_wait += c3 - c2;
        }
        out[0] = t_issue / reps; out[1] = t_commit / reps; out[2] = t_wait / reps;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

int main() {
    long long* d_out;
    cudaMalloc(&d_out, 64);
    long long h[3];
    for (int nacc : {1, 2, 5})
        for (int nm : {5, 20}) {
            bench<1><<<1, 128>>>(d_out, 200, nm, 32, nacc);
            cudaError_t e = cudaDeviceSynchronize();
            cudaMemcpy(h, d_out, sizeof h, cudaMemcpyDeviceToHost);
            printf("uniform nacc %d nmma %2d: issue %lld cyc (%.1f/mma) commit %lld wait %lld total %lld [%s]\n",
                   nacc, nm, h[0], (double)h[0] / nm, h[1], h[2], h[0] + h[1] + h[2], cudaGetErrorString(e));
        }
    return 0;
}
