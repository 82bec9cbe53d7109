// mufu_rate_bench.cu -- measured MUFU (XU pipe) throughput on this GPU: tanh.approx.f32
// and ex2.approx.f32 issued back to back from every SM, 8 independent
// chains per thread so the rate, not the latency, is measured.  This is the peak the
// eval_map roofline divides by.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mufu tools/mufu_rate_bench.cu && /tmp/mufu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void __launch_bounds__(1024) mufu_loop(float* out, int iters, float seed) {
    float x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = seed + 1e-3f * (threadIdx.x + 7 * k);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            float y;
            if (OP == 0) asm volatile("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x[k]));
            else asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[k]));
            x[k] = y;
        }
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.f) out[threadIdx.x] = s;
}

template <int OP>
double rate(int sms, int clk_khz) {
    float* out;
    cudaMalloc(&out, 4096);
    const int iters = 4096, threads = 1024, blocks = sms * 2;
    mufu_loop<OP><<<blocks, threads>>>(out, 16, 0.1f);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    mufu_loop<OP><<<blocks, threads>>>(out, iters, 0.1f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaFree(out);
    const double ops = (double)blocks * threads * iters * 8;
    return ops / (ms * 1e-3) / 1e9;   // G ops/s
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const double t = rate<0>(sms, clk), e = rate<1>(sms, clk);
    const double per_clk = 1e9 / (sms * (double)clk * 1e3);
    std::printf("{\"sms\": %d, \"max_clock_mhz\": %.0f, \"tanh_G_per_s\": %.1f, \"ex2_G_per_s\": %.1f, "
                "\"tanh_per_clk_per_sm_at_max_clock\": %.2f}\n",
                sms, clk / 1e3, t, e, t * per_clk);
    return 0;
}
