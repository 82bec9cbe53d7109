// pipe_mix_bench.cu -- which execution pipe do eval_map's epilogue instructions use?
// Throughput of MUFU.TANH, F2FP.BF16.F32.PACK_AB (cvt.rn.bf16x2.f32), FHFMA.BF16 (mixed
// fma.rn.f32.bf16), IMAD.U32 / LOP3 (bf16 -> f32 unpacking) alone and mixed 1:1 with tanh:
// if a mix takes the SUM of the two alone-times the instructions share a pipe, if it takes
// the MAX they issue to different pipes.  8 independent chains per thread, 2 blocks of 1024
// threads per SM.  Also the scalar half-precision tanh (tanh.approx.f16x2 / .bf16x2 compile to
// two of these per pair on sm_100a).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipemix tools/pipe_mix_bench.cu && /tmp/pipemix
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ float op_tanh(float x) { float y; asm volatile("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float op_cvt(float x) {
    uint32_t d; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %1;" : "=r"(d) : "f"(x)); return __uint_as_float(d);
}
__device__ __forceinline__ float op_fhfma(float x) {
    float y;
    asm volatile("{.reg .b16 l, h, m; mov.b32 {l, h}, %1; mov.b16 m, 0xBF80; fma.rn.f32.bf16 %0, h, m, %1;}" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float op_tanh_f16(float x) {   // MUFU.TANH.F16 on the low half
    uint32_t u = __float_as_uint(x);
    asm volatile("{.reg .b16 l, h; mov.b32 {l, h}, %0; tanh.approx.f16 l, l; mov.b32 %0, {l, h};}" : "+r"(u));
    return __uint_as_float(u);
}
__device__ __forceinline__ float op_tanh_bf16(float x) {  // MUFU.TANH.BF16 on the low half
    uint32_t u = __float_as_uint(x);
    asm volatile("{.reg .b16 l, h; mov.b32 {l, h}, %0; tanh.approx.bf16 l, l; mov.b32 %0, {l, h};}" : "+r"(u));
    return __uint_as_float(u);
}
__device__ __forceinline__ float op_shl(float x) { uint32_t u; asm volatile("shl.b32 %0, %1, 16;" : "=r"(u) : "r"(__float_as_uint(x))); return __uint_as_float(u); }

template <int A, int B>   // A, B: 0 tanh, 1 cvt, 2 fhfma, 3 shl, 4 tanh f16, 5 tanh bf16, -1 none
__device__ __forceinline__ float apply(int which, float x) {
    const int k = which == 0 ? A : B;
    if (k == 0) return op_tanh(x);
    if (k == 1) return op_cvt(x);
    if (k == 2) return op_fhfma(x);
    if (k == 3) return op_shl(x);
    if (k == 4) return op_tanh_f16(x);
    if (k == 5) return op_tanh_bf16(x);
    return x;
}

template <int A, int B>
__global__ void __launch_bounds__(1024) loop(float* out, int iters, float seed) {
    float x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = seed + 1e-3f * (threadIdx.x + 7 * k);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            x[k] = apply<A, B>(0, x[k]);
            if (B >= 0) x[k] = apply<A, B>(1, x[k]);
        }
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.f) out[threadIdx.x] = s;
}

template <int A, int B>
double time_ms(int sms) {
    float* out;
    cudaMalloc(&out, 4096);
    const int iters = 2048, threads = 1024, blocks = sms * 2;
    loop<A, B><<<blocks, threads>>>(out, 16, 0.1f);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(a);
        loop<A, B><<<blocks, threads>>>(out, iters, 0.1f);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    cudaFree(out);
    return best;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    const double ops = (double)sms * 2 * 1024 * 2048 * 8;   // per instruction kind
    const double per = 1.0 / (sms * (double)clk * 1e3);     // seconds per SM-clock
    auto rate = [&](double ms) { return ops / (ms * 1e-3) * per; };   // lanes / clk / SM
    const double t_tanh = time_ms<0, -1>(sms), t_cvt = time_ms<1, -1>(sms), t_fh = time_ms<2, -1>(sms),
                 t_shl = time_ms<3, -1>(sms);
    const double m_cvt = time_ms<0, 1>(sms), m_fh = time_ms<0, 2>(sms), m_shl = time_ms<0, 3>(sms);
    const double t_th = time_ms<4, -1>(sms), t_tb = time_ms<5, -1>(sms), m_th = time_ms<0, 4>(sms);
    std::printf("{\"sms\": %d, \"clock_mhz\": %.0f, \"lanes_per_clk_per_sm\": {\"tanh\": %.2f, \"cvt_bf16x2\": %.2f, "
                "\"fhfma_bf16\": %.2f, \"shl\": %.2f, \"tanh_f16\": %.2f, \"tanh_bf16\": %.2f}, \"tanh+tanh_f16_ms\": %.3f, \"ms\": {\"tanh\": %.3f, \"cvt\": %.3f, \"fhfma\": %.3f, "
                "\"shl\": %.3f, \"tanh+cvt\": %.3f, \"tanh+fhfma\": %.3f, \"tanh+shl\": %.3f}}\n",
                sms, clk / 1e3, rate(t_tanh), rate(t_cvt), rate(t_fh), rate(t_shl), rate(t_th), rate(t_tb), m_th, t_tanh, t_cvt, t_fh, t_shl, m_cvt,
                m_fh, m_shl);
    return 0;
}
