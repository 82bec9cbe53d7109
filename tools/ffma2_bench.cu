// Throughput of scalar FFMA vs packed FFMA2 (fma.rn.f32x2) on one B200 SM-wide launch.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ffma2 tools/ffma2_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kChains = 8;

__global__ void scalar_fma(float* out, float a, float b) {
  float x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = fmaf(x[c], a, b);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void packed_fma(float* out, float a, float b) {
  float2 x[kChains / 2];
  const float2 A = make_float2(a, a), B = make_float2(b, b);
#pragma unroll
  for (int c = 0; c < kChains / 2; ++c) x[c] = make_float2(threadIdx.x * 1e-3f + 2 * c, 2 * c + 1);
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains / 2; ++c) x[c] = __ffma2_rn(x[c], A, B);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < kChains / 2; ++c) s += x[c].x + x[c].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// mixed: packed FMA interleaved with independent scalar integer/ALU work (dual issue?)
__global__ void packed_fma_plus_alu(float* out, float a, float b) {
  float2 x[kChains / 2];
  unsigned u[kChains / 2];
  const float2 A = make_float2(a, a), B = make_float2(b, b);
#pragma unroll
  for (int c = 0; c < kChains / 2; ++c) { x[c] = make_float2(threadIdx.x * 1e-3f + 2 * c, 2 * c + 1); u[c] = threadIdx.x + c; }
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains / 2; ++c) { x[c] = __ffma2_rn(x[c], A, B); u[c] = (u[c] ^ (u[c] >> 3)) + 7u; }
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < kChains / 2; ++c) s += x[c].x + x[c].y + (float)u[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const int threads = 1024, blocks = sms * 2;
  float* out;
  cudaMalloc(&out, sizeof(float) * threads * blocks);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double flops = 2.0 * kIters * kChains * (double)threads * blocks;
  auto run = [&](const char* name, void (*k)(float*, float, float)) {
    for (int w = 0; w < 3; ++w) k<<<blocks, threads>>>(out, 0.999f, 1e-3f);
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) k<<<blocks, threads>>>(out, 0.999f, 1e-3f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double tf = flops * 10 / (ms * 1e-3) / 1e12;
    printf("%-22s %8.3f ms  %6.1f TFLOP/s  %.1f FMA lanes/clk/SM (at %d MHz nominal)\n", name, ms / 10, tf,
           tf * 1e12 / 2 / sms / (clk_khz * 1e3), clk_khz / 1000);
  };
  run("scalar FFMA", scalar_fma);
  run("packed FFMA2", packed_fma);
  run("packed FFMA2 + ALU", packed_fma_plus_alu);
  cudaError_t err = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
