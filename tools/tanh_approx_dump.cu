// Dump tanh.approx.f32 on a uniform grid of [-12, 12] (diagnostic for the map tolerance).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tanhdump tools/tanh_approx_dump.cu
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
__global__ void k(float* y, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float x = -12.f + 24.f * (float)i / (float)(n - 1), r;
    asm("tanh.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    y[i] = r;
}
int main(int argc, char** argv) {
    const int n = 1 << 22;
    float* d;
    cudaMalloc(&d, n * 4);
    k<<<n / 256, 256>>>(d, n);
    std::vector<float> h(n);
    cudaMemcpy(h.data(), d, n * 4, cudaMemcpyDeviceToHost);
    FILE* f = fopen(argc > 1 ? argv[1] : "tanh_approx.bin", "wb");
    fwrite(h.data(), 4, n, f);
    fclose(f);
    printf("ok\n");
    return 0;
}
