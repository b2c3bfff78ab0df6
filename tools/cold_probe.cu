#include <cstdio>
#include <chrono>
#include <cuda_runtime.h>
__global__ void k(int* p) { if (p) *p = 1; }
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main() {
    double t0 = now();
    int n; cudaGetDeviceCount(&n);
    double t1 = now();
    cudaFree(0);
    double t2 = now();
    cudaDeviceSetLimit(cudaLimitStackSize, 4096);
    double t3 = now();
    void* h; cudaHostAlloc(&h, 1 << 20, cudaHostAllocDefault);
    double t4 = now();
    void* h2; cudaHostAlloc(&h2, 256 << 20, cudaHostAllocDefault);
    double t5 = now();
    int* d; cudaMalloc(&d, 4); k<<<1,1>>>(d); cudaDeviceSynchronize();
    double t6 = now();
    void* d2; cudaMalloc(&d2, 8ull << 30);
    double t7 = now();
    printf("{\"device_count_s\": %.3f, \"context_s\": %.3f, \"stack_limit_s\": %.3f, \"pinned_1MB_s\": %.3f, \"pinned_256MB_s\": %.3f, \"first_kernel_s\": %.3f, \"malloc_8GB_s\": %.3f}\n",
           t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4, t6 - t5, t7 - t6);
}
