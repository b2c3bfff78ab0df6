// Integer-ALU peak of this B200 ("the per-SM INT/LOP3 lane
// count is not in MEASURED_PEAKS.json -- measure it with a LOP3-chain
// microbenchmark on the box before quoting fractions").
//
// Each thread runs 8 independent dependency chains of LOP3 (and, separately,
// IADD3 and IMNMX compare/select) for ITER rounds; the grid fills every SM
// with 64 warps.  Reported: thread-instructions per second over the
// whole GPU and per SM per cycle, at the SM clock measured INSIDE the kernel
// (block 0's clock64 cycles over its %globaltimer nanoseconds, the same
// interval), for each instruction kind.  The chains are unrolled so the
// loop overhead is < 3% of the issued instructions (checked in the SASS).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o alu_peak tools/alu_peak.cu && ./alu_peak
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

constexpr int ITER = 4096;
constexpr int CH = 8;

__global__ void lop3_kernel(unsigned* out, unsigned seed, long long* cycles) {
    unsigned a[CH];
    for (int c = 0; c < CH; c++) a[c] = seed ^ (threadIdx.x * 0x9E3779B9u + c);
    const unsigned b = seed * 3u + 1u, d = seed * 7u + 5u;
    const unsigned long long g0 = gtimer();
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < ITER; i++) {
#pragma unroll
        for (int c = 0; c < CH; c++) {
            unsigned r;
            asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(r) : "r"(a[c]), "r"(b), "r"(d));
            a[c] = r;
        }
    }
    long long t1 = clock64();
    const unsigned long long g1 = gtimer();
    unsigned x = 0;
    for (int c = 0; c < CH; c++) x ^= a[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        cycles[0] = t1 - t0;
        cycles[1] = (long long)(g1 - g0);
    }
}

__global__ void iadd3_kernel(unsigned* out, unsigned seed, long long* cycles) {
    unsigned a[CH];
    for (int c = 0; c < CH; c++) a[c] = seed + threadIdx.x * 17u + c;
    const unsigned b = seed * 3u + 1u, d = seed * 7u + 5u;
    const unsigned long long g0 = gtimer();
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < ITER; i++) {
#pragma unroll
        for (int c = 0; c < CH; c++) {
            unsigned r;
            asm volatile("add.u32 %0, %1, %2;" : "=r"(r) : "r"(a[c]), "r"(b));
            asm volatile("add.u32 %0, %1, %2;" : "=r"(a[c]) : "r"(r), "r"(d));
        }
    }
    long long t1 = clock64();
    const unsigned long long g1 = gtimer();
    unsigned x = 0;
    for (int c = 0; c < CH; c++) x ^= a[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        cycles[0] = t1 - t0;
        cycles[1] = (long long)(g1 - g0);
    }
}

__global__ void setp_sel_kernel(unsigned* out, unsigned seed, long long* cycles) {
    // the interval kernels' bread and butter: compare + select (min/max of bounds)
    int a[CH];
    for (int c = 0; c < CH; c++) a[c] = (int)(seed + threadIdx.x * 13u + c);
    const int b = (int)(seed * 3u + 1u);
    const unsigned long long g0 = gtimer();
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < ITER; i++) {
#pragma unroll
        for (int c = 0; c < CH; c++) {
            int r;
            asm volatile("max.s32 %0, %1, %2;" : "=r"(r) : "r"(a[c]), "r"(b));
            asm volatile("min.s32 %0, %1, %2;" : "=r"(a[c]) : "r"(r), "r"(b ^ i));
        }
    }
    long long t1 = clock64();
    const unsigned long long g1 = gtimer();
    int x = 0;
    for (int c = 0; c < CH; c++) x ^= a[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = (unsigned)x;
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        cycles[0] = t1 - t0;
        cycles[1] = (long long)(g1 - g0);
    }
}

template <typename K>
void run(const char* name, K kernel, int insts_per_chain_step, int sms) {
    const int threads = 1024, blocks = sms * 2;  // 64 warps per SM
    unsigned* out;
    long long* cyc;
    cudaMalloc(&out, (size_t)threads * blocks * 4);
    cudaMalloc(&cyc, 16);
    kernel<<<blocks, threads>>>(out, 1u, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    long long cyc_ns[2] = {0, 1};
    for (int r = 0; r < 5; r++) {
        cudaEventRecord(e0);
        kernel<<<blocks, threads>>>(out, (unsigned)r + 2u, cyc);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) {
            best = ms;
            cudaMemcpy(cyc_ns, cyc, 16, cudaMemcpyDeviceToHost);
        }
    }
    const double insts = (double)threads * blocks * ITER * CH * insts_per_chain_step;
    const double per_s = insts / (best * 1e-3);
    const double mhz = (double)cyc_ns[0] / (double)cyc_ns[1] * 1e3;  // cycles per ns of the same interval
    std::printf("{\"kind\": \"%s\", \"thread_inst_per_s\": %.4e, \"warp_inst_per_s\": %.4e, "
                "\"thread_inst_per_sm_per_clk\": %.1f, \"sm_mhz_in_kernel\": %.0f, \"ms\": %.3f, \"sms\": %d}\n",
                name, per_s, per_s / 32, per_s / sms / (mhz * 1e6), mhz, best, sms);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run("lop3", lop3_kernel, 1, sms);
    run("iadd", iadd3_kernel, 2, sms);
    run("imnmx", setp_sel_kernel, 2, sms);
    return 0;
}
