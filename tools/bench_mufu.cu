// Microbenchmark: MUFU.EX2 throughput vs an FMA-pipe polynomial exp2 on this GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bench_mufu tools/bench_mufu.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2a(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// 2^x for x <= 0 on the FMA pipe: x = n + f, f in [-0.5, 0.5], degree-6 minimax of 2^f
__device__ __forceinline__ float ex2p(float x) {
    x = fmaxf(x, -127.f);
    const float n = rintf(x);
    const float f = x - n;
    float p = 1.5353362e-4f;
    p = fmaf(p, f, 1.3398874e-3f);
    p = fmaf(p, f, 9.6181291e-3f);
    p = fmaf(p, f, 5.5504109e-2f);
    p = fmaf(p, f, 2.4022651e-1f);
    p = fmaf(p, f, 6.9314718e-1f);
    p = fmaf(p, f, 1.0f);
    return __int_as_float(__float_as_int(p) + ((int)n << 23));
}

template <int MODE>
__global__ void k(float* out, int iters) {
    float a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = -0.001f * (threadIdx.x + j);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (MODE == 0) a[j] = ex2a(a[j]) - 1.0f;
            else if (MODE == 1) a[j] = ex2p(a[j]) - 1.0f;
            else a[j] = ((j & 1) ? ex2p(a[j]) : ex2a(a[j])) - 1.0f;
        }
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += a[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int dev = 0, nsm = 0, clk = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    float* out;
    cudaMalloc(&out, 64 << 20);
    const int blocks = nsm * 8, threads = 256, iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char* names[3] = {"MUFU.EX2", "poly (FMA pipe)", "half/half"};
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (mode == 0) k<0><<<blocks, threads>>>(out, iters);
            else if (mode == 1) k<1><<<blocks, threads>>>(out, iters);
            else k<2><<<blocks, threads>>>(out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double n = (double)blocks * threads * iters * 8;
        printf("%-18s %.3f ms  %.3e exp/s  %.2f exp/clk/SM (at %.0f MHz max)\n", names[mode], ms, n / (ms * 1e-3),
               n / (ms * 1e-3) / nsm / (clk * 1e3), clk / 1e3);
    }
    return 0;
}
