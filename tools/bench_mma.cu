// Microbenchmark: tcgen05.mma throughput (kind::f16 / kind::tf32, M=128, no-swizzle K-major
// operands) vs N, dependent vs interleaved accumulators, A from SMEM vs TMEM (dev tool).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2605_08123_b200/csrc/st_sm100.cuh"
using namespace st::sm100;

template <int kFmt, bool kTS>
__global__ void k_mma(int N, int nacc, int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t tb;
    __shared__ uint64_t bar;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) { tc_alloc(&tb, 512); tc_relinquish(); }
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0x3c003c00u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tbase = tb;
    const int row_bytes = 256;  // K = 128 bf16 / 64 tf32 per row
    const uint32_t sbo = (row_bytes / 16) * 128;
    const uint32_t a_addr = smem_u32(sm), b_addr = smem_u32(sm + 128 * row_bytes);
    const uint32_t idesc = make_idesc(128, N, kFmt == 0 ? 1u : 2u);
    unsigned long long t0 = 0, t1 = 0;
    if (warp == 0) {
        const uint64_t ad = make_desc(a_addr, 128, sbo), bd = make_desc(b_addr, 128, sbo);
        if (kTS && elect_one()) {
            for (int kk = 0; kk < 8; ++kk) tc_cp_128x256b(tbase + 384 + kk * 8, ad + kk * 16);
        }
        __syncwarp();
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
        if (elect_one()) {
            for (int it = 0; it < iters; ++it)
                for (int kk = 0; kk < 8; ++kk)
                    for (int c = 0; c < nacc; ++c) {
                        const uint32_t d = tbase + (uint32_t)(c * N) % 384;
                        if (kTS) {
                            if (kFmt == 0) mma_bf16_ts(d, tbase + 384 + kk * 8, bd + kk * 16, idesc, 1);
                            else mma_tf32_ts(d, tbase + 384 + kk * 8, bd + kk * 16, idesc, 1);
                        } else {
                            if (kFmt == 0) mma_bf16(d, ad + kk * 16, bd + kk * 16, idesc, 1);
                            else mma_tf32(d, ad + kk * 16, bd + kk * 16, idesc, 1);
                        }
                    }
            tc_commit(&bar);
        }
        __syncwarp();
        mbar_wait(&bar, 0);
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
        if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before(); __syncthreads();
    if (warp == 0) { tc_fence_after(); tc_dealloc(tbase, 512); }
}

template <int kFmt, bool kTS>
void run(int N, int nacc) {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* out; cudaMalloc(&out, nsm * 8);
    auto k = k_mma<kFmt, kTS>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const int iters = 200;
    k<<<nsm, 128, 200 * 1024>>>(N, nacc, iters, out);
    k<<<nsm, 128, 200 * 1024>>>(N, nacc, iters, out);
    cudaDeviceSynchronize();
    unsigned long long h[256]; cudaMemcpy(h, out, nsm * 8, cudaMemcpyDeviceToHost);
    double mx = 0; for (int i = 0; i < nsm; ++i) mx = h[i] > mx ? h[i] : mx;
    const double K = kFmt == 0 ? 16 : 8;
    const double n_mma = (double)iters * 8 * nacc;
    const double flops = n_mma * 2.0 * 128 * N * K * nsm;
    printf("%s %s N=%3d nacc=%d: %.1f ns/MMA, %.0f TFLOP/s chip (%s)\n", kFmt == 0 ? "bf16" : "tf32", kTS ? "TS" : "SS",
           N, nacc, mx / n_mma, flops / (mx * 1e-9) / 1e12, cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}

int main() {
    for (int N : {32, 64, 128, 256})
        for (int nacc : {1, 4}) {
            if (N * nacc > 384 && nacc > 1) continue;
            run<0, false>(N, nacc);
            run<0, true>(N, nacc);
            run<1, false>(N, nacc);
            run<1, true>(N, nacc);
        }
    return 0;
}
