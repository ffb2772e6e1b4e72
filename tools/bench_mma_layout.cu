// Microbenchmark: tcgen05.mma (kind::f16, M = 128) time per instruction for the operand layouts the band
// kernels use or could use: K-major no-swizzle ("interleave") vs K-major 128-byte swizzle for the SS
// score tiles; MN-major no-swizzle vs MN-major 128-byte swizzle for the B operand of the TS-form
// accumulation.  Timing only (operand contents are irrelevant).  Dev tool.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2605_08123_b200/csrc/st_sm100.cuh"
using namespace st::sm100;

__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1u << 46;
    d |= (uint64_t)2u << 61;  // SWIZZLE_128B
    return d;
}

// variant 0: SS K-major interleave; 1: SS K-major SW128; 2: TS, B MN-major interleave; 3: TS, B MN-major SW128
__global__ void k_mma(int variant, int N, int nacc, int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t tb;
    __shared__ uint64_t bar;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) { tc_alloc(&tb, 512); tc_relinquish(); }
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0x3c003c00u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tbase = tb;
    const int row_bytes = 256;  // d = 128 bf16
    const uint32_t a_addr = smem_u32(sm), b_addr = smem_u32(sm + 32 * 1024);
    unsigned long long t0 = 0, t1 = 0;
    if (warp == 0) {
        const uint32_t idesc_kk = make_idesc(128, N, 1u);
        const uint32_t idesc_mn = idesc_kk | (1u << 16);
        __syncwarp();
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
        if (elect_one()) {
            for (int it = 0; it < iters; ++it)
                for (int kk = 0; kk < 8; ++kk)
                    for (int c = 0; c < nacc; ++c) {
                        const uint32_t d = tbase + (uint32_t)(c * N) % 256;
                        if (variant == 0) {
                            const uint64_t ad = make_desc(a_addr, 128, 8 * row_bytes), bd = make_desc(b_addr, 128, 8 * row_bytes);
                            mma_bf16(d, ad + kk * 16, bd + kk * 16, idesc_kk, 1);
                        } else if (variant == 1) {
                            // K block kb = kk / 4 at + rows * 128 bytes; 32 bytes per K step inside the 128-byte row
                            const uint64_t ad = desc_sw128(a_addr + (kk / 4) * 128 * 128 + (kk % 4) * 32, 16, 1024);
                            const uint64_t bd = desc_sw128(b_addr + (kk / 4) * N * 128 + (kk % 4) * 32, 16, 1024);
                            mma_bf16(d, ad, bd, idesc_kk, 1);
                        } else if (variant == 2) {
                            const uint64_t bd = make_desc(b_addr + (kk % 4) * 16 * row_bytes, 8 * row_bytes, 128);
                            mma_bf16_ts(d, tbase + 384 + kk * 8, bd, idesc_mn, 1);
                        } else {
                            // MN-major SW128: 64-element groups of N at LBO = 64 rows * 128 B, 8-row K groups at SBO = 1024
                            const uint64_t bd = desc_sw128(b_addr + (kk % 4) * 2048, 64 * 128, 1024);
                            mma_bf16_ts(d, tbase + 384 + kk * 8, bd, idesc_mn, 1);
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

int main() {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* out; cudaMalloc(&out, nsm * 8);
    cudaFuncSetAttribute(k_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const char* names[4] = {"SS K-major interleave", "SS K-major SW128    ", "TS B MN-major interl.", "TS B MN-major SW128 "};
    for (int v = 0; v < 4; ++v)
        for (int N : {64, 128})
            for (int nacc : {1, 2}) {
                const int iters = 200;
                k_mma<<<nsm, 128, 200 * 1024>>>(v, N, nacc, iters, out);
                k_mma<<<nsm, 128, 200 * 1024>>>(v, N, nacc, iters, out);
                cudaDeviceSynchronize();
                unsigned long long h[256]; cudaMemcpy(h, out, nsm * 8, cudaMemcpyDeviceToHost);
                double mx = 0; for (int i = 0; i < nsm; ++i) mx = h[i] > mx ? h[i] : mx;
                printf("%s N=%3d nacc=%d: %.1f ns/MMA (%s)\n", names[v], N, nacc, mx / (iters * 8.0 * nacc), cudaGetErrorString(cudaGetLastError()));
            }
    return 0;
}
