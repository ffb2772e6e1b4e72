// Microbenchmark: per-SM throughput of 1-D cp.async.bulk (TMA engine) global->shared
// copies issued by one thread into a ring of SMEM slots (dev tool).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2605_08123_b200/csrc/st_sm100.cuh"
using namespace st::sm100;

__global__ void k_bulk(const uint8_t* src, size_t src_bytes, int chunk, int nslot, int ncopy, unsigned long long* out, int issuers) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t* full = (uint64_t*)(sm + (size_t)nslot * chunk);
    if (threadIdx.x == 0) { for (int k = 0; k < nslot; ++k) mbar_init(&full[k], 1); fence_mbar_init(); }
    __syncthreads();
    unsigned long long t0;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    if (threadIdx.x == 0) {
        size_t off = (size_t)blockIdx.x * 1315423911ull % (src_bytes - chunk);
        off &= ~(size_t)127;
        for (int n = 0; n < ncopy; ++n) {
            const int sl = n % nslot;
            if (n >= nslot) mbar_wait(&full[sl], ((n / nslot) - 1) & 1);
            mbar_arrive_expect_tx(&full[sl], chunk);
            bulk_g2s(sm + (size_t)sl * chunk, src + off, chunk, &full[sl]);
            off += chunk; if (off + chunk > src_bytes) off = 0;
        }
        for (int n = ncopy; n < ncopy + nslot; ++n) { const int sl = n % nslot; mbar_wait(&full[sl], ((n / nslot) - 1) & 1); }
    }
    __syncthreads();
    unsigned long long t1;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    uint8_t* buf; size_t big = 2ull << 30; cudaMalloc(&buf, big); cudaMemset(buf, 1, big);
    unsigned long long* out; cudaMalloc(&out, nsm * 8);
    unsigned long long h[256];
    for (size_t srcb : {size_t(32) << 20, big})
    for (int chunk : {4096, 16384, 32768}) {
        for (int nslot : {2, 4, 8}) {
            size_t smem = (size_t)nslot * chunk + 1024;
            if (smem > 200 * 1024) continue;
            cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            int ncopy = (int)((64ll << 20) / chunk / 16);
            k_bulk<<<nsm, 32, smem>>>(buf, srcb, chunk, nslot, ncopy, out, 1);
            k_bulk<<<nsm, 32, smem>>>(buf, srcb, chunk, nslot, ncopy, out, 1);
            cudaDeviceSynchronize();
            cudaMemcpy(h, out, nsm * 8, cudaMemcpyDeviceToHost);
            double mx = 0; for (int i = 0; i < nsm; ++i) mx = h[i] > mx ? h[i] : mx;
            double per = (double)ncopy * chunk / (mx * 1e-9) / 1e9;
            printf("src %5zu MiB chunk %6d slots %d: per-SM %.1f GB/s, total %.0f GB/s (%s)\n", srcb >> 20, chunk, nslot, per, per * nsm, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
