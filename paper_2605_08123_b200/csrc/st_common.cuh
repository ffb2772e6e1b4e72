// st_common.cuh -- shared device helpers for the sm_100a band kernels.
//
// Internal units: every score and dual is carried in base 2,
//   s2 = S * log2(e) = (q.k) * log2(e) / (sqrt(d) * eps),   u2 = u * log2(e), ...
// so a plan entry is ex2(s2 + u2_i + v2_j) (one MUFU.EX2) and a half-step is
//   u2_new = o - lg2( sum_j ex2(s2_ij + v2_j + o) )
// with the offset o = -max (cold start) or o = u2_prev (every later step; the
// previous plan is column-balanced, so every term is <= 1 and the sum lies
// in [1/W, W] -- no max pass).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace st {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

// Problem geometry, passed by value to every kernel.
struct Geo {
    int BH, H;       // heads = B*H, heads per example
    int Lq, Lk;      // rows / cols without the dustbin token
    int Lrq, Lrk;    // rows / cols of the stored tensors (+1 with the dustbin)
    int Lqp, Lkp;    // rows / cols of the stored score bands (multiples of 128)
    int d, w, Wf;    // head dim, half band, full band 2w+1
    int dustbin;     // 0 / 1
    int esz;         // input element bytes (4 f32, 2 bf16)
    int dbg;         // timing studies only (ST_BWD_DBG)
    float sd2;       // base-2 dustbin score: -cost * log2(e) / eps
    float c2;        // log2(e) / (sqrt(d) * eps)
    float inv_qk;    // 1 / (sqrt(d) * eps)
    float eps;
    const uint8_t* row_mask;  // [B, Lq] or null
    const uint8_t* col_mask;  // [B, Lk] or null
};

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float lg2(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}
__device__ __forceinline__ float warp_max(float x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
    return x;
}

__device__ __forceinline__ float ldf(const float* p) { return *p; }
__device__ __forceinline__ float ldf(const __nv_bfloat16* p) { return __bfloat162float(*p); }

// the same geometry seen from the key side (rows <-> columns): the column
// half-step is the row half-step of the transposed band
__host__ __device__ inline Geo transposed(const Geo& g) {
    Geo t = g;
    t.Lq = g.Lk;
    t.Lk = g.Lq;
    t.Lrq = g.Lrk;
    t.Lrk = g.Lrq;
    t.Lqp = g.Lkp;
    t.Lkp = g.Lqp;
    t.row_mask = g.col_mask;
    t.col_mask = g.row_mask;
    return t;
}

__device__ __forceinline__ bool row_on(const Geo& g, int bh, int i) {
    if (i >= g.Lq) return true;  // the dustbin row (exists only when g.dustbin)
    return g.row_mask == nullptr || g.row_mask[(size_t)(bh / g.H) * g.Lq + i] != 0;
}
__device__ __forceinline__ bool col_on(const Geo& g, int bh, int j) {
    if (j >= g.Lk) return true;
    return g.col_mask == nullptr || g.col_mask[(size_t)(bh / g.H) * g.Lk + j] != 0;
}

// Cell enumeration of one row / column of the (spoke-augmented) band support.
// Regular row i < Lq: k in [0, Wf) -> j = i - w + k (band), plus k = Wf -> the
// dustbin column j = Lk when dustbin.  The dustbin row i = Lq: k in [0, Lk]
// -> j = k.  Absent cells return s2 = -inf and a clamped, valid index.
__device__ __forceinline__ int row_ncells(const Geo& g, int i) { return i < g.Lq ? g.Wf + g.dustbin : g.Lk + 1; }
__device__ __forceinline__ void row_cell(const Geo& g, const float* __restrict__ S2, int bh, int i, int k, int& j,
                                         float& s2) {
    if (i < g.Lq) {
        if (k < g.Wf) {
            const int jj = i - g.w + k;
            if (jj >= 0 && jj < g.Lk) {
                j = jj;
                s2 = S2[((size_t)bh * g.Lqp + i) * g.Wf + k];
            } else {
                j = 0;
                s2 = -INFINITY;
            }
        } else {
            j = g.Lk;
            s2 = g.sd2;
        }
    } else {
        j = k;
        s2 = (k == g.Lk || col_on(g, bh, k)) ? g.sd2 : -INFINITY;
    }
}
__device__ __forceinline__ int col_ncells(const Geo& g, int j) { return j < g.Lk ? g.Wf + g.dustbin : g.Lq + 1; }
__device__ __forceinline__ void col_cell(const Geo& g, const float* __restrict__ S2, int bh, int j, int k, int& i,
                                         float& s2) {
    if (j < g.Lk) {
        if (k < g.Wf) {
            const int ii = j - g.w + k;
            if (ii >= 0 && ii < g.Lq) {
                i = ii;
                s2 = S2[((size_t)bh * g.Lqp + ii) * g.Wf + (2 * g.w - k)];
            } else {
                i = 0;
                s2 = -INFINITY;
            }
        } else {
            i = g.Lq;
            s2 = g.sd2;
        }
    } else {
        i = k;
        s2 = (k == g.Lq || row_on(g, bh, k)) ? g.sd2 : -INFINITY;
    }
}

}  // namespace st
