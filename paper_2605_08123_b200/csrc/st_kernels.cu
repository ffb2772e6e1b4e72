// st_kernels.cu -- sm_100a kernels of the band operator (generic path).
//
// Forward (run_surrogate, sinkhorn.hpp:288-302):
//   k_scores    S2 band field [BH][Lq][Wf] = q.k * log2e/(sqrt(d) eps), -inf off support
//   k_row_step  u half-step  (row_half_step,  sinkhorn.hpp:15-61)
//   k_col_step  v half-step  (col_half_step,  sinkhorn.hpp:64-107)
//   k_output    O = P V      (apply_transport, sinkhorn.hpp:262-277)
//   k_gauges    ledger gauges (center, sinkhorn.hpp:118-140) -- duals run raw
// Backward (r2_backward, adjoint.hpp:232-373): k_bwd_row / k_bwd_col sweeps.
//
// Every reduction is owned by one warp (one row or one column), so results are
// deterministic and independent of launch geometry.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "st_common.cuh"
#include "st_kernels.cuh"
#include "st_sm100.cuh"

namespace st {

// ---------------------------------------------------------------------------
// Band dot products: S2[bh][i][k] = (q_i . k_j) * c2 for j = i - w + k (kZ: the
// cotangent band Z = dO_i . V_j, unscaled).  One CTA = 64 rows x one head; the
// row tile and the column window [i0-w, i0+63+w] sit K-major in SMEM (x-major,
// float4 reads), 256 threads each own a 4 x 4 micro-tile per 64-column block.
// fp32 inputs accumulate in f64 (products of floats are exact in f64, so the
// stored score is the correctly rounded fp32 value); bf16 inputs accumulate in
// fp32 (bf16 products are exact in fp32), the tensor-core contract.
// Off-support cells: -inf (scores) / 0 (Z).
// ---------------------------------------------------------------------------
constexpr int kScoreRows = 64;

template <class TIn, class TAcc, bool kZ>
__global__ void __launch_bounds__(256) k_scores(Geo g, const TIn* __restrict__ Q, const TIn* __restrict__ K,
                                                float* __restrict__ S2) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* smem = reinterpret_cast<float*>(smem_raw);
    const int bh = blockIdx.y;
    const int i0 = blockIdx.x * kScoreRows;
    const int ncol = ((kScoreRows + 2 * g.w + 63) / 64) * 64;  // window columns, padded to 64
    const int c0 = i0 - g.w;                                     // original column of window column 0
    const int dp = g.d + 1;                                      // odd pitch: conflict-free column walks
    float* sq = smem;                                            // [64][dp]
    float* sk = smem + kScoreRows * dp;                          // [ncol][dp]
    const int tid = threadIdx.x;
    const TIn* Qh = Q + (size_t)bh * g.Lrq * g.d;
    const TIn* Kh = K + (size_t)bh * g.Lrk * g.d;
    for (int e = tid; e < kScoreRows * g.d; e += 256) {
        const int r = e / g.d, x = e % g.d;
        sq[r * dp + x] = ((i0 + r < g.Lq) ? ldf(Qh + (size_t)(i0 + r) * g.d + x) : 0.f);
    }
    for (int e = tid; e < ncol * g.d; e += 256) {
        const int c = e / g.d, x = e % g.d;
        const int j = c0 + c;
        sk[c * dp + x] = ((j >= 0 && j < g.Lk) ? ldf(Kh + (size_t)j * g.d + x) : 0.f);
    }
    __syncthreads();
    // thread (ty, tx) owns rows ty + 16a and columns cb + tx + 16b (a, b < 4) of each 64-column block
    const int ty = tid >> 4, tx = tid & 15;
    for (int cb = 0; cb < ncol; cb += 64) {
        TAcc acc[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = TAcc(0);
        const float* qr = sq + ty * dp;
        const float* kr = sk + (cb + tx) * dp;
#pragma unroll 4
        for (int x = 0; x < g.d; ++x) {
            TAcc q4[4], k4[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) q4[a] = (TAcc)qr[16 * a * dp + x];
#pragma unroll
            for (int b = 0; b < 4; ++b) k4[b] = (TAcc)kr[16 * b * dp + x];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b] = fma(q4[a], k4[b], acc[a][b]);
        }
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const int i = i0 + ty + 16 * a;
            if (i >= g.Lq) continue;
            const bool ron = row_on(g, bh, i);
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int j = c0 + cb + tx + 16 * b;
                const int k = j - i + g.w;
                if (k < 0 || k >= g.Wf) continue;
                const bool on = ron && j >= 0 && j < g.Lk && col_on(g, bh, j);
                float val;
                if (kZ) val = on ? (float)acc[a][b] : 0.f;
                else val = on ? (float)(acc[a][b] * (TAcc)g.c2) : -INFINITY;
                S2[((size_t)bh * g.Lqp + i) * g.Wf + k] = val;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Band dot products on the FP64 tensor cores (mma.sync m8n8k4 .f64): the same
// field as k_scores, exact products and f64 accumulation, rounded once to fp32.
// CTA = 128 rows of one head; warp = RT 8-row tiles, its A fragments (query
// rows, converted to f64) register-resident; the key window [i0-w, ...) sits
// in SMEM as fp32 with pitch D+4 (B fragment loads are bank-conflict free).
// A warp visits only the 8-column tiles its rows' bands touch (~1.1x the band).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

template <int D>
struct BandMma {
    static constexpr int CP = D <= 64 ? 2 : 1;   // key column tiles per warp pass (B fragments in registers)
    static constexpr int NWARP = 8;
    static constexpr int P = D + 4;               // SMEM pitch (doubles): conflict-free A fragment loads
    static constexpr int RB = D <= 64 ? 128 : 64; // query rows per CTA (d = 128: 64 rows -> 3 CTAs / SM)
    static size_t smem() { return (size_t)RB * P * 8; }
};

// Warp pass = CP key column tiles (8 keys each, B fragments converted to f64
// once, register-resident); it walks the query row tiles whose bands touch
// those columns, A fragments (f64) streamed from SMEM: one LDS.64 feeds CP
// DMMAs and the inner loop has no conversions.
template <class TIn, bool kZ, int D>
__global__ void __launch_bounds__(256) k_band_mma(Geo g, const TIn* __restrict__ A, const TIn* __restrict__ B,
                                                  float* __restrict__ out, float* __restrict__ outT) {
    using M = BandMma<D>;
    constexpr int CP = M::CP, P = M::P, KS = D / 4, RB = M::RB, NRT = RB / 8;
    extern __shared__ __align__(16) double sqa[];  // [RB][P] query rows of the block, f64
    const int bh = blockIdx.y, i0 = blockIdx.x * RB, j0 = i0 - g.w;
    const TIn* Ah = A + (size_t)bh * g.Lrq * D;
    const TIn* Bh = B + (size_t)bh * g.Lrk * D;
    for (int e = threadIdx.x; e < RB * (D / 4); e += 256) {
        const int r = e / (D / 4), x = (e % (D / 4)) * 4;
        const int i = i0 + r;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (i < g.Lq) {
            const TIn* src = Ah + (size_t)i * D + x;
            if constexpr (sizeof(TIn) == 4) {
                v = *reinterpret_cast<const float4*>(src);
            } else {
                v.x = ldf(src); v.y = ldf(src + 1); v.z = ldf(src + 2); v.w = ldf(src + 3);
            }
        }
        double* dst = sqa + r * P + x;
        dst[0] = v.x;
        dst[1] = v.y;
        dst[2] = v.z;
        dst[3] = v.w;
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gq = lane >> 2, tq = lane & 3;
    const int CT = (7 + 2 * g.w) / 8 + 1;     // column tiles one row tile touches
    const int NCT = NRT - 1 + CT;             // column tiles of the block window
    const int npass = (NCT + CP - 1) / CP;
    for (int pass = warp; pass < npass; pass += M::NWARP) {
        const int c0 = pass * CP;
        double bf[CP][KS];
        bool jon[CP][2];
#pragma unroll
        for (int u = 0; u < CP; ++u) {
            const int jr = j0 + 8 * (c0 + u) + gq;  // key row of this lane's B fragment
            const bool ok = jr >= 0 && jr < g.Lk;
#pragma unroll
            for (int s = 0; s < KS; ++s) bf[u][s] = ok ? (double)ldf(Bh + (size_t)jr * D + 4 * s + tq) : 0.0;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int j = j0 + 8 * (c0 + u) + 2 * tq + h;
                jon[u][h] = j >= 0 && j < g.Lk && col_on(g, bh, j);
            }
        }
        // row tiles touching column tiles [c0, c0 + CP): ri in [c0 - CT + 1, c0 + CP - 1]
        const int rlo = max(0, c0 - CT + 1), rhi = min(NRT - 1, c0 + CP - 1);
        // two row tiles per iteration: 2*CP independent accumulation chains per warp
        for (int ri = rlo; ri <= rhi; ri += 2) {
            const bool two = ri + 1 <= rhi;
            double c[2][CP][2];
#pragma unroll
            for (int q = 0; q < 2; ++q)
#pragma unroll
                for (int u = 0; u < CP; ++u) c[q][u][0] = c[q][u][1] = 0.0;
            const double* ap = sqa + (8 * ri + gq) * P + tq;
            const double* ap2 = ap + (two ? 8 * P : 0);
#pragma unroll
            for (int s = 0; s < KS; ++s) {
                const double av = ap[4 * s], av2 = ap2[4 * s];
#pragma unroll
                for (int u = 0; u < CP; ++u) {
                    dmma884(c[0][u][0], c[0][u][1], av, bf[u][s]);
                    dmma884(c[1][u][0], c[1][u][1], av2, bf[u][s]);
                }
            }
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                if (q == 1 && !two) break;
                const int i = i0 + 8 * (ri + q) + gq;
                if (i >= g.Lqp) continue;
                const bool rr = i < g.Lq && row_on(g, bh, i);
#pragma unroll
                for (int u = 0; u < CP; ++u)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int j = j0 + 8 * (c0 + u) + 2 * tq + h;
                        const int k = j - i + g.w;
                        if (k < 0 || k >= g.Wf) continue;
                        const bool on = rr && jon[u][h];
                        float val;
                        if (kZ) val = on ? (float)c[q][u][h] : 0.f;
                        else val = on ? (float)(c[q][u][h] * (double)g.c2) : -INFINITY;
                        out[((size_t)bh * g.Lqp + i) * g.Wf + k] = val;
                        // the same cell of the transposed band (key side): row j, k' = 2w - k
                        if (outT != nullptr && j >= 0 && j < g.Lkp)
                            outT[((size_t)bh * g.Lkp + j) * g.Wf + (2 * g.w - k)] = val;
                    }
            }
        }
    }
    // transposed-band cells whose row i falls outside [0, Lqp) (no row block produces them):
    // the head's edge cells are split evenly over its row-block CTAs
    if (outT != nullptr) {
        const float fill = kZ ? 0.f : -INFINITY;
        const int ne = min(g.w, g.Lkp), tot = 2 * ne * g.Wf;
        const int per = (tot + gridDim.x - 1) / gridDim.x;
        const int e0 = blockIdx.x * per, e1 = min(tot, e0 + per);
        for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
            const int rr = e / g.Wf, kp = e % g.Wf;
            const int j = rr < ne ? rr : g.Lkp - 2 * ne + rr;
            const int i = j - g.w + kp;
            if (i < 0 || i >= g.Lqp) outT[((size_t)bh * g.Lkp + j) * g.Wf + kp] = fill;
        }
    }
}

// ---------------------------------------------------------------------------
// S2T[bh][j][k'] = S2[bh][j - w + k'][2w - k']  (the band seen from the key side;
// -inf where the row is outside [0, Lq)).  Coalesced writes, L2-served gathers.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_transpose_band(Geo g, const float* __restrict__ S2, float* __restrict__ S2T,
                                                        float fill) {
    const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const long total = (long)g.BH * g.Lkp * g.Wf;
    if (t >= total) return;
    const int kp = (int)(t % g.Wf);
    const long rj = t / g.Wf;
    const int j = (int)(rj % g.Lkp), bh = (int)(rj / g.Lkp);
    const int i = j - g.w + kp;
    float v = fill;
    if (j < g.Lk && i >= 0 && i < g.Lq) v = S2[((size_t)bh * g.Lqp + i) * g.Wf + (2 * g.w - kp)];
    S2T[t] = v;
}

// ---------------------------------------------------------------------------
// Tile half-step over a stored band (fp32 path).  One CTA = 128 rows of one
// head: the 128 x Wf band tile is contiguous in HBM/L2 and lands in SMEM with a
// single bulk async copy (TMA engine); the window duals land beside it; thread
// r owns row i0 + r and reduces in-thread (stride Wf is odd: conflict-free).
// The column half-step runs this kernel on the transposed band.
// ---------------------------------------------------------------------------
template <bool kFirst>
__global__ void __launch_bounds__(128) k_stepT(Geo g, const float* __restrict__ S2, const float* __restrict__ dual_other,
                                               const float* off_own, float* out_own, int* err) {
    extern __shared__ __align__(16) float smf[];
    __shared__ __align__(8) uint64_t bar;
    if (g.dustbin && blockIdx.x == gridDim.x - 1) {
        // the extra CTA column: the own side's dustbin dual (a full-length line over the other side's
        // active duals and the corner, constant score sd2), same launch as the band rows
        __shared__ float red[4];
        const int bh = blockIdx.y, t = threadIdx.x, lane = t & 31, wid = t >> 5;
        const float* dual = dual_other + (size_t)bh * g.Lrk;
        const int n = g.Lk + 1;
        float off;
        if (kFirst) {
            float m = -INFINITY;
            for (int j = t; j < n; j += 128)
                if (j == g.Lk || col_on(g, bh, j)) m = fmaxf(m, g.sd2 + dual[j]);
            m = warp_max(m);
            if (lane == 0) red[wid] = m;
            __syncthreads();
            off = -fmaxf(fmaxf(red[0], red[1]), fmaxf(red[2], red[3]));
            __syncthreads();
        } else {
            off = off_own[(size_t)bh * g.Lrq + g.Lq];
        }
        float sum = 0.f;
        for (int j = t; j < n; j += 128)
            if (j == g.Lk || col_on(g, bh, j)) sum += ex2(g.sd2 + dual[j] + off);
        sum = warp_sum(sum);
        if (lane == 0) red[wid] = sum;
        __syncthreads();
        if (t == 0) {
            const float tot = (red[0] + red[1]) + (red[2] + red[3]);
            float u = off - lg2(tot);
            if (!(tot > 0.f) || !isfinite(u)) {
                atomicOr(err, 8);
                u = 0.f;
            }
            out_own[(size_t)bh * g.Lrq + g.Lq] = u;
        }
        return;
    }
    const int bh = blockIdx.y, i0 = blockIdx.x * 128, r = threadIdx.x, i = i0 + r;
    const bool active = i < g.Lq && row_on(g, bh, i);
    if (!__syncthreads_or(active)) {
        if (i < g.Lq) out_own[(size_t)bh * g.Lrq + i] = 0.f;
        return;
    }
    float* tile = smf;
    float* vw = smf + 128 * g.Wf;
    if (threadIdx.x == 0) {
        sm100::mbar_init(&bar, 1);
        sm100::fence_mbar_init();
    }
    __syncthreads();
    const uint32_t bytes = 128u * (uint32_t)g.Wf * 4u;
    if (threadIdx.x == 0) {
        sm100::mbar_arrive_expect_tx(&bar, bytes);
        sm100::bulk_g2s(tile, S2 + ((size_t)bh * g.Lqp + i0) * g.Wf, bytes, &bar);
    }
    const float* dual = dual_other + (size_t)bh * g.Lrk;
    for (int c = threadIdx.x; c < 128 + 2 * g.w; c += 128) {
        const int j = i0 - g.w + c;
        vw[c] = (j >= 0 && j < g.Lk && col_on(g, bh, j)) ? dual[j] : -INFINITY;
    }
    __syncthreads();
    sm100::mbar_wait(&bar, 0);
    if (i >= g.Lq) return;
    float u = 0.f;
    if (active) {
        const float* trow = tile + r * g.Wf;
        const float* vr = vw + r;
        const float xd = g.dustbin ? g.sd2 + dual[g.Lk] : -INFINITY;  // spoke cell (i, dustbin)
        float o;
        if (kFirst) {
            float m = xd;
            for (int k = 0; k < g.Wf; ++k) m = fmaxf(m, trow[k] + vr[k]);
            o = -m;
        } else {
            o = off_own[(size_t)bh * g.Lrq + i];
        }
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
        int k = 0;
        for (; k + 4 <= g.Wf; k += 4) {
            s0 += ex2(trow[k] + vr[k] + o);
            s1 += ex2(trow[k + 1] + vr[k + 1] + o);
            s2 += ex2(trow[k + 2] + vr[k + 2] + o);
            s3 += ex2(trow[k + 3] + vr[k + 3] + o);
        }
        for (; k < g.Wf; ++k) s0 += ex2(trow[k] + vr[k] + o);
        float s = (s0 + s1) + (s2 + s3);
        if (g.dustbin) s += ex2(xd + o);
        u = o - lg2(s);
        if (!(s > 0.f) || !isfinite(u)) {
            atomicOr(err, 16);
            u = 0.f;
        }
    }
    out_own[(size_t)bh * g.Lrq + i] = u;
}

// ---------------------------------------------------------------------------
// Fused full step over the stored band (fp32 path, no dustbin).  Launch t:
//   1. combine: v_{t-1}(window) from the column partials of launch t-1 (fixed
//      order over the <= 3 contributing blocks) and v_{t-2}; the owner block
//      writes v_{t-1} for its own 128 columns
//   2. row pass: e_ij = 2^(s2 + v_{t-1,j} + u_{t-1,i}), r_i = sum_j e_ij,
//      u_t = u_{t-1} - lg2 r_i  (row_half_step, sinkhorn.hpp:15-61)
//   3. column partials: sum_{i in block} e_ij / r_i, i.e. the column half-step
//      (col_half_step, sinkhorn.hpp:64-107) reuses the row pass exponentials:
//      e_ij / r_i = 2^(s2 + u_t,i + v_{t-1,j}) -- one exp per cell per full step.
// Cold start (t = 1): row max offsets, and log-domain (max, sum) column
// partials so that no column can underflow.
// ---------------------------------------------------------------------------
struct FStep {
    const float* S2;
    const float* u_prev;  // [BH][Lrq] u_{t-1} (offsets)
    float* u_out;         // [BH][Lrq] u_t
    const float* v_pp;    // [BH][Lrk] v_{t-2} (null when t-2 == 0)
    float* v_p_out;       // [BH][Lrk] v_{t-1} written by owners (null at t = 1)
    float* v_p_slot;      // optional extra copy of v_{t-1} (saved slot) or null
    const float* part_in;   // [BH][NB][Nw] partials of launch t-1
    const float* partm_in;  // [BH][NB][Nw] partial maxima (launch 1 only) or null
    float* part_out;
    float* partm_out;     // written at t = 1
    int NB, Nw;
    int* err;
};

__device__ __forceinline__ float combine_col(const Geo& g, const FStep& f, int bh, int j, bool pairs) {
    // blocks whose window [128b - w, 128b + 127 + w] contains column j
    const int a = j - 127 - g.w;
    const int blo = max(0, a > 0 ? (a + 127) / 128 : 0);  // ceil((j - 127 - w) / 128)
    const int bhi = min(f.NB - 1, (j + g.w) / 128);
    const size_t base = (size_t)bh * f.NB * f.Nw;
    if (!pairs) {
        float s = 0.f;
        for (int b = blo; b <= bhi; ++b) s += f.part_in[base + (size_t)b * f.Nw + (j - (128 * b - g.w))];
        return lg2(s);  // v_{t-1} = v_{t-2} - lg2(s)
    }
    float M = -INFINITY;
    for (int b = blo; b <= bhi; ++b) M = fmaxf(M, f.partm_in[base + (size_t)b * f.Nw + (j - (128 * b - g.w))]);
    float s = 0.f;
    for (int b = blo; b <= bhi; ++b) {
        const size_t k = base + (size_t)b * f.Nw + (j - (128 * b - g.w));
        const float m = f.partm_in[k];
        if (m != -INFINITY) s += f.part_in[k] * ex2(m - M);
    }
    return M + lg2(s);  // v_1 = -(M + lg2 s)   (v_0 = 0)
}

// One CTA = one 128-row block, its band tile bulk-copied whole into SMEM.
// 256 threads: in the row pass two threads share a row (lanes r and r+16 of a
// warp; thread h takes the 16-cell groups h, h+2, ... -- with the odd pitch Wf
// the 32 lanes hit 32 distinct banks); in the column pass one thread per
// window column.  The prologue issues every global load it needs (mask bytes,
// v_{t-2}, the block partials, u_{t-1}) before consuming any of them, so
// their latencies overlap one another and the tile copy.
constexpr int kFsThreads = 256;
constexpr int kFsCols = 2;    // window columns per thread (Nw <= 512)

template <bool kFirst, bool kPairsIn>
__global__ void __launch_bounds__(kFsThreads) k_fstep(Geo g, FStep f) {
    extern __shared__ __align__(16) float smf[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ float inv_r[128];
    const int bh = blockIdx.y, b = blockIdx.x, i0 = b * 128, tid = threadIdx.x;
    const int lane = tid & 31, h = lane >> 4, r = (tid >> 5) * 16 + (lane & 15), i = i0 + r;
    const unsigned pmask = (1u << (lane & 15)) | (1u << ((lane & 15) + 16));  // the two lanes of row r
    const int Nw = f.Nw, Wf = g.Wf;
    float* tile = smf;               // [128][Wf]: scores, then e (or x at cold start)
    float* vw = smf + 128 * Wf;      // [Nw] window duals v_{t-1}
    const bool in_rows = i < g.Lq;
    const uint8_t* rmask = g.row_mask ? g.row_mask + (size_t)(bh / g.H) * g.Lq : nullptr;
    const uint8_t* cmask = g.col_mask ? g.col_mask + (size_t)(bh / g.H) * g.Lk : nullptr;
    const bool active = in_rows && (rmask == nullptr || rmask[i] != 0);
    const float uo = (!kFirst && in_rows) ? f.u_prev[(size_t)bh * g.Lrq + i] : 0.f;
    const bool any = __syncthreads_or(active);
    if (any && tid == 0) {
        sm100::mbar_init(&bar, 1);
        sm100::fence_mbar_init();
        const uint32_t bytes = 128u * (uint32_t)Wf * 4u;
        sm100::mbar_arrive_expect_tx(&bar, bytes);
        sm100::bulk_g2s(tile, f.S2 + ((size_t)bh * g.Lqp + i0) * Wf, bytes, &bar);
    }
    // ---- 1. combine: v_{t-1} on the window; owners write their 128 columns
    const size_t pb = (size_t)bh * f.NB * Nw;
#pragma unroll
    for (int a = 0; a < kFsCols; ++a) {
        const int c = tid + kFsThreads * a;
        if (c >= Nw) break;
        const int j = i0 - g.w + c;
        const bool inr = j >= 0 && j < g.Lk;
        const int jc = inr ? j : 0;
        const bool con = inr && (cmask == nullptr || cmask[jc] != 0);
        float v = -INFINITY;
        if (kFirst) {
            if (con) v = 0.f;
        } else {
            // contributing blocks b-2 .. b+2 (w <= 128); window column of j in block b' = c + 128 (b - b')
            float pv[5], pm[5];
#pragma unroll
            for (int d = 0; d < 5; ++d) {
                const int bb = b - 2 + d;
                const int cc = c + 128 * (2 - d);
                const bool ok = bb >= 0 && bb < f.NB && cc >= 0 && cc < Nw;
                const size_t k = pb + (size_t)(ok ? bb : 0) * Nw + (ok ? cc : 0);
                pv[d] = ok ? f.part_in[k] : 0.f;
                pm[d] = (kPairsIn && ok) ? f.partm_in[k] : -INFINITY;
            }
            const float prev = (f.v_pp && inr) ? f.v_pp[(size_t)bh * g.Lrk + jc] : 0.f;
            if (con) {
                if (kPairsIn) {
                    float M = -INFINITY;
#pragma unroll
                    for (int d = 0; d < 5; ++d) M = fmaxf(M, pm[d]);
                    float sum = 0.f;
#pragma unroll
                    for (int d = 0; d < 5; ++d)
                        if (pm[d] != -INFINITY) sum += pv[d] * ex2(pm[d] - M);
                    v = -(M + lg2(sum));
                } else {
                    float sum = 0.f;
#pragma unroll
                    for (int d = 0; d < 5; ++d) sum += pv[d];
                    v = prev - lg2(sum);
                }
                if (!isfinite(v)) {
                    atomicOr(f.err, 32);
                    v = 0.f;
                }
            }
        }
        vw[c] = v;
        if (!kFirst && c >= g.w && c < g.w + 128 && j < g.Lk) {  // owner of column j
            const float vo = (v == -INFINITY) ? 0.f : v;
            f.v_p_out[(size_t)bh * g.Lrk + j] = vo;
            if (f.v_p_slot) f.v_p_slot[(size_t)bh * g.Lrk + j] = vo;
        }
    }
    const size_t pbase = pb + (size_t)b * Nw;
    if (!any) {  // fully masked block: zero partials, zero duals
        for (int c = tid; c < Nw; c += kFsThreads) {
            f.part_out[pbase + c] = 0.f;
            if (kFirst) f.partm_out[pbase + c] = -INFINITY;
        }
        if (in_rows && h == 0) f.u_out[(size_t)bh * g.Lrq + i] = 0.f;
        return;
    }
    __syncthreads();
    sm100::mbar_wait(&bar, 0);
    // ---- 2. row pass (threads (r, h)); tile row becomes e (or x)
    float* trow = tile + r * Wf;
    const float* vr = vw + r;
    if (active) {
        float o;
        if (kFirst) {
            float m = -INFINITY;
            for (int k0 = 16 * h; k0 < Wf; k0 += 32)
#pragma unroll
                for (int kk = 0; kk < 16; ++kk)
                    if (k0 + kk < Wf) m = fmaxf(m, trow[k0 + kk] + vr[k0 + kk]);
            m = fmaxf(m, __shfl_xor_sync(pmask, m, 16));
            o = -m;
        } else {
            o = uo;
        }
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
        for (int k0 = 16 * h; k0 < Wf; k0 += 32) {
            if (k0 + 16 <= Wf) {
#pragma unroll
                for (int kk = 0; kk < 16; kk += 4) {
                    const int k = k0 + kk;
                    const float x0 = trow[k] + vr[k] + o, x1 = trow[k + 1] + vr[k + 1] + o;
                    const float x2 = trow[k + 2] + vr[k + 2] + o, x3 = trow[k + 3] + vr[k + 3] + o;
                    const float e0 = ex2(x0), e1 = ex2(x1), e2 = ex2(x2), e3 = ex2(x3);
                    trow[k] = kFirst ? x0 : e0;
                    trow[k + 1] = kFirst ? x1 : e1;
                    trow[k + 2] = kFirst ? x2 : e2;
                    trow[k + 3] = kFirst ? x3 : e3;
                    s0 += e0;
                    s1 += e1;
                    s2 += e2;
                    s3 += e3;
                }
            } else {
                for (int k = k0; k < Wf; ++k) {
                    const float x = trow[k] + vr[k] + o;
                    const float e = ex2(x);
                    trow[k] = kFirst ? x : e;
                    s0 += e;
                }
            }
        }
        float rs = (s0 + s1) + (s2 + s3);
        rs += __shfl_xor_sync(pmask, rs, 16);
        const float lr = lg2(rs);
        float u = o - lr;
        if (!(rs > 0.f) || !isfinite(u)) {
            if (h == 0) atomicOr(f.err, 64);
            u = 0.f;
        }
        if (h == 0) {
            f.u_out[(size_t)bh * g.Lrq + i] = u;
            inv_r[r] = kFirst ? lr : 1.f / rs;  // cold start keeps lg2 r_i (log-domain partials)
        }
    } else {
        if (h == 0) {
            if (in_rows) f.u_out[(size_t)bh * g.Lrq + i] = 0.f;
            inv_r[r] = kFirst ? INFINITY : 0.f;
        }
        const float z = kFirst ? -INFINITY : 0.f;  // no -inf * 0 in the column pass
        for (int k = h; k < Wf; k += 2) trow[k] = z;
    }
    __syncthreads();
    // ---- 3. column partials: window column c collects rows ii with c - 2w <= ii <= c
#pragma unroll
    for (int a = 0; a < kFsCols; ++a) {
        const int c = tid + kFsThreads * a;
        if (c >= Nw) break;
        const int lo = max(0, c - 2 * g.w), hi = min(127, c);
        const float* tp = tile + lo * Wf + (c - lo);
        const int step = Wf - 1;
        if (kFirst) {
            float M = -INFINITY;
            for (int ii = lo; ii <= hi; ++ii) M = fmaxf(M, tp[(ii - lo) * step] - inv_r[ii]);
            float sum = 0.f;
            if (M != -INFINITY)
                for (int ii = lo; ii <= hi; ++ii) sum += ex2(tp[(ii - lo) * step] - inv_r[ii] - M);
            f.part_out[pbase + c] = sum;
            f.partm_out[pbase + c] = M;
        } else {
            float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
            int ii = lo;
            for (; ii + 3 <= hi; ii += 4, tp += 4 * step) {
                s0 = fmaf(tp[0], inv_r[ii], s0);
                s1 = fmaf(tp[step], inv_r[ii + 1], s1);
                s2 = fmaf(tp[2 * step], inv_r[ii + 2], s2);
                s3 = fmaf(tp[3 * step], inv_r[ii + 3], s3);
            }
            for (; ii <= hi; ++ii, tp += step) s0 = fmaf(tp[0], inv_r[ii], s0);
            f.part_out[pbase + c] = (s0 + s1) + (s2 + s3);
        }
    }
}

// v_{T+R} from the last partials (the finishing half of the last full step)
template <bool kPairsIn>
__global__ void k_ffinal(Geo g, FStep f) {
    const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (long)g.BH * g.Lk) return;
    const int bh = (int)(t / g.Lk), j = (int)(t % g.Lk);
    float v = 0.f;
    if (col_on(g, bh, j)) {
        const float prev = f.v_pp ? f.v_pp[(size_t)bh * g.Lrk + j] : 0.f;
        v = kPairsIn ? -combine_col(g, f, bh, j, true) : prev - combine_col(g, f, bh, j, false);
        if (!isfinite(v)) {
            atomicOr(f.err, 32);
            v = 0.f;
        }
    }
    f.v_p_out[(size_t)bh * g.Lrk + j] = v;
    if (f.v_p_slot) f.v_p_slot[(size_t)bh * g.Lrk + j] = v;
}

// ---------------------------------------------------------------------------
// Half-steps (warp per row / column).  kFirst: explicit max offset (cold
// start); otherwise the previous dual of the same row/column is the offset.
// ---------------------------------------------------------------------------
template <bool kFirst>
__global__ void __launch_bounds__(256) k_row_step(Geo g, const float* __restrict__ S2, const float* __restrict__ v,
                                                  const float* u_prev, float* u_out, int* err) {
    const int lane = threadIdx.x & 31;
    const long gw = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (gw >= (long)g.BH * g.Lrq) return;
    const int bh = (int)(gw / g.Lrq), i = (int)(gw % g.Lrq);
    const float* vv = v + (size_t)bh * g.Lrk;
    float* uo = u_out + (size_t)bh * g.Lrq;
    if (!row_on(g, bh, i)) {
        if (lane == 0) uo[i] = 0.f;
        return;
    }
    const int n = row_ncells(g, i);
    float off;
    if (kFirst) {
        float m = -INFINITY;
        for (int k = lane; k < n; k += 32) {
            int j;
            float s2;
            row_cell(g, S2, bh, i, k, j, s2);
            m = fmaxf(m, s2 + vv[j]);
        }
        off = -warp_max(m);
    } else {
        off = u_prev[(size_t)bh * g.Lrq + i];
    }
    float s = 0.f;
    for (int k = lane; k < n; k += 32) {
        int j;
        float s2;
        row_cell(g, S2, bh, i, k, j, s2);
        s += ex2(s2 + vv[j] + off);
    }
    s = warp_sum(s);
    if (lane == 0) {
        float u = off - lg2(s);
        if (!(s > 0.f) || !isfinite(u)) {
            atomicOr(err, 1);
            u = 0.f;
        }
        uo[i] = u;
    }
}

template <bool kFirst>
__global__ void __launch_bounds__(256) k_col_step(Geo g, const float* __restrict__ S2, const float* __restrict__ u,
                                                  const float* v_prev, float* v_out, int* err) {
    const int lane = threadIdx.x & 31;
    const long gw = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (gw >= (long)g.BH * g.Lrk) return;
    const int bh = (int)(gw / g.Lrk), j = (int)(gw % g.Lrk);
    const float* uu = u + (size_t)bh * g.Lrq;
    float* vo = v_out + (size_t)bh * g.Lrk;
    if (!col_on(g, bh, j)) {
        if (lane == 0) vo[j] = 0.f;
        return;
    }
    const int n = col_ncells(g, j);
    float off;
    if (kFirst) {
        float m = -INFINITY;
        for (int k = lane; k < n; k += 32) {
            int i;
            float s2;
            col_cell(g, S2, bh, j, k, i, s2);
            m = fmaxf(m, s2 + uu[i]);
        }
        off = -warp_max(m);
    } else {
        off = v_prev[(size_t)bh * g.Lrk + j];
    }
    float s = 0.f;
    for (int k = lane; k < n; k += 32) {
        int i;
        float s2;
        col_cell(g, S2, bh, j, k, i, s2);
        s += ex2(s2 + uu[i] + off);
    }
    s = warp_sum(s);
    if (lane == 0) {
        float v = off - lg2(s);
        if (!(s > 0.f) || !isfinite(v)) {
            atomicOr(err, 2);
            v = 0.f;
        }
        vo[j] = v;
    }
}

// ---------------------------------------------------------------------------
// O_i = sum_j P_ij V_j (warp per row; lanes own cells for the exp, then own
// head-dim slices for the accumulation, exchanging p through shuffles).
// ---------------------------------------------------------------------------
template <class TIn>
__global__ void __launch_bounds__(256) k_output(Geo g, const float* __restrict__ S2, const float* __restrict__ u,
                                                const float* __restrict__ v, const TIn* __restrict__ V,
                                                float* __restrict__ O, int last_only) {
    const int lane = threadIdx.x & 31;
    const long gw = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (gw >= (long)g.BH * (last_only ? 1 : g.Lrq)) return;
    const int bh = last_only ? (int)gw : (int)(gw / g.Lrq), i = last_only ? g.Lrq - 1 : (int)(gw % g.Lrq);
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    if (row_on(g, bh, i)) {
        const float ui = u[(size_t)bh * g.Lrq + i];
        const float* vv = v + (size_t)bh * g.Lrk;
        const TIn* Vh = V + (size_t)bh * g.Lrk * g.d;
        const int n = row_ncells(g, i);
        for (int base = 0; base < n; base += 32) {
            const int k = base + lane;
            int j = 0;
            float p = 0.f;
            if (k < n) {
                float s2;
                row_cell(g, S2, bh, i, k, j, s2);
                p = ex2(s2 + ui + vv[j]);
            }
            const int cnt = min(32, n - base);
            for (int t = 0; t < cnt; ++t) {
                const float pt = __shfl_sync(0xffffffffu, p, t);
                const int jt = __shfl_sync(0xffffffffu, j, t);
                if (pt == 0.f) continue;
                const TIn* vr = Vh + (size_t)jt * g.d;
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    const int x = lane + 32 * m;
                    if (x < g.d) acc[m] = fmaf(pt, ldf(vr + x), acc[m]);
                }
            }
        }
    }
    float* orow = O + ((size_t)bh * g.Lrq + i) * g.d;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
        const int x = lane + 32 * m;
        if (x < g.d) orow[x] = acc[m];
    }
}

// Ledger gauges: gauge[r][bh] = mean over active rows of u2 slot r (base 2).
__global__ void __launch_bounds__(256) k_gauges(Geo g, const float* __restrict__ u_slots, int nslots,
                                                float* __restrict__ gauge) {
    const int bh = blockIdx.x, r = blockIdx.y;
    if (r >= nslots) return;
    const float* u = u_slots + ((size_t)r * g.BH + bh) * g.Lrq;
    double s = 0.0;
    int cnt = 0;
    for (int i = threadIdx.x; i < g.Lrq; i += blockDim.x)
        if (row_on(g, bh, i)) {
            s += (double)u[i];
            ++cnt;
        }
    __shared__ double ss[256];
    __shared__ int sc[256];
    ss[threadIdx.x] = s;
    sc[threadIdx.x] = cnt;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            ss[threadIdx.x] += ss[threadIdx.x + o];
            sc[threadIdx.x] += sc[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) gauge[(size_t)r * g.BH + bh] = sc[0] > 0 ? (float)(ss[0] / sc[0]) : 0.f;
}

// ---------------------------------------------------------------------------
// Backward sweeps.  Duals are the raw tail duals (base 2): u1, u2, v0, v1, v2;
// with raw duals every ledger gauge factor g21 = g10 = 1.
//   alpha_i = 2^(u1-u2), beta_j = 2^(v1-v2), delta_j = 2^(v0-v2)
// One-reference:  Sbar = P22 (Z - v2b_j - beta_j u2b_i - alpha_i beta_j v1b_j - alpha_i delta_j u1b_i)
// Direct:         Sbar = P22 Z - P22 v2b_j - u2b_i P21 - P11 v1b_j - u1b_i P10
// ---------------------------------------------------------------------------
template <class TIn>
struct BwdArgs {
    const float* S2;
    const float *u1, *u2, *v0, *v1, *v2;  // slots of the saved state
    float *g_u, *g_v, *u2b, *v1b, *u1b, *v0b;
    const TIn *Q, *K, *V, *dO;
    float *dQ, *dK, *dV, *deps_part;
};

__device__ __forceinline__ float sbar_cell(bool direct, float s2, float u1i, float u2i, float v0j, float v1j,
                                           float v2j, float z, float u2bi, float u1bi, float v2bj, float v1bj) {
    const float p22 = ex2(s2 + u2i + v2j);
    if (p22 == 0.f) return 0.f;
    if (!direct) {
        const float a = ex2(u1i - u2i), b = ex2(v1j - v2j), dl = ex2(v0j - v2j);
        return p22 * (z - v2bj - b * u2bi - a * b * v1bj - a * dl * u1bi);
    }
    const float p21 = ex2(s2 + u2i + v1j), p11 = ex2(s2 + u1i + v1j), p10 = ex2(s2 + u1i + v0j);
    return p22 * z - p22 * v2bj - u2bi * p21 - p11 * v1bj - u1bi * p10;
}

enum { RB_GU = 0, RB_U2B = 1, RB_U1B = 2, RB_DQ = 3 };
enum { CB_GV = 0, CB_V1B = 1, CB_V0B = 2, CB_DK = 3 };

// ---------------------------------------------------------------------------
// The dustbin row / column of the spoke support (full-length lines): each line is split over
// kDustSplit CTAs per head (one cell per thread; vector terms warp-cooperative), partials in a fixed
// order, then one combine CTA per head.  Cell scores are the constant sd2 on active cells and the
// corner; Z of a line cell comes from the precomputed dustbin dots (Zd / ZdT) and the corner dot.
//   row line (own = dustbin row Lq):    RB_GU, RB_U2B, RB_U1B, RB_DQ (d_eps part; dQ_L = 0), kRO (O_L)
//   column line (own = dustbin col Lk): CB_GV (+dV_L), CB_V1B, CB_V0B, CB_DK (dK_L = 0)
// ---------------------------------------------------------------------------
constexpr int kDustSplit = 8;
constexpr int kRO = 9;  // forward transport output of the dustbin row

template <bool kCol, int kOp, bool kDirect, class TIn>
__global__ void __launch_bounds__(256) k_dust_line(Geo g, BwdArgs<TIn> a, const float* __restrict__ Zd,
                                                   const float* __restrict__ ZdT, float* __restrict__ part) {
    __shared__ float wsum[8];
    __shared__ float vsum[8][128];
    const int s = blockIdx.x, bh = blockIdx.y, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int n = kCol ? g.Lq + 1 : g.Lk + 1;  // cells of the line (last = corner)
    const int chunk = (n + kDustSplit - 1) / kDustSplit;
    const int c_lo = s * chunk, c_hi = min(n, c_lo + chunk);
    const size_t ro = (size_t)bh * g.Lrq, co = (size_t)bh * g.Lrk;
    constexpr bool kVecOut = (kOp == kRO) || (kCol && kOp == CB_GV);
    constexpr bool kNeedZ = kCol ? (kOp == CB_GV) : (kOp == RB_GU || kOp == RB_DQ);
    // own duals of the line
    const size_t own = kCol ? co + g.Lk : ro + g.Lq;
    const float o2 = kCol ? a.v2[own] : a.u2[own];
    const float o1 = kCol ? a.v1[own] : a.u1[own];
    const float o0 = kCol ? a.v0[own] : 0.f;
    float zc = 0.f;  // corner dot dO_dustbin . V_dustbin
    if (kNeedZ) {
        for (int x = lane; x < g.d; x += 32) zc += ldf(a.dO + (ro + g.Lq) * g.d + x) * ldf(a.V + (co + g.Lk) * g.d + x);
        zc = warp_sum(zc);
    }
    const float sd2 = g.sd2;
    float acc = 0.f;
    float vacc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int b0 = c_lo + wid * 32; b0 < c_hi; b0 += 256) {
        const int t = b0 + lane;  // other-side index of this lane's cell (t == Lq / Lk: the corner)
        float contrib = 0.f, vw = 0.f;
        if (t < c_hi) {
            const bool corner = kCol ? t == g.Lq : t == g.Lk;
            const bool on = corner || (kCol ? row_on(g, bh, t) : col_on(g, bh, t));
            if (on) {
                if (kCol) {
                    const size_t oi = ro + t;
                    const float u2i = a.u2[oi];
                    const float p = ex2(sd2 + u2i + o2);
                    if (kOp == CB_GV) {
                        const float z = corner ? zc : Zd[(size_t)bh * g.Lqp + t];
                        contrib = p * z;
                        vw = p;
                    } else if (kOp == CB_V1B) {
                        contrib = (kDirect ? ex2(sd2 + u2i + o1) : p) * a.u2b[oi];
                    } else if (kOp == CB_V0B) {
                        const float u1i = a.u1[oi];
                        contrib = (kDirect ? ex2(sd2 + u1i + o0) : p * ex2(u1i - u2i)) * a.u1b[oi];
                    }
                } else {
                    const size_t oj = co + t;
                    const float v2j = a.v2[oj];
                    const float p = ex2(sd2 + o2 + v2j);
                    if (kOp == kRO) {
                        vw = p;
                    } else if (kOp == RB_GU) {
                        contrib = p * (corner ? zc : ZdT[(size_t)bh * g.Lkp + t]);
                    } else if (kOp == RB_U2B) {
                        contrib = p * a.g_v[oj];
                    } else if (kOp == RB_U1B) {
                        const float v1j = a.v1[oj];
                        contrib = (kDirect ? ex2(sd2 + o1 + v1j) : p * ex2(v1j - v2j)) * a.v1b[oj];
                    } else if (kOp == RB_DQ) {
                        const float z = corner ? zc : ZdT[(size_t)bh * g.Lkp + t];
                        const float sb = sbar_cell(kDirect, sd2, o1, o2, a.v0[oj], a.v1[oj], v2j, z, a.u2b[ro + g.Lq],
                                                   a.u1b[ro + g.Lq], a.g_v[oj], a.v1b[oj]);
                        contrib = sb * (sd2 * kLn2);
                    }
                }
            }
        }
        acc += contrib;
        if (kVecOut) {  // vector term: sum over this batch's cells of vw * (V_j | dO_i)
            const TIn* X = kCol ? a.dO + ro * g.d : a.V + co * g.d;
            const int cnt = min(32, c_hi - b0);
            for (int q = 0; q < cnt; ++q) {
                const float wq = __shfl_sync(0xffffffffu, vw, q);
                if (wq == 0.f) continue;
                const TIn* xr = X + (size_t)(b0 + q) * g.d;
#pragma unroll
                for (int m = 0; m < 4; ++m)
                    if (lane + 32 * m < g.d) vacc[m] = fmaf(wq, ldf(xr + lane + 32 * m), vacc[m]);
            }
        }
    }
    acc = warp_sum(acc);
    if (lane == 0) wsum[wid] = acc;
    if (kVecOut) {
#pragma unroll
        for (int m = 0; m < 4; ++m)
            if (lane + 32 * m < g.d) vsum[wid][lane + 32 * m] = vacc[m];
    }
    __syncthreads();
    float* out = part + ((size_t)bh * kDustSplit + s) * 129;
    if (tid == 0) {
        float t = 0.f;
        for (int w = 0; w < 8; ++w) t += wsum[w];
        out[0] = t;
    }
    if (kVecOut && tid < g.d) {
        float t = 0.f;
        for (int w = 0; w < 8; ++w) t += vsum[w][tid];
        out[1 + tid] = t;
    }
}

template <bool kCol, int kOp, bool kDirect, class TIn>
__global__ void __launch_bounds__(128) k_dust_line_fin(Geo g, BwdArgs<TIn> a, const float* __restrict__ part,
                                                       float* __restrict__ O) {
    const int bh = blockIdx.x, tid = threadIdx.x;
    const size_t ro = (size_t)bh * g.Lrq, co = (size_t)bh * g.Lrk;
    const float* pp = part + (size_t)bh * kDustSplit * 129;
    const size_t own = kCol ? co + g.Lk : ro + g.Lq;
    if (tid == 0) {
        float tot = 0.f;
        for (int s = 0; s < kDustSplit; ++s) tot += pp[s * 129];
        if (kCol) {
            if (kOp == CB_GV) a.g_v[own] = tot;
            if (kOp == CB_V1B) a.v1b[own] = kDirect ? -tot : -ex2(a.v1[own] - a.v2[own]) * tot;
            if (kOp == CB_V0B) a.v0b[own] = kDirect ? -tot : -ex2(a.v0[own] - a.v2[own]) * tot;
        } else {
            if (kOp == RB_GU) a.g_u[own] = tot;
            if (kOp == RB_U2B) a.u2b[own] = a.g_u[own] - tot;
            if (kOp == RB_U1B) a.u1b[own] = kDirect ? -tot : -ex2(a.u1[own] - a.u2[own]) * tot;
            if (kOp == RB_DQ) a.deps_part[own] = tot;
        }
    }
    for (int x = tid; x < g.d; x += 128) {
        float v = 0.f;
        if (kOp == kRO || (kCol && kOp == CB_GV))
            for (int s = 0; s < kDustSplit; ++s) v += pp[s * 129 + 1 + x];
        if (kOp == kRO) O[own * g.d + x] = v;
        if (kCol && kOp == CB_GV) a.dV[own * g.d + x] = v;
        if (kCol && kOp == CB_DK) a.dK[own * g.d + x] = 0.f;  // constant cost: no dK of the dustbin key
        if (!kCol && kOp == RB_DQ) a.dQ[own * g.d + x] = 0.f;
    }
}

void add_launches(long long n);

template <bool kCol, int kOp, bool kDirect, class TIn>
static void dust_line(const Geo& g, const BwdArgs<TIn>& a, const float* Zd, const float* ZdT, float* part, float* O,
                      cudaStream_t s) {
    if (!(kCol && kOp == CB_DK))
        k_dust_line<kCol, kOp, kDirect, TIn><<<dim3(kDustSplit, g.BH), 256, 0, s>>>(g, a, Zd, ZdT, part);
    k_dust_line_fin<kCol, kOp, kDirect, TIn><<<g.BH, 128, 0, s>>>(g, a, part, O);
    add_launches(2);
}


template <int kOp, bool kDirect, class TIn>
__global__ void __launch_bounds__(256) k_bwd_row(Geo g, BwdArgs<TIn> a, int last_only) {
    __shared__ float sh_vec[8][128];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const long gw = (long)blockIdx.x * 8 + wid;
    if (gw >= (long)g.BH * (last_only ? 1 : g.Lrq)) return;
    const int bh = last_only ? (int)gw : (int)(gw / g.Lrq), i = last_only ? g.Lrq - 1 : (int)(gw % g.Lrq);
    const size_t ri = (size_t)bh * g.Lrq + i;
    const size_t cbase = (size_t)bh * g.Lrk;
    const bool on = row_on(g, bh, i);
    if (!on) {
        if (lane == 0) {
            if (kOp == RB_GU) a.g_u[ri] = 0.f;
            if (kOp == RB_U2B) a.u2b[ri] = 0.f;
            if (kOp == RB_U1B) a.u1b[ri] = 0.f;
            if (kOp == RB_DQ) a.deps_part[ri] = 0.f;
        }
        if (kOp == RB_DQ)
            for (int x = lane; x < g.d; x += 32) a.dQ[ri * g.d + x] = 0.f;
        return;
    }
    const bool need_z = (kOp == RB_GU || kOp == RB_DQ);
    if (need_z) {
        for (int x = lane; x < g.d; x += 32) sh_vec[wid][x] = ldf(a.dO + ri * g.d + x);
        __syncwarp();
    }
    const float u1i = a.u1[ri], u2i = a.u2[ri];
    const float u2bi = (kOp == RB_DQ) ? a.u2b[ri] : 0.f;
    const float u1bi = (kOp == RB_DQ) ? a.u1b[ri] : 0.f;
    const int n = row_ncells(g, i);
    float sacc = 0.f, dacc = 0.f;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int base = 0; base < n; base += 32) {
        const int k = base + lane;
        int j = 0;
        float s2 = -INFINITY, contrib = 0.f;
        if (k < n) {
            row_cell(g, a.S2, bh, i, k, j, s2);
            const float v2j = a.v2[cbase + j];
            float z = 0.f;
            if (need_z && s2 != -INFINITY) {
                const TIn* vr = a.V + (cbase + j) * g.d;
                for (int x = 0; x < g.d; ++x) z = fmaf(sh_vec[wid][x], ldf(vr + x), z);
            }
            if (kOp == RB_GU) {
                contrib = ex2(s2 + u2i + v2j) * z;
            } else if (kOp == RB_U2B) {
                contrib = ex2(s2 + u2i + v2j) * a.g_v[cbase + j];
            } else if (kOp == RB_U1B) {
                const float v1j = a.v1[cbase + j];
                contrib = kDirect ? ex2(s2 + u1i + v1j) * a.v1b[cbase + j]
                                  : ex2(s2 + u2i + v2j) * ex2(v1j - v2j) * a.v1b[cbase + j];
            } else {  // RB_DQ
                contrib = sbar_cell(kDirect, s2, u1i, u2i, a.v0[cbase + j], a.v1[cbase + j], v2j, z, u2bi, u1bi,
                                    a.g_v[cbase + j], a.v1b[cbase + j]);
                if (contrib != 0.f) dacc += contrib * (s2 * kLn2);
            }
        }
        if (kOp == RB_DQ) {
            // dQ_i += Sbar_ij K_j on QK cells (dustbin cells carry a constant cost)
            const bool qk_cell = (i < g.Lq) && (j < g.Lk);
            const float sb = qk_cell ? contrib : 0.f;
            const int cnt = min(32, n - base);
            for (int t = 0; t < cnt; ++t) {
                const float st_ = __shfl_sync(0xffffffffu, sb, t);
                const int jt = __shfl_sync(0xffffffffu, j, t);
                if (st_ == 0.f) continue;
                const TIn* kr = a.K + (cbase + jt) * g.d;
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    const int x = lane + 32 * m;
                    if (x < g.d) acc[m] = fmaf(st_, ldf(kr + x), acc[m]);
                }
            }
        } else {
            sacc += contrib;
        }
    }
    if (kOp == RB_DQ) {
        dacc = warp_sum(dacc);
        if (lane == 0) a.deps_part[ri] = dacc;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const int x = lane + 32 * m;
            if (x < g.d) a.dQ[ri * g.d + x] = acc[m] * g.inv_qk;
        }
        return;
    }
    sacc = warp_sum(sacc);
    if (lane == 0) {
        if (kOp == RB_GU) a.g_u[ri] = sacc;
        if (kOp == RB_U2B) a.u2b[ri] = a.g_u[ri] - sacc;
        if (kOp == RB_U1B) a.u1b[ri] = kDirect ? -sacc : -ex2(u1i - u2i) * sacc;
    }
}

template <int kOp, bool kDirect, class TIn>
__global__ void __launch_bounds__(256) k_bwd_col(Geo g, BwdArgs<TIn> a, int last_only) {
    __shared__ float sh_vec[8][128];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const long gw = (long)blockIdx.x * 8 + wid;
    if (gw >= (long)g.BH * (last_only ? 1 : g.Lrk)) return;
    const int bh = last_only ? (int)gw : (int)(gw / g.Lrk), j = last_only ? g.Lrk - 1 : (int)(gw % g.Lrk);
    const size_t cj = (size_t)bh * g.Lrk + j;
    const size_t rbase = (size_t)bh * g.Lrq;
    const bool on = col_on(g, bh, j);
    if (!on) {
        if (lane == 0) {
            if (kOp == CB_GV) a.g_v[cj] = 0.f;
            if (kOp == CB_V1B) a.v1b[cj] = 0.f;
            if (kOp == CB_V0B) a.v0b[cj] = 0.f;
        }
        if (kOp == CB_GV)
            for (int x = lane; x < g.d; x += 32) a.dV[cj * g.d + x] = 0.f;
        if (kOp == CB_DK)
            for (int x = lane; x < g.d; x += 32) a.dK[cj * g.d + x] = 0.f;
        return;
    }
    const bool need_z = (kOp == CB_GV || kOp == CB_DK);
    if (need_z) {
        for (int x = lane; x < g.d; x += 32) sh_vec[wid][x] = ldf(a.V + cj * g.d + x);
        __syncwarp();
    }
    const float v0j = a.v0[cj], v1j = a.v1[cj], v2j = a.v2[cj];
    const float v2bj = (kOp == CB_DK) ? a.g_v[cj] : 0.f;
    const float v1bj = (kOp == CB_DK) ? a.v1b[cj] : 0.f;
    const int n = col_ncells(g, j);
    float sacc = 0.f;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int base = 0; base < n; base += 32) {
        const int k = base + lane;
        int i = 0;
        float s2 = -INFINITY, contrib = 0.f, vecw = 0.f;
        if (k < n) {
            col_cell(g, a.S2, bh, j, k, i, s2);
            const float u2i = a.u2[rbase + i];
            float z = 0.f;
            if (need_z && s2 != -INFINITY) {
                const TIn* dr = a.dO + (rbase + i) * g.d;
                for (int x = 0; x < g.d; ++x) z = fmaf(sh_vec[wid][x], ldf(dr + x), z);
            }
            if (kOp == CB_GV) {
                const float p = ex2(s2 + u2i + v2j);
                contrib = p * z;
                vecw = p;
            } else if (kOp == CB_V1B) {
                contrib = (kDirect ? ex2(s2 + u2i + v1j) : ex2(s2 + u2i + v2j)) * a.u2b[rbase + i];
            } else if (kOp == CB_V0B) {
                const float u1i = a.u1[rbase + i];
                contrib = kDirect ? ex2(s2 + u1i + v0j) * a.u1b[rbase + i]
                                  : ex2(s2 + u2i + v2j) * ex2(u1i - u2i) * a.u1b[rbase + i];
            } else {  // CB_DK
                const float sb = sbar_cell(kDirect, s2, a.u1[rbase + i], u2i, v0j, v1j, v2j, z, a.u2b[rbase + i],
                                           a.u1b[rbase + i], v2bj, v1bj);
                vecw = (i < g.Lq && j < g.Lk) ? sb : 0.f;
            }
        }
        if (kOp == CB_GV || kOp == CB_DK) {
            const TIn* src = (kOp == CB_GV) ? a.dO : a.Q;
            const int cnt = min(32, n - base);
            for (int t = 0; t < cnt; ++t) {
                const float wt = __shfl_sync(0xffffffffu, vecw, t);
                const int it = __shfl_sync(0xffffffffu, i, t);
                if (wt == 0.f) continue;
                const TIn* rr = src + (rbase + it) * g.d;
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    const int x = lane + 32 * m;
                    if (x < g.d) acc[m] = fmaf(wt, ldf(rr + x), acc[m]);
                }
            }
        }
        sacc += contrib;
    }
    if (kOp == CB_GV || kOp == CB_DK) {
        float* dst = (kOp == CB_GV) ? a.dV : a.dK;
        const float sc = (kOp == CB_GV) ? 1.f : g.inv_qk;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const int x = lane + 32 * m;
            if (x < g.d) dst[cj * g.d + x] = acc[m] * sc;
        }
        if (kOp == CB_DK) return;
    }
    sacc = warp_sum(sacc);
    if (lane == 0) {
        if (kOp == CB_GV) a.g_v[cj] = sacc;
        if (kOp == CB_V1B) a.v1b[cj] = kDirect ? -sacc : -ex2(v1j - v2j) * sacc;
        if (kOp == CB_V0B) a.v0b[cj] = kDirect ? -sacc : -ex2(v0j - v2j) * sacc;
    }
}

// d_eps[bh] = -(1/eps) * sum_i deps_part[bh][i]  (fixed-order reduction)
__global__ void __launch_bounds__(1024) k_deps_reduce(Geo g, const float* __restrict__ part, float* __restrict__ out,
                                                      int i_begin, int i_end) {
    const int bh = blockIdx.x;
    double s = 0.0;
#pragma unroll 4
    for (int i = i_begin + threadIdx.x; i < i_end; i += 1024) s += (double)part[(size_t)bh * g.Lrq + i];
    __shared__ double ss[1024];
    ss[threadIdx.x] = s;
    __syncthreads();
    for (int o = 512; o > 0; o >>= 1) {
        if (threadIdx.x < o) ss[threadIdx.x] += ss[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[bh] = (float)(-ss[0] / (double)g.eps);
}

// base-2 raw duals -> natural units (eta_v and friends)
__global__ void k_scale(const float* __restrict__ src, float* __restrict__ dst, long n, float s) {
    const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) dst[t] = src[t] * s;
}

// ---------------------------------------------------------------------------
// Launchers
// ---------------------------------------------------------------------------
static thread_local long long g_launches = 0;
void add_launches(long long n) { g_launches += n; }
long long launch_count(bool reset) {
    const long long c = g_launches;
    if (reset) g_launches = 0;
    return c;
}
static inline unsigned nblocks(long items, int per) { return (unsigned)((items + per - 1) / per); }

static size_t scores_smem(const Geo& g, size_t elem) {
    const int ncol = ((kScoreRows + 2 * g.w + 63) / 64) * 64;
    return (size_t)(kScoreRows + ncol) * (g.d + 1) * elem;
}

template <class TIn, class TAcc, bool kZ>
static cudaError_t launch_band_dot(const Geo& g, const void* A, const void* B, float* out, cudaStream_t s) {
    const size_t smem = scores_smem(g, sizeof(float));
    auto kern = k_scores<TIn, TAcc, kZ>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<dim3((g.Lq + kScoreRows - 1) / kScoreRows, g.BH), 256, smem, s>>>(g, (const TIn*)A, (const TIn*)B, out);
    ++g_launches;
    return cudaGetLastError();
}

template <class TIn, bool kZ, int D>
static cudaError_t launch_band_mma(const Geo& g, const void* A, const void* B, float* out, float* outT,
                                   cudaStream_t s) {
    using M = BandMma<D>;
    const size_t smem = M::smem();
    auto kern = k_band_mma<TIn, kZ, D>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<dim3((g.Lq + M::RB - 1) / M::RB, g.BH), 256, smem, s>>>(g, (const TIn*)A, (const TIn*)B, out, outT);
    ++g_launches;
    return cudaGetLastError();
}

// FP64-tensor-core band dot when the head dim has a specialisation
template <bool kZ>
static bool band_mma(const Geo& g, int dtype, const void* A, const void* B, float* out, float* outT, cudaStream_t s,
                     cudaError_t& err) {
    if (getenv("ST_NO_DMMA")) return false;
    if (g.d == 32)
        err = dtype == 0 ? launch_band_mma<float, kZ, 32>(g, A, B, out, outT, s) : launch_band_mma<__nv_bfloat16, kZ, 32>(g, A, B, out, outT, s);
    else if (g.d == 64)
        err = dtype == 0 ? launch_band_mma<float, kZ, 64>(g, A, B, out, outT, s) : launch_band_mma<__nv_bfloat16, kZ, 64>(g, A, B, out, outT, s);
    else if (g.d == 128)
        err = dtype == 0 ? launch_band_mma<float, kZ, 128>(g, A, B, out, outT, s) : launch_band_mma<__nv_bfloat16, kZ, 128>(g, A, B, out, outT, s);
    else
        return false;
    return true;
}

cudaError_t launch_scores(const Geo& g, int dtype, const void* Q, const void* K, float* S2, cudaStream_t s) {
    cudaError_t e = cudaSuccess;
    if (band_mma<false>(g, dtype, Q, K, S2, nullptr, s, e)) return e;
    return dtype == 0 ? launch_band_dot<float, double, false>(g, Q, K, S2, s)
                      : launch_band_dot<__nv_bfloat16, float, false>(g, Q, K, S2, s);
}

// transposed-band cells whose row i lies outside [0, Lqp): no row block produces them
__global__ void k_fillT_edges(Geo g, float* __restrict__ outT, float fill) {
    const int bh = blockIdx.y;
    const int e = blockIdx.x * blockDim.x + threadIdx.x;  // over 2 * min(w, Lkp) rows x Wf
    const int ne = min(g.w, g.Lkp);
    if (e >= 2 * ne * g.Wf) return;
    const int rr = e / g.Wf, kp = e % g.Wf;
    const int j = rr < ne ? rr : g.Lkp - 2 * ne + rr;
    const int i = j - g.w + kp;
    if (i < 0 || i >= g.Lqp) outT[((size_t)bh * g.Lkp + j) * g.Wf + kp] = fill;
}

bool band_dual_supported(const Geo& g) {
    return g.Lq == g.Lk && (g.d == 32 || g.d == 64 || g.d == 128) && !getenv("ST_NO_DMMA") && !getenv("ST_NO_DUAL");
}

// band + its transpose in one pass (band_dual_supported)
cudaError_t launch_band_dual(const Geo& g, int dtype, bool z, const void* A, const void* B, float* out, float* outT,
                             cudaStream_t s) {
    cudaError_t e = cudaSuccess;
    const bool ok = z ? band_mma<true>(g, dtype, A, B, out, outT, s, e) : band_mma<false>(g, dtype, A, B, out, outT, s, e);
    if (!ok) return cudaErrorNotSupported;
    if (e != cudaSuccess) return e;
    return cudaGetLastError();  // edge cells of the transposed band: filled by k_band_mma's end blocks
}

cudaError_t launch_zband(const Geo& g, int dtype, const void* dO, const void* V, float* Z, cudaStream_t s) {
    cudaError_t e = cudaSuccess;
    if (band_mma<true>(g, dtype, dO, V, Z, nullptr, s, e)) return e;
    return dtype == 0 ? launch_band_dot<float, float, true>(g, dO, V, Z, s)
                      : launch_band_dot<__nv_bfloat16, float, true>(g, dO, V, Z, s);
}

cudaError_t launch_row_step(const Geo& g, bool first, const float* S2, const float* v, const float* u_prev,
                            float* u_out, int* err, cudaStream_t s) {
    const unsigned nb = nblocks((long)g.BH * g.Lrq, 8);
    if (first) k_row_step<true><<<nb, 256, 0, s>>>(g, S2, v, u_prev, u_out, err);
    else k_row_step<false><<<nb, 256, 0, s>>>(g, S2, v, u_prev, u_out, err);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_transpose_band(const Geo& g, const float* S2, float* S2T, cudaStream_t s, float fill) {
    const long total = (long)g.BH * g.Lkp * g.Wf;
    k_transpose_band<<<nblocks(total, 256), 256, 0, s>>>(g, S2, S2T, fill);
    ++g_launches;
    return cudaGetLastError();
}

size_t stepT_smem_bytes(const Geo& g) { return (size_t)128 * g.Wf * 4 + (size_t)(128 + 2 * g.w) * 4 + 16; }

cudaError_t launch_stepT(const Geo& g, bool first, const float* S2, const float* dual_other, const float* off_own,
                         float* out_own, int* err, cudaStream_t s) {
    const size_t smem = stepT_smem_bytes(g);
    auto k = first ? k_stepT<true> : k_stepT<false>;
    static size_t set_true = 0, set_false = 0;
    size_t& cur = first ? set_true : set_false;
    if (smem > cur) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        cur = smem;
    }
    // dustbin problems: one more CTA column computes the own dustbin dual in the same launch
    k<<<dim3((g.Lq + 127) / 128 + (g.dustbin ? 1 : 0), g.BH), 128, smem, s>>>(g, S2, dual_other, off_own, out_own, err);
    ++g_launches;
    return cudaGetLastError();
}

size_t fstep_smem_bytes(const Geo& g) {
    if (g.w > 128) return SIZE_MAX;  // <= 5 contributing blocks per column, <= kFsCols columns per thread
    return (size_t)128 * g.Wf * 4 + (size_t)(128 + 2 * g.w) * 4;
}

cudaError_t launch_fstep(const Geo& g, int t, const FStepPtrs& p, cudaStream_t s) {
    FStep f;
    f.S2 = p.S2;
    f.u_prev = p.u_prev;
    f.u_out = p.u_out;
    f.v_pp = p.v_pp;
    f.v_p_out = p.v_p_out;
    f.v_p_slot = p.v_p_slot;
    f.part_in = p.part_in;
    f.partm_in = p.partm_in;
    f.part_out = p.part_out;
    f.partm_out = p.partm_out;
    f.NB = (g.Lq + 127) / 128;
    f.Nw = 128 + 2 * g.w;
    f.err = p.err;
    const size_t smem = fstep_smem_bytes(g);
    auto k = (t == 1) ? k_fstep<true, false> : (t == 2) ? k_fstep<false, true> : k_fstep<false, false>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<dim3(f.NB, g.BH), kFsThreads, smem, s>>>(g, f);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_ffinal(const Geo& g, int t_last, const FStepPtrs& p, cudaStream_t s) {
    FStep f{};
    f.v_pp = p.v_pp;
    f.v_p_out = p.v_p_out;
    f.v_p_slot = p.v_p_slot;
    f.part_in = p.part_in;
    f.partm_in = p.partm_in;
    f.NB = (g.Lq + 127) / 128;
    f.Nw = 128 + 2 * g.w;
    f.err = p.err;
    const unsigned nb = nblocks((long)g.BH * g.Lk, 256);
    if (t_last == 1) k_ffinal<true><<<nb, 256, 0, s>>>(g, f);
    else k_ffinal<false><<<nb, 256, 0, s>>>(g, f);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_col_step(const Geo& g, bool first, const float* S2, const float* u, const float* v_prev,
                            float* v_out, int* err, cudaStream_t s) {
    const unsigned nb = nblocks((long)g.BH * g.Lrk, 8);
    if (first) k_col_step<true><<<nb, 256, 0, s>>>(g, S2, u, v_prev, v_out, err);
    else k_col_step<false><<<nb, 256, 0, s>>>(g, S2, u, v_prev, v_out, err);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_output(const Geo& g, int dtype, const float* S2, const float* u, const float* v, const void* V,
                          float* O, cudaStream_t s, int last_only, float* dpart) {
    if (last_only && dpart != nullptr && g.d <= 128) {  // the dustbin row: split line kernel
        auto go = [&](auto tag) {
            using TIn = decltype(tag);
            BwdArgs<TIn> a{};
            a.u1 = a.u2 = u;
            a.v0 = a.v1 = a.v2 = v;
            a.V = (const TIn*)V;
            dust_line<false, kRO, false, TIn>(g, a, nullptr, nullptr, dpart, O, s);
        };
        if (dtype == 0) go(float{});
        else go(__nv_bfloat16{});
        return cudaGetLastError();
    }
    const unsigned nb = nblocks((long)g.BH * (last_only ? 1 : g.Lrq), 8);
    if (dtype == 0) k_output<float><<<nb, 256, 0, s>>>(g, S2, u, v, (const float*)V, O, last_only);
    else k_output<__nv_bfloat16><<<nb, 256, 0, s>>>(g, S2, u, v, (const __nv_bfloat16*)V, O, last_only);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_gauges(const Geo& g, const float* u_slots, int nslots, float* gauge, cudaStream_t s) {
    k_gauges<<<dim3(g.BH, 3), 256, 0, s>>>(g, u_slots, nslots, gauge);
    ++g_launches;
    return cudaGetLastError();
}

template <class TIn>
static cudaError_t run_backward_t(const Geo& g, const BwdPtrs& p, bool direct, cudaStream_t s) {
    BwdArgs<TIn> a;
    a.S2 = p.S2;
    a.u1 = p.u1;
    a.u2 = p.u2;
    a.v0 = p.v0;
    a.v1 = p.v1;
    a.v2 = p.v2;
    a.g_u = p.g_u;
    a.g_v = p.g_v;
    a.u2b = p.u2b;
    a.v1b = p.v1b;
    a.u1b = p.u1b;
    a.v0b = p.v0b;
    a.Q = (const TIn*)p.Q;
    a.K = (const TIn*)p.K;
    a.V = (const TIn*)p.V;
    a.dO = (const TIn*)p.dO;
    a.dQ = p.dQ;
    a.dK = p.dK;
    a.dV = p.dV;
    a.deps_part = p.deps_part;
    const unsigned nr = nblocks((long)g.BH * g.Lrq, 8), nc = nblocks((long)g.BH * g.Lrk, 8);
    cudaError_t e;
#define ST_CHECK_LAUNCH()                        \
    do {                                         \
        ++g_launches;                            \
        if ((e = cudaGetLastError()) != cudaSuccess) return e; \
    } while (0)
    k_bwd_row<RB_GU, false, TIn><<<nr, 256, 0, s>>>(g, a, 0);
    ST_CHECK_LAUNCH();
    k_bwd_col<CB_GV, false, TIn><<<nc, 256, 0, s>>>(g, a, 0);
    ST_CHECK_LAUNCH();
    k_bwd_row<RB_U2B, false, TIn><<<nr, 256, 0, s>>>(g, a, 0);
    ST_CHECK_LAUNCH();
    if (direct) {
        k_bwd_col<CB_V1B, true, TIn><<<nc, 256, 0, s>>>(g, a, 0);
        ST_CHECK_LAUNCH();
        k_bwd_row<RB_U1B, true, TIn><<<nr, 256, 0, s>>>(g, a, 0);
        ST_CHECK_LAUNCH();
        k_bwd_col<CB_V0B, true, TIn><<<nc, 256, 0, s>>>(g, a, 0);
        ST_CHECK_LAUNCH();
        k_bwd_row<RB_DQ, true, TIn><<<nr, 256, 0, s>>>(g, a, 0);
        ST_CHECK_LAUNCH();
        k_bwd_col<CB_DK, true, TIn><<<nc, 256, 0, s>>>(g, a, 0);
        ST_CHECK_LAUNCH();
    } else {
        k_bwd_col<CB_V1B, false, TIn><<<nc, 256, 0, s>>>(g, a, 0);
        ST_CHECK_LAUNCH();
        k_bwd_row<RB_U1B, false, TIn><<<nr, 256, 0, s>>>(g, a, 0);
        ST_CHECK_LAUNCH();
        k_bwd_col<CB_V0B, false, TIn><<<nc, 256, 0, s>>>(g, a, 0);
        ST_CHECK_LAUNCH();
        k_bwd_row<RB_DQ, false, TIn><<<nr, 256, 0, s>>>(g, a, 0);
        ST_CHECK_LAUNCH();
        k_bwd_col<CB_DK, false, TIn><<<nc, 256, 0, s>>>(g, a, 0);
        ST_CHECK_LAUNCH();
    }
#undef ST_CHECK_LAUNCH
    return cudaSuccess;
}

template <class TIn>
static BwdArgs<TIn> bwd_args(const BwdPtrs& p) {
    BwdArgs<TIn> a;
    a.S2 = p.S2;
    a.u1 = p.u1;
    a.u2 = p.u2;
    a.v0 = p.v0;
    a.v1 = p.v1;
    a.v2 = p.v2;
    a.g_u = p.g_u;
    a.g_v = p.g_v;
    a.u2b = p.u2b;
    a.v1b = p.v1b;
    a.u1b = p.u1b;
    a.v0b = p.v0b;
    a.Q = (const TIn*)p.Q;
    a.K = (const TIn*)p.K;
    a.V = (const TIn*)p.V;
    a.dO = (const TIn*)p.dO;
    a.dQ = p.dQ;
    a.dK = p.dK;
    a.dV = p.dV;
    a.deps_part = p.deps_part;
    return a;
}

template <class TIn, bool kD>
static cudaError_t dust_stage_t(const Geo& g, const BwdPtrs& p, int stage, cudaStream_t s) {
    const BwdArgs<TIn> a = bwd_args<TIn>(p);
    if (p.dpart != nullptr && g.d <= 128) {  // split line kernels
        switch (stage) {
            case 0:
                dust_line<false, RB_GU, kD, TIn>(g, a, p.Zd, p.ZdT, p.dpart, nullptr, s);
                dust_line<true, CB_GV, kD, TIn>(g, a, p.Zd, p.ZdT, p.dpart, nullptr, s);
                break;
            case 1: dust_line<false, RB_U2B, kD, TIn>(g, a, p.Zd, p.ZdT, p.dpart, nullptr, s); break;
            case 2: dust_line<true, CB_V1B, kD, TIn>(g, a, p.Zd, p.ZdT, p.dpart, nullptr, s); break;
            case 3: dust_line<false, RB_U1B, kD, TIn>(g, a, p.Zd, p.ZdT, p.dpart, nullptr, s); break;
            case 4: dust_line<true, CB_V0B, kD, TIn>(g, a, p.Zd, p.ZdT, p.dpart, nullptr, s); break;
            default:
                dust_line<false, RB_DQ, kD, TIn>(g, a, p.Zd, p.ZdT, p.dpart, nullptr, s);
                dust_line<true, CB_DK, kD, TIn>(g, a, p.Zd, p.ZdT, p.dpart, nullptr, s);
        }
        return cudaGetLastError();
    }
    const unsigned nb = nblocks(g.BH, 8);
    switch (stage) {
        case 0:
            k_bwd_row<RB_GU, kD, TIn><<<nb, 256, 0, s>>>(g, a, 1);
            k_bwd_col<CB_GV, kD, TIn><<<nb, 256, 0, s>>>(g, a, 1);
            g_launches += 2;
            break;
        case 1: k_bwd_row<RB_U2B, kD, TIn><<<nb, 256, 0, s>>>(g, a, 1); ++g_launches; break;
        case 2: k_bwd_col<CB_V1B, kD, TIn><<<nb, 256, 0, s>>>(g, a, 1); ++g_launches; break;
        case 3: k_bwd_row<RB_U1B, kD, TIn><<<nb, 256, 0, s>>>(g, a, 1); ++g_launches; break;
        case 4: k_bwd_col<CB_V0B, kD, TIn><<<nb, 256, 0, s>>>(g, a, 1); ++g_launches; break;
        default:
            k_bwd_row<RB_DQ, kD, TIn><<<nb, 256, 0, s>>>(g, a, 1);
            k_bwd_col<CB_DK, kD, TIn><<<nb, 256, 0, s>>>(g, a, 1);
            g_launches += 2;
    }
    return cudaGetLastError();
}

cudaError_t launch_backward_dustbin_stage(const Geo& g, int dtype, const BwdPtrs& p, bool direct, int stage,
                                          cudaStream_t s) {
    if (dtype == 0) return direct ? dust_stage_t<float, true>(g, p, stage, s) : dust_stage_t<float, false>(g, p, stage, s);
    return direct ? dust_stage_t<__nv_bfloat16, true>(g, p, stage, s)
                  : dust_stage_t<__nv_bfloat16, false>(g, p, stage, s);
}

cudaError_t launch_backward(const Geo& g, int dtype, const BwdPtrs& p, bool direct, cudaStream_t s) {
    return dtype == 0 ? run_backward_t<float>(g, p, direct, s) : run_backward_t<__nv_bfloat16>(g, p, direct, s);
}

cudaError_t launch_deps_reduce(const Geo& g, const float* part, float* out, cudaStream_t s, int i_begin, int i_end) {
    if (i_end < 0) i_end = g.Lrq;
    k_deps_reduce<<<g.BH, 1024, 0, s>>>(g, part, out, i_begin, i_end);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_scale(const float* src, float* dst, long n, float sc, cudaStream_t s) {
    k_scale<<<nblocks(n, 256), 256, 0, s>>>(src, dst, n, sc);
    ++g_launches;
    return cudaGetLastError();
}

}  // namespace st
