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
#include <cstdio>

#include "st_common.cuh"
#include "st_kernels.cuh"
#include "st_sm100.cuh"

namespace st {

// ---------------------------------------------------------------------------
// Scores: S2[bh][i][k] for j = i - w + k.  One CTA = 64 query rows x one head;
// the key window [i0-w, i0+63+w] streams through shared memory in 64-row
// chunks.  fp32 inputs accumulate in f64 (products of floats are exact in
// f64), so the stored score is the correctly rounded fp32 value; bf16 inputs
// accumulate in fp32 (bf16 products are exact in fp32), the tensor-core
// contract.
// ---------------------------------------------------------------------------
constexpr int kScoreRows = 64;
constexpr int kScoreChunk = 64;

template <class TIn, bool kF64Acc, bool kZ>
__global__ void __launch_bounds__(256) k_scores(Geo g, const TIn* __restrict__ Q, const TIn* __restrict__ K,
                                                float* __restrict__ S2) {
    // kZ: the output-cotangent band Z_ij = dO_i . V_j (Q := dO, K := V), unscaled, 0 off support
    extern __shared__ float smem[];
    const int dp = g.d + 1;  // padded row pitch: conflict-free column walks
    float* sq = smem;                          // [64][dp]
    float* sk = smem + kScoreRows * dp;        // [64][dp]
    const int bh = blockIdx.y;
    const int i0 = blockIdx.x * kScoreRows;
    const int tid = threadIdx.x;
    const TIn* Qh = Q + (size_t)bh * g.Lrq * g.d;
    const TIn* Kh = K + (size_t)bh * g.Lrk * g.d;
    for (int e = tid; e < kScoreRows * g.d; e += blockDim.x) {
        const int r = e / g.d, x = e % g.d;
        sq[r * dp + x] = (i0 + r < g.Lq) ? ldf(Qh + (size_t)(i0 + r) * g.d + x) : 0.f;
    }
    const int jlo = max(0, i0 - g.w), jhi = min(g.Lk - 1, i0 + kScoreRows - 1 + g.w);
    const int r = tid >> 2;          // 4 threads per row
    const int i = i0 + r;
    const bool row_ok = i < g.Lq && row_on(g, bh, i);
    for (int c0 = jlo; c0 <= jhi; c0 += kScoreChunk) {
        __syncthreads();
        for (int e = tid; e < kScoreChunk * g.d; e += blockDim.x) {
            const int rr = e / g.d, x = e % g.d;
            sk[rr * dp + x] = (c0 + rr <= jhi) ? ldf(Kh + (size_t)(c0 + rr) * g.d + x) : 0.f;
        }
        __syncthreads();
        if (!row_ok) continue;
        for (int c = (tid & 3); c < kScoreChunk; c += 4) {
            const int j = c0 + c;
            if (j > jhi || j < i - g.w || j > i + g.w || !col_on(g, bh, j)) continue;
            const float* qa = sq + r * dp;
            const float* kb = sk + c * dp;
            float val;
            if (kF64Acc) {
                double acc = 0.0;
                for (int x = 0; x < g.d; ++x) acc = fma((double)qa[x], (double)kb[x], acc);
                val = kZ ? (float)acc : (float)(acc * (double)g.c2);
            } else {
                float acc = 0.f;
                for (int x = 0; x < g.d; ++x) acc = fmaf(qa[x], kb[x], acc);
                val = kZ ? acc : acc * g.c2;
            }
            S2[((size_t)bh * g.Lqp + i) * g.Wf + (j - i + g.w)] = val;
        }
    }
    // off-support cells of this CTA's rows -> -inf (disjoint from the cells written above)
    for (int e = tid; e < kScoreRows * g.Wf; e += blockDim.x) {
        const int rr = e / g.Wf, k = e % g.Wf;
        const int ii = i0 + rr;
        if (ii >= g.Lq) continue;
        const int j = ii - g.w + k;
        const bool on = row_on(g, bh, ii) && j >= 0 && j < g.Lk && col_on(g, bh, j);
        if (!on) S2[((size_t)bh * g.Lqp + ii) * g.Wf + k] = kZ ? 0.f : -INFINITY;
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
                                                float* __restrict__ O) {
    const int lane = threadIdx.x & 31;
    const long gw = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (gw >= (long)g.BH * g.Lrq) return;
    const int bh = (int)(gw / g.Lrq), i = (int)(gw % g.Lrq);
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
__global__ void __launch_bounds__(256) k_deps_reduce(Geo g, const float* __restrict__ part, float* __restrict__ out) {
    const int bh = blockIdx.x;
    double s = 0.0;
    for (int i = threadIdx.x; i < g.Lrq; i += blockDim.x) s += (double)part[(size_t)bh * g.Lrq + i];
    __shared__ double ss[256];
    ss[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
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

cudaError_t launch_scores(const Geo& g, int dtype, const void* Q, const void* K, float* S2, cudaStream_t s) {
    const size_t smem = (size_t)2 * kScoreRows * (g.d + 1) * sizeof(float);
    dim3 grid((g.Lq + kScoreRows - 1) / kScoreRows, g.BH);
    if (dtype == 0) {
        auto kern = k_scores<float, true, false>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<grid, 256, smem, s>>>(g, (const float*)Q, (const float*)K, S2);
    } else {
        auto kern = k_scores<__nv_bfloat16, false, false>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<grid, 256, smem, s>>>(g, (const __nv_bfloat16*)Q, (const __nv_bfloat16*)K, S2);
    }
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_zband(const Geo& g, int dtype, const void* dO, const void* V, float* Z, cudaStream_t s) {
    const size_t smem = (size_t)2 * kScoreRows * (g.d + 1) * sizeof(float);
    dim3 grid((g.Lq + kScoreRows - 1) / kScoreRows, g.BH);
    if (dtype == 0) {
        auto kern = k_scores<float, false, true>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<grid, 256, smem, s>>>(g, (const float*)dO, (const float*)V, Z);
    } else {
        auto kern = k_scores<__nv_bfloat16, false, true>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<grid, 256, smem, s>>>(g, (const __nv_bfloat16*)dO, (const __nv_bfloat16*)V, Z);
    }
    ++g_launches;
    return cudaGetLastError();
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
    k<<<dim3((g.Lq + 127) / 128, g.BH), 128, smem, s>>>(g, S2, dual_other, off_own, out_own, err);
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
                          float* O, cudaStream_t s) {
    const unsigned nb = nblocks((long)g.BH * g.Lrq, 8);
    if (dtype == 0) k_output<float><<<nb, 256, 0, s>>>(g, S2, u, v, (const float*)V, O);
    else k_output<__nv_bfloat16><<<nb, 256, 0, s>>>(g, S2, u, v, (const __nv_bfloat16*)V, O);
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

cudaError_t launch_deps_reduce(const Geo& g, const float* part, float* out, cudaStream_t s) {
    k_deps_reduce<<<g.BH, 256, 0, s>>>(g, part, out);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_scale(const float* src, float* dst, long n, float sc, cudaStream_t s) {
    k_scale<<<nblocks(n, 256), 256, 0, s>>>(src, dst, n, sc);
    ++g_launches;
    return cudaGetLastError();
}

}  // namespace st
