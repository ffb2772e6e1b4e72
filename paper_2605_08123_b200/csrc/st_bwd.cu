// st_bwd.cu -- tile kernels of the exact R=2 adjoint on the stored bands
// (r2_backward, adjoint.hpp:232-373).
//
// Stages (one launch each; row stages own 128 query rows per CTA over the score
// band S2 and the cotangent band Z, column stages own 128 key columns per CTA
// over the transposed bands S2T / ZT, so every reduction is in-thread):
//   R1  g_u_i  = sum_j P22 Z                      C1  g_v_j = sum_i P22 Z,  dV_j = sum_i P22 dO_i
//   R2  u2b_i  = g_u_i - sum_j P22 g_v_j          C3  v1b_j = -beta_j sum_i P22 u2b_i
//   R4  u1b_i  = -alpha_i sum_j P22 beta_j v1b_j  C5  v0b_j = -delta_j sum_i P22 alpha_i u1b_i
//   R6  dQ_i   = inv sum_j Sbar K_j, d_eps part   C6  dK_j  = inv sum_i Sbar Q_i
// one-reference:  Sbar = P22 (Z - v2b_j - beta_j u2b_i - alpha_i beta_j v1b_j - alpha_i delta_j u1b_i)
// (adjoint.hpp:202-226; raw duals, so every ledger gauge factor is 1), or the
// direct four-plan form (adjoint.hpp:349-361) for the ablation.
// The band tile of each CTA is contiguous in memory and arrives with one 1-D
// bulk async copy per band; window vectors and operand rows are staged beside it.
// The dustbin row / column (full-length reductions) run in the generic kernels.
#include <type_traits>

#include "st_common.cuh"
#include "st_kernels.cuh"
#include "st_sm100.cuh"

namespace st {

namespace {

template <class TIn>
struct BT {
    const float *S2, *S2T, *Z, *ZT;
    const float *Zd, *ZdT;                // dO_i . V_dustbin [BH][Lqp], dO_dustbin . V_j [BH][Lkp]
    const float *u1, *u2, *v0, *v1, *v2;  // raw tail duals (base 2)
    float *g_u, *g_v, *u2b, *v1b, *u1b, *v0b;
    const TIn *Q, *K, *V, *dO;
    float *dQ, *dK, *dV, *deps_part;
    float* O;  // transport output (RO)
};

enum { R1 = 0, R2 = 1, R4 = 2, R6 = 3, RO = 4, C1 = 10, C3 = 11, C5 = 12, C6 = 13 };

__device__ __forceinline__ float sbar_of(bool direct, float s2, float p22, float z, float u1i, float u2i,
                                         float v0j, float v1j, float v2j, float u2bi, float u1bi, float v2bj,
                                         float v1bj) {
    if (p22 == 0.f) return 0.f;
    if (!direct) {
        const float a = ex2(u1i - u2i), b = ex2(v1j - v2j), dl = ex2(v0j - v2j);
        return p22 * (z - v2bj - b * u2bi - a * b * v1bj - a * dl * u1bi);
    }
    const float p21 = ex2(s2 + u2i + v1j), p11 = ex2(s2 + u1i + v1j), p10 = ex2(s2 + u1i + v0j);
    return p22 * z - p22 * v2bj - u2bi * p21 - p11 * v1bj - u1bi * p10;
}

}  // namespace

// smem: [tile S | tile Z (opt) | nvec window vectors x Nw | operand rows Nw x (D+4)]
template <int kOp, bool kDirect, int D, class TIn>
__global__ void __launch_bounds__(128) k_bwdT(Geo g, BT<TIn> a) {
    extern __shared__ __align__(16) float smf[];
    __shared__ __align__(8) uint64_t bar;
    constexpr bool kRow = kOp < 10;
    constexpr bool kNeedZ = (kOp == R1 || kOp == R6 || kOp == C1 || kOp == C6);
    constexpr bool kVec = (kOp == R6 || kOp == C1 || kOp == C6 || kOp == RO);
    // own = rows (row stages) or columns (column stages)
    const int Lo = kRow ? g.Lq : g.Lk, Lx = kRow ? g.Lk : g.Lq;
    const int Lro = kRow ? g.Lrq : g.Lrk, Lrx = kRow ? g.Lrk : g.Lrq;
    const int Lpo = kRow ? g.Lqp : g.Lkp;
    const uint8_t* mo = kRow ? g.row_mask : g.col_mask;
    const uint8_t* mx = kRow ? g.col_mask : g.row_mask;
    const int bh = blockIdx.y, i0 = blockIdx.x * 128, r = threadIdx.x, i = i0 + r;
    const size_t bo = (size_t)bh * Lro, bx = (size_t)bh * Lrx;
    auto on_o = [&](int k) { return k < Lo && (mo == nullptr || mo[(size_t)(bh / g.H) * Lo + k] != 0); };
    auto on_x = [&](int k) { return k >= 0 && k < Lx && (mx == nullptr || mx[(size_t)(bh / g.H) * Lx + k] != 0); };
    const bool active = on_o(i);

    if (!__syncthreads_or(active)) {
        if (i < Lo) {
            if (kOp == R1) a.g_u[bo + i] = 0.f;
            if (kOp == R2) a.u2b[bo + i] = 0.f;
            if (kOp == R4) a.u1b[bo + i] = 0.f;
            if (kOp == R6) a.deps_part[bo + i] = 0.f;
            if (kOp == C1) a.g_v[bo + i] = 0.f;
            if (kOp == C3) a.v1b[bo + i] = 0.f;
            if (kOp == C5) a.v0b[bo + i] = 0.f;
            float* vo = kOp == R6 ? a.dQ : kOp == C1 ? a.dV : kOp == C6 ? a.dK : kOp == RO ? a.O : nullptr;
            if (kVec)
                for (int x = 0; x < g.d; ++x) vo[(bo + i) * g.d + x] = 0.f;
        }
        return;
    }
    const int Wf = g.Wf, Nw = 128 + 2 * g.w;
    float* tS = smf;
    float* tZ = tS + 128 * Wf;
    float* wv = tZ + (kNeedZ ? 128 * Wf : 0);  // window vectors [nvec][Nw]
    constexpr int nvec = 5;
    float* ops = wv + ((nvec * Nw + 3) & ~3);  // operand rows [Nw][D + 4], 16-byte aligned
    if (threadIdx.x == 0) {
        sm100::mbar_init(&bar, 1);
        sm100::fence_mbar_init();
    }
    __syncthreads();
    const uint32_t tb = 128u * (uint32_t)Wf * 4u;
    if (threadIdx.x == 0) {
        sm100::mbar_arrive_expect_tx(&bar, kNeedZ ? 2 * tb : tb);
        const size_t off = ((size_t)bh * Lpo + i0) * Wf;
        sm100::bulk_g2s(tS, (kRow ? a.S2 : a.S2T) + off, tb, &bar);
        if (kNeedZ) sm100::bulk_g2s(tZ, (kRow ? a.Z : a.ZT) + off, tb, &bar);
    }
    // window vectors over the other side, index c <-> x = i0 - w + c (0 where invalid:
    // the band tile already carries -inf scores there, so P = 0 and no 0*inf appears)
    for (int c = threadIdx.x; c < Nw; c += 128) {
        const int x = i0 - g.w + c;
        const bool ok = on_x(x);
        float w0 = 0.f, w1 = 0.f, w2 = 0.f, w3 = 0.f, w4 = 0.f;
        if (ok) {
            if (kRow) {  // columns: v2, v1, v0, g_v(=v2b), v1b
                w0 = a.v2[bx + x];
                w1 = a.v1[bx + x];
                w2 = a.v0[bx + x];
                if (kOp == R2 || kOp == R6) w3 = a.g_v[bx + x];
                if (kOp == R4 || kOp == R6) w4 = a.v1b[bx + x];
            } else {  // rows: u2, u1, u2b, u1b
                w0 = a.u2[bx + x];
                w1 = a.u1[bx + x];
                if (kOp == C3 || kOp == C6) w3 = a.u2b[bx + x];
                if (kOp == C5 || kOp == C6) w4 = a.u1b[bx + x];
            }
        }
        wv[c] = w0;
        wv[Nw + c] = w1;
        wv[2 * Nw + c] = w2;
        wv[3 * Nw + c] = w3;
        wv[4 * Nw + c] = w4;
        if (kVec) {
            const TIn* src = (kOp == R6) ? a.K : (kOp == C1) ? a.dO : (kOp == RO) ? a.V : a.Q;
            for (int e = 0; e < D; ++e)
                ops[c * (D + 4) + e] = (x >= 0 && x < Lx && e < g.d) ? ldf(src + (bx + x) * g.d + e) : 0.f;
        }
    }
    __syncthreads();
    sm100::mbar_wait(&bar, 0);
    if (i >= Lo) return;
    if (!active) {
        if (kOp == R1) a.g_u[bo + i] = 0.f;
        if (kOp == R2) a.u2b[bo + i] = 0.f;
        if (kOp == R4) a.u1b[bo + i] = 0.f;
        if (kOp == R6) a.deps_part[bo + i] = 0.f;
        if (kOp == C1) a.g_v[bo + i] = 0.f;
        if (kOp == C3) a.v1b[bo + i] = 0.f;
        if (kOp == C5) a.v0b[bo + i] = 0.f;
        float* vo = kOp == R6 ? a.dQ : kOp == C1 ? a.dV : kOp == C6 ? a.dK : kOp == RO ? a.O : nullptr;
        if (kVec)
            for (int x = 0; x < g.d; ++x) vo[(bo + i) * g.d + x] = 0.f;
        return;
    }
    // own-side values
    float o2, o1 = 0.f, o0 = 0.f, ob2 = 0.f, ob1 = 0.f;
    if (kRow) {
        o2 = a.u2[bo + i];
        o1 = a.u1[bo + i];
        if (kOp == R6) {
            ob2 = a.u2b[bo + i];
            ob1 = a.u1b[bo + i];
        }
    } else {
        o2 = a.v2[bo + i];
        o1 = a.v1[bo + i];
        o0 = a.v0[bo + i];
        if (kOp == C6) {
            ob2 = a.g_v[bo + i];
            ob1 = a.v1b[bo + i];
        }
    }
    const float* ts = tS + r * Wf;
    const float* tz = tZ + r * Wf;
    float acc = 0.f, dacc = 0.f;
    float vacc[kVec ? D : 1];
#pragma unroll
    for (int e = 0; e < (kVec ? D : 1); ++e) vacc[e] = 0.f;
    for (int k = 0; k < Wf; ++k) {
        const int c = r + k;
        const float s2 = ts[k];
        if (s2 == -INFINITY) continue;
        const float x2 = wv[c], x1 = wv[Nw + c];
        const float p = ex2(s2 + o2 + x2);
        float wgt = 0.f;
        if (kOp == R1 || kOp == C1) {
            acc += p * tz[k];
            wgt = p;
        } else if (kOp == RO) {
            wgt = p;
        } else if (kOp == R2) {
            acc += p * wv[3 * Nw + c];
        } else if (kOp == R4) {
            acc += kDirect ? ex2(s2 + o1 + x1) * wv[4 * Nw + c] : p * ex2(x1 - x2) * wv[4 * Nw + c];
        } else if (kOp == C3) {
            acc += (kDirect ? ex2(s2 + x2 + o1) : p) * wv[3 * Nw + c];
        } else if (kOp == C5) {
            acc += kDirect ? ex2(s2 + x1 + o0) * wv[4 * Nw + c] : p * ex2(x1 - x2) * wv[4 * Nw + c];
        } else if (kOp == R6) {
            wgt = sbar_of(kDirect, s2, p, tz[k], o1, o2, wv[2 * Nw + c], x1, x2, ob2, ob1, wv[3 * Nw + c],
                          wv[4 * Nw + c]);
            dacc += wgt * (s2 * kLn2);
        } else {  // C6: rows are the window side
            wgt = sbar_of(kDirect, s2, p, tz[k], x1, x2, o0, o1, o2, wv[3 * Nw + c], wv[4 * Nw + c], ob2, ob1);
        }
        if (kVec && wgt != 0.f) {
            const float4* orow = reinterpret_cast<const float4*>(ops + c * (D + 4));
#pragma unroll
            for (int e = 0; e < (kVec ? D / 4 : 0); ++e) {
                const float4 q4 = orow[e];
                vacc[4 * e + 0] = fmaf(wgt, q4.x, vacc[4 * e + 0]);
                vacc[4 * e + 1] = fmaf(wgt, q4.y, vacc[4 * e + 1]);
                vacc[4 * e + 2] = fmaf(wgt, q4.z, vacc[4 * e + 2]);
                vacc[4 * e + 3] = fmaf(wgt, q4.w, vacc[4 * e + 3]);
            }
        }
    }
    // the spoke cell (row i, dustbin column) / (dustbin row, column j)
    if (g.dustbin) {
        const int xd = Lx;  // dustbin index on the other side
        const float s2 = g.sd2;
        const float x2 = kRow ? a.v2[bx + xd] : a.u2[bx + xd];
        const float x1 = kRow ? a.v1[bx + xd] : a.u1[bx + xd];
        const float p = ex2(s2 + o2 + x2);
        const float z = (kOp == RO) ? 0.f : kRow ? a.Zd[(size_t)bh * g.Lqp + i] : a.ZdT[(size_t)bh * g.Lkp + i];
        if (kOp == RO) {  // O_i += p * V_dustbin
#pragma unroll
            for (int e = 0; e < (kVec ? D : 1); ++e) vacc[e] = fmaf(p, ldf(a.V + (bx + xd) * g.d + e), vacc[e]);
        } else if (kOp == R1 || kOp == C1) {
            acc += p * z;
            if (kOp == C1) {  // dV_j += p * dO_dustbin
#pragma unroll
                for (int e = 0; e < (kVec ? D : 1); ++e) vacc[e] = fmaf(p, ldf(a.dO + (bx + xd) * g.d + e), vacc[e]);
            }
        } else if (kOp == R2) {
            acc += p * a.g_v[bx + xd];
        } else if (kOp == R4) {
            acc += kDirect ? ex2(s2 + o1 + x1) * a.v1b[bx + xd] : p * ex2(x1 - x2) * a.v1b[bx + xd];
        } else if (kOp == C3) {
            acc += (kDirect ? ex2(s2 + x2 + o1) : p) * a.u2b[bx + xd];
        } else if (kOp == C5) {
            acc += kDirect ? ex2(s2 + x1 + o0) * a.u1b[bx + xd] : p * ex2(x1 - x2) * a.u1b[bx + xd];
        } else if (kOp == R6) {
            const float sb = sbar_of(kDirect, s2, p, z, o1, o2, a.v0[bx + xd], x1, x2, ob2, ob1, a.g_v[bx + xd],
                                     a.v1b[bx + xd]);
            dacc += sb * (s2 * kLn2);  // constant cost: no dQ contribution
        }
        // C6: no dK contribution from constant-cost cells
    }
    if (kOp == R1) a.g_u[bo + i] = acc;
    if (kOp == C1) a.g_v[bo + i] = acc;
    if (kOp == R2) a.u2b[bo + i] = a.g_u[bo + i] - acc;
    if (kOp == R4) a.u1b[bo + i] = kDirect ? -acc : -ex2(o1 - o2) * acc;
    if (kOp == C3) a.v1b[bo + i] = kDirect ? -acc : -ex2(o1 - o2) * acc;
    if (kOp == C5) a.v0b[bo + i] = kDirect ? -acc : -ex2(o0 - o2) * acc;
    if (kOp == R6) a.deps_part[bo + i] = dacc;
    if (kVec) {
        float* vo = kOp == R6 ? a.dQ : kOp == C1 ? a.dV : kOp == RO ? a.O : a.dK;
        const float sc = (kOp == C1 || kOp == RO) ? 1.f : g.inv_qk;
#pragma unroll
        for (int e = 0; e < (kVec ? D : 1); ++e) vo[(bo + i) * g.d + e] = vacc[e] * sc;
    }
}

// Zd_i = dO_i . V_dustbin (rows) and ZdT_j = dO_dustbin . V_j (columns)
template <class TIn>
__global__ void k_dust_dots(Geo g, const TIn* __restrict__ dO, const TIn* __restrict__ V, float* Zd, float* ZdT) {
    const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const long nq = (long)g.BH * g.Lq, nk = (long)g.BH * g.Lk;
    if (t < nq) {
        const int bh = (int)(t / g.Lq), i = (int)(t % g.Lq);
        const TIn* a = dO + ((size_t)bh * g.Lrq + i) * g.d;
        const TIn* b = V + ((size_t)bh * g.Lrk + g.Lk) * g.d;
        float s = 0.f;
        for (int x = 0; x < g.d; ++x) s = fmaf(ldf(a + x), ldf(b + x), s);
        Zd[(size_t)bh * g.Lqp + i] = s;
    } else if (t < nq + nk) {
        const long u = t - nq;
        const int bh = (int)(u / g.Lk), j = (int)(u % g.Lk);
        const TIn* a = dO + ((size_t)bh * g.Lrq + g.Lq) * g.d;
        const TIn* b = V + ((size_t)bh * g.Lrk + j) * g.d;
        float s = 0.f;
        for (int x = 0; x < g.d; ++x) s = fmaf(ldf(a + x), ldf(b + x), s);
        ZdT[(size_t)bh * g.Lkp + j] = s;
    }
}

// ---------------------------------------------------------------------------
size_t bwdT_smem_bytes(const Geo& g) {
    const int Nw = 128 + 2 * g.w;
    const int D = g.d <= 32 ? 32 : g.d <= 64 ? 64 : 128;
    return (size_t)2 * 128 * g.Wf * 4 + (size_t)((5 * Nw + 3) & ~3) * 4 + (size_t)Nw * (D + 4) * 4 + 64;
}

bool bwdT_supported(const Geo& g) {
    return (g.d == 32 || g.d == 64 || g.d == 128) && bwdT_smem_bytes(g) <= 227 * 1024;
}

template <int kOp, bool kDirect, int D, class TIn>
static cudaError_t run_op(const Geo& g, const BT<TIn>& a, cudaStream_t s) {
    const bool row = kOp < 10;
    const size_t smem = bwdT_smem_bytes(g);
    auto k = k_bwdT<kOp, kDirect, D, TIn>;
    static size_t cur = 0;
    if (smem > cur) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        cur = smem;
    }
    const int n = row ? g.Lq : g.Lk;
    k<<<dim3((n + 127) / 128, g.BH), 128, smem, s>>>(g, a);
    return cudaGetLastError();
}

template <bool kDirect, int D, class TIn>
static cudaError_t run_all(const Geo& g, const BwdPtrs& p, const BwdTPtrs& t, int dtype, cudaStream_t s,
                           long long& launches) {
    BT<TIn> a;
    a.S2 = p.S2;
    a.S2T = t.S2T;
    a.Z = t.Z;
    a.ZT = t.ZT;
    a.Zd = t.Zd;
    a.ZdT = t.ZdT;
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
    cudaError_t e;
#define ST_RUN(op)                                                     \
    do {                                                               \
        if ((e = run_op<op, kDirect, D, TIn>(g, a, s)) != cudaSuccess) return e; \
        ++launches;                                                    \
    } while (0)
#define ST_DUST(stage)                                                                           \
    do {                                                                                         \
        if (g.dustbin) {                                                                         \
            if ((e = launch_backward_dustbin_stage(g, dtype, p, kDirect, stage, s)) != cudaSuccess) return e; \
        }                                                                                        \
    } while (0)
    ST_RUN(R1);
    ST_RUN(C1);
    ST_DUST(0);
    ST_RUN(R2);
    ST_DUST(1);
    ST_RUN(C3);
    ST_DUST(2);
    ST_RUN(R4);
    ST_DUST(3);
    ST_RUN(C5);
    ST_DUST(4);
    ST_RUN(R6);
    ST_RUN(C6);
    ST_DUST(5);
#undef ST_RUN
#undef ST_DUST
    return cudaSuccess;
}

// O = P^(T+R,T+R) V on the stored band (apply_transport, sinkhorn.hpp:262-277): the RO row stage
cudaError_t launch_output_tile(const Geo& g, int dtype, const float* S2, const float* u, const float* v, const void* V,
                               float* O, cudaStream_t s) {
    auto go = [&](auto tag, auto dtag) -> cudaError_t {
        using TIn = decltype(tag);
        constexpr int D = decltype(dtag)::value;
        BT<TIn> a{};
        a.S2 = S2;
        a.u2 = u;
        a.u1 = u;
        a.v2 = v;
        a.v1 = v;
        a.v0 = v;
        a.V = (const TIn*)V;
        a.O = O;
        return run_op<RO, false, D, TIn>(g, a, s);
    };
    cudaError_t e;
    if (g.d == 32) e = dtype == 0 ? go(float{}, std::integral_constant<int, 32>{}) : go(__nv_bfloat16{}, std::integral_constant<int, 32>{});
    else if (g.d == 64) e = dtype == 0 ? go(float{}, std::integral_constant<int, 64>{}) : go(__nv_bfloat16{}, std::integral_constant<int, 64>{});
    else e = dtype == 0 ? go(float{}, std::integral_constant<int, 128>{}) : go(__nv_bfloat16{}, std::integral_constant<int, 128>{});
    add_launches(1);
    return e;
}

cudaError_t launch_backward_tile(const Geo& g, int dtype, const BwdPtrs& p, const BwdTPtrs& t, bool direct,
                                 cudaStream_t s, long long& launches) {
    if (g.dustbin) {
        const long n = (long)g.BH * (g.Lq + g.Lk);
        if (dtype == 0) k_dust_dots<float><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(g, (const float*)p.dO, (const float*)p.V, t.Zd, t.ZdT);
        else k_dust_dots<__nv_bfloat16><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(g, (const __nv_bfloat16*)p.dO, (const __nv_bfloat16*)p.V, t.Zd, t.ZdT);
        ++launches;
    }
#define ST_DISPATCH(D)                                                                                 \
    if (dtype == 0) return direct ? run_all<true, D, float>(g, p, t, dtype, s, launches)               \
                                  : run_all<false, D, float>(g, p, t, dtype, s, launches);            \
    return direct ? run_all<true, D, __nv_bfloat16>(g, p, t, dtype, s, launches)                      \
                  : run_all<false, D, __nv_bfloat16>(g, p, t, dtype, s, launches);
    if (g.d == 32) { ST_DISPATCH(32) }
    if (g.d == 64) { ST_DISPATCH(64) }
    ST_DISPATCH(128)
#undef ST_DISPATCH
}

}  // namespace st
