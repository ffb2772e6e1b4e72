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
#include <cstdlib>
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
    int fuse_c5;  // C6 also produces v0b (the C5 sweep) -- no dustbin
};

enum { R1 = 0, R2 = 1, R4 = 2, R6 = 3, RO = 4, R12 = 5, RW = 6, C1 = 10, C3 = 11, C5 = 12, C6 = 13, CW = 14 };
// RW / CW: dQ (+ d_eps) / dK from a materialised score-cotangent band (generic-R tail adjoint)
// R12 = R1 and R2 in one sweep (g_u_i = sum P22 Z, u2b_i = g_u_i - sum P22 g_v_j): needs C1 first

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
    constexpr bool kNeedZ = (kOp == R1 || kOp == R12 || kOp == R6 || kOp == C1 || kOp == C6);
    constexpr bool kVec = (kOp == R6 || kOp == C1 || kOp == C6 || kOp == RO || kOp == RW || kOp == CW);
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
            if (kOp == R1 || kOp == R12) a.g_u[bo + i] = 0.f;
            if (kOp == R2 || kOp == R12) a.u2b[bo + i] = 0.f;
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
    constexpr int nvec = 5;  // (layout must match bwdT_op_smem)
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
                if (kOp == R2 || kOp == R12 || kOp == R6) w3 = a.g_v[bx + x];
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
        if (kOp == R1 || kOp == R12) a.g_u[bo + i] = 0.f;
        if (kOp == R2 || kOp == R12) a.u2b[bo + i] = 0.f;
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
    float acc = 0.f, dacc = 0.f, acc2 = 0.f;
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
        } else if (kOp == R12) {
            acc += p * tz[k];
            acc2 += p * wv[3 * Nw + c];
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
        } else if (kOp == R12) {
            acc += p * z;
            acc2 += p * a.g_v[bx + xd];
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
    if (kOp == R12) {
        a.g_u[bo + i] = acc;
        a.u2b[bo + i] = acc - acc2;
    }
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

// ---------------------------------------------------------------------------
// Vector stages (R6 dQ, C6 dK, C1 dV, RO output) as weights + band GEMM.
// Phase 1 (two threads per own row): the per-cell weight W (P22 or Sbar) is
// computed once and written over the S tile in place; scalar partials
// (g_v, d_eps) are combined over the two halves in a fixed order.
// Phase 2: out[i][:] = sum_k W[i][k] X[i - w + k][:] as a register-tiled band
// GEMM: thread = 4 own rows x (D/8) columns, per band step 4 broadcast W loads
// + D/32 LDS.128 of the operand row feed 4 D/8 FMAs.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float2 ffma2w(float2 a, float2 b, float2 c) {  // FFMA2 (packed fp32, sm_100)
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "mov.b64 rc, {%6, %7};\n\tfma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}

template <int kOp, bool kDirect, int D, class TIn>
__global__ void __launch_bounds__(256) k_bwdV(Geo g, BT<TIn> a) {
    extern __shared__ __align__(16) float smf[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ float sacc[2][128], sdacc[2][128], pd[128];
    constexpr bool kRow = kOp < 10;
    constexpr bool kNeedZ = (kOp == R6 || kOp == C1 || kOp == C6 || kOp == RW || kOp == CW);
    constexpr int CPT = D / 8;  // output columns per thread
    const int Lo = kRow ? g.Lq : g.Lk, Lx = kRow ? g.Lk : g.Lq;
    const int Lro = kRow ? g.Lrq : g.Lrk, Lrx = kRow ? g.Lrk : g.Lrq;
    const int Lpo = kRow ? g.Lqp : g.Lkp;
    const uint8_t* mo = kRow ? g.row_mask : g.col_mask;
    const uint8_t* mx = kRow ? g.col_mask : g.row_mask;
    const int bh = blockIdx.y, i0 = blockIdx.x * 128, tid = threadIdx.x;
    const size_t bo = (size_t)bh * Lro, bx = (size_t)bh * Lrx;
    auto on_o = [&](int k) { return k < Lo && (mo == nullptr || mo[(size_t)(bh / g.H) * Lo + k] != 0); };
    auto on_x = [&](int k) { return k >= 0 && k < Lx && (mx == nullptr || mx[(size_t)(bh / g.H) * Lx + k] != 0); };
    const int r = tid & 127, hh = tid >> 7, i = i0 + r;
    const bool active = on_o(i);
    float* vo = (kOp == R6 || kOp == RW) ? a.dQ : kOp == C1 ? a.dV : kOp == RO ? a.O : a.dK;
    if (!__syncthreads_or(active)) {
        if (hh == 0 && i < Lo) {
            if (kOp == R6 || kOp == RW) a.deps_part[bo + i] = 0.f;
            if (kOp == C1) a.g_v[bo + i] = 0.f;
            if (kOp == C6 && a.fuse_c5) a.v0b[bo + i] = 0.f;
            for (int x = 0; x < g.d; ++x) vo[(bo + i) * g.d + x] = 0.f;
        }
        return;
    }
    const int Wf = g.Wf, Nw = 128 + 2 * g.w;
    float* tS = smf;
    float* tZ = tS + 128 * Wf;
    float* wv = tZ + (kNeedZ ? 128 * Wf : 0);  // window vectors [5][Nw]
    float* ops = wv + ((5 * Nw + 3) & ~3);     // operand rows [Nw][D] (window row c <-> x = i0 - w + c)
    const TIn* osrc = (kOp == R6 || kOp == RW) ? a.K : (kOp == C1) ? a.dO : (kOp == RO) ? a.V : a.Q;
    // f32 operands: the valid window rows are one contiguous run in global memory -> one bulk copy
    const int xlo = max(0, i0 - g.w), xhi = min(Lx, i0 - g.w + Nw);
    const int clo = xlo - (i0 - g.w), chi = clo + max(0, xhi - xlo);
    const uint32_t obytes = (sizeof(TIn) == 4 && chi > clo) ? (uint32_t)(chi - clo) * D * 4u : 0u;
    if (tid == 0) {
        sm100::mbar_init(&bar, 1);
        sm100::fence_mbar_init();
        const uint32_t tb = 128u * (uint32_t)Wf * 4u;
        sm100::mbar_arrive_expect_tx(&bar, (kNeedZ ? 2 * tb : tb) + obytes);
        const size_t off = ((size_t)bh * Lpo + i0) * Wf;
        sm100::bulk_g2s(tS, (kRow ? a.S2 : a.S2T) + off, tb, &bar);
        if (kNeedZ) sm100::bulk_g2s(tZ, (kRow ? a.Z : a.ZT) + off, tb, &bar);
        if (obytes) sm100::bulk_g2s(ops + clo * D, osrc + (bx + xlo) * D, obytes, &bar);
    }
    // window vectors (other side), c <-> x = i0 - w + c; 0 where invalid (tile carries -inf there)
    //   R6: v2, beta|v1, delta|v0, v2b(=g_v), v1b     C6: u2, alpha|u1, -, u2b, u1b
    //   C1: u2                                         RO: v
    for (int c = tid; c < Nw; c += 256) {
        const int x = i0 - g.w + c;
        float w0 = 0.f, w1 = 0.f, w2 = 0.f, w3 = 0.f, w4 = 0.f;
        if (on_x(x)) {
            if (kRow) {
                w0 = a.v2[bx + x];
                if (kOp == R6) {
                    const float v1 = a.v1[bx + x], v0 = a.v0[bx + x];
                    w1 = kDirect ? v1 : ex2(v1 - w0);
                    w2 = kDirect ? v0 : ex2(v0 - w0);
                    w3 = a.g_v[bx + x];
                    w4 = a.v1b[bx + x];
                }
            } else {
                w0 = a.u2[bx + x];
                if (kOp == C6) {
                    const float u1 = a.u1[bx + x];
                    w1 = kDirect ? u1 : ex2(u1 - w0);
                    w3 = a.u2b[bx + x];
                    w4 = a.u1b[bx + x];
                }
            }
        }
        wv[c] = w0;
        wv[Nw + c] = w1;
        wv[2 * Nw + c] = w2;
        wv[3 * Nw + c] = w3;
        wv[4 * Nw + c] = w4;
    }
    if constexpr (sizeof(TIn) == 4) {  // zero the rows outside the sequence (the bulk copy fills the rest)
        for (int e = tid; e < clo * D; e += 256) ops[e] = 0.f;
        for (int e = chi * D + tid; e < Nw * D; e += 256) ops[e] = 0.f;
    } else {  // bf16 operands, converted to f32
        for (int e = tid; e < Nw * (D / 4); e += 256) {
            const int c = e / (D / 4), q = (e % (D / 4)) * 4;
            const int x = i0 - g.w + c;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (x >= 0 && x < Lx) {
                const TIn* sp = osrc + (bx + x) * D + q;
                v.x = ldf(sp); v.y = ldf(sp + 1); v.z = ldf(sp + 2); v.w = ldf(sp + 3);
            }
            *reinterpret_cast<float4*>(ops + c * D + q) = v;
        }
    }
    __syncthreads();
    sm100::mbar_wait(&bar, 0);
    // ---- phase 1: weights
    const int half = (Wf + 1) >> 1;
    const int kb = hh ? half : 0, ke = hh ? Wf : half;
    float* ts = tS + r * Wf;
    const float* tz = tZ + r * Wf;
    float acc = 0.f, dacc = 0.f;
    if (active) {
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
        // one-reference modifiers of the own index: R6 alpha_i; C6 beta_j, delta_j
        const float ma = ex2(o1 - o2), mb = kRow ? 0.f : ex2(o0 - o2);
        for (int k = kb; k < ke; ++k) {
            const int c = r + k;
            const float s2 = ts[k];
            float wgt = 0.f;
            if (s2 != -INFINITY) {
                const float p = (kOp == RW || kOp == CW) ? 0.f : ex2(s2 + o2 + wv[c]);
                if (kOp == RW || kOp == CW) {  // the band already holds Sbar
                    wgt = tz[k];
                    if (kOp == RW) dacc += wgt * (s2 * kLn2);
                } else if (kOp == RO) {
                    wgt = p;
                } else if (kOp == C1) {
                    acc += p * tz[k];
                    wgt = p;
                } else if (kOp == R6) {
                    const float z = tz[k];
                    if (kDirect) {
                        wgt = sbar_of(true, s2, p, z, o1, o2, wv[2 * Nw + c], wv[Nw + c], wv[c], ob2, ob1,
                                      wv[3 * Nw + c], wv[4 * Nw + c]);
                    } else {  // Sbar = P22 (Z - v2b_j - beta_j u2b_i - alpha_i beta_j v1b_j - alpha_i delta_j u1b_i)
                        const float bj = wv[Nw + c], dj = wv[2 * Nw + c];
                        wgt = p * (z - wv[3 * Nw + c] - bj * ob2 - ma * bj * wv[4 * Nw + c] - ma * dj * ob1);
                    }
                    dacc += wgt * (s2 * kLn2);
                } else {  // C6: own = column j, window = rows i
                    const float z = tz[k];
                    if (kDirect) {
                        wgt = sbar_of(true, s2, p, z, wv[Nw + c], wv[c], o0, o1, o2, wv[3 * Nw + c], wv[4 * Nw + c],
                                      ob2, ob1);
                        if (a.fuse_c5) acc += ex2(s2 + wv[Nw + c] + o0) * wv[4 * Nw + c];  // C5: P10 u1b
                    } else {  // alpha_i = wv[Nw + c], beta_j = ma, delta_j = mb
                        const float ai = wv[Nw + c];
                        wgt = p * (z - ob2 - ma * wv[3 * Nw + c] - ai * ma * ob1 - ai * mb * wv[4 * Nw + c]);
                        acc += p * ai * wv[4 * Nw + c];  // C5: P22 alpha_i u1b_i (used when fuse_c5)
                    }
                }
            }
            ts[k] = wgt;
        }
        if (hh == 0) {
            float pdv = 0.f;
            if (g.dustbin) {  // the spoke cell (row i, dustbin column) / (dustbin row, column j)
                const int xd = Lx;
                const float s2 = g.sd2;
                const float x2 = kRow ? a.v2[bx + xd] : a.u2[bx + xd];
                const float p = ex2(s2 + o2 + x2);
                if (kOp == RO) {
                    pdv = p;
                } else if (kOp == C1) {
                    acc += p * a.ZdT[(size_t)bh * g.Lkp + i];
                    pdv = p;
                } else if (kOp == R6) {
                    const float x1 = a.v1[bx + xd];
                    const float sb = sbar_of(kDirect, s2, p, a.Zd[(size_t)bh * g.Lqp + i], o1, o2, a.v0[bx + xd], x1,
                                             x2, ob2, ob1, a.g_v[bx + xd], a.v1b[bx + xd]);
                    dacc += sb * (s2 * kLn2);  // constant cost: no dQ contribution
                }
            }
            pd[r] = pdv;
        }
    } else {
        for (int k = kb; k < ke; ++k) ts[k] = 0.f;
        if (hh == 0) pd[r] = 0.f;
    }
    sacc[hh][r] = acc;
    sdacc[hh][r] = dacc;
    __syncthreads();
    if (hh == 0 && i < Lo) {
        if (kOp == C1) a.g_v[bo + i] = active ? sacc[0][r] + sacc[1][r] : 0.f;
        if (kOp == R6 || kOp == RW) a.deps_part[bo + i] = active ? sdacc[0][r] + sdacc[1][r] : 0.f;
        if (kOp == C6 && a.fuse_c5) {  // v0b_j = -delta_j sum_i P22 alpha_i u1b_i  (direct: -sum P10 u1b)
            const float s5 = sacc[0][r] + sacc[1][r];
            a.v0b[bo + i] = !active ? 0.f : kDirect ? -s5 : -ex2(a.v0[bo + i] - a.v2[bo + i]) * s5;
        }
    }
    // ---- phase 2: band GEMM.  thread = rows 4 rg .. 4 rg + 3, column chunks {4 cg + 32 m}
    if (g.dbg & 1) return;  // timing studies only (ST_BWD_DBG)
    const int rg = tid >> 3, cg = tid & 7;
    float2 accv[4][CPT / 2];  // column pairs (FFMA2)
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int e = 0; e < CPT / 2; ++e) accv[q][e] = make_float2(0.f, 0.f);
    const float* wrow = tS + (4 * rg) * Wf;
    // band step kk feeds rows q with cell k = kk - q; only the first / last 3 steps need the
    // k in [0, Wf) guard, the interior runs check-free
    auto step = [&](int kk, bool guard) {
        float2 wq[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int k = kk - q;
            const float wk = (!guard || (k >= 0 && k < Wf)) ? wrow[q * Wf + k] : 0.f;
            wq[q] = make_float2(wk, wk);
        }
        const float* xr = ops + (4 * rg + kk) * D + 4 * cg;
#pragma unroll
        for (int m = 0; m < CPT / 4; ++m) {
            const float4 x4 = *reinterpret_cast<const float4*>(xr + 32 * m);
            const float2 xa = make_float2(x4.x, x4.y), xb = make_float2(x4.z, x4.w);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                accv[q][2 * m + 0] = ffma2w(xa, wq[q], accv[q][2 * m + 0]);
                accv[q][2 * m + 1] = ffma2w(xb, wq[q], accv[q][2 * m + 1]);
            }
        }
    };
    const int kin = min(3, Wf + 3);
    for (int kk = 0; kk < kin; ++kk) step(kk, true);
#pragma unroll 2
    for (int kk = 3; kk < Wf; ++kk) step(kk, false);
    for (int kk = max(Wf, kin); kk < Wf + 3; ++kk) step(kk, true);
    const float sc = (kOp == C1 || kOp == RO) ? 1.f : g.inv_qk;
    const TIn* dsrc = (kOp == RO) ? a.V : (kOp == C1) ? a.dO : nullptr;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int row = 4 * rg + q, ii = i0 + row;
        if (ii >= Lo) continue;
        const float pdq = pd[row];
#pragma unroll
        for (int m = 0; m < CPT / 4; ++m) {
            const int col = 4 * cg + 32 * m;
            float4 o4 = make_float4(accv[q][2 * m].x * sc, accv[q][2 * m].y * sc, accv[q][2 * m + 1].x * sc,
                                    accv[q][2 * m + 1].y * sc);
            if (dsrc != nullptr && g.dustbin) {  // + p_dust * (V | dO)_dustbin
                const TIn* dr = dsrc + (bx + Lx) * D + col;
                o4.x = fmaf(pdq, ldf(dr), o4.x);
                o4.y = fmaf(pdq, ldf(dr + 1), o4.y);
                o4.z = fmaf(pdq, ldf(dr + 2), o4.z);
                o4.w = fmaf(pdq, ldf(dr + 3), o4.w);
            }
            *reinterpret_cast<float4*>(vo + (bo + ii) * D + col) = o4;
        }
    }
}

// ---------------------------------------------------------------------------
// Wide-band variants (RB = 64 / 32 rows per CTA, for bands whose 128-row tiles do
// not fit SMEM: configs 4 and 5).  Same stage math as k_bwdT / k_bwdV; a row is
// shared by TPR threads that take interleaved groups of GS = 32 / TPR cells (the
// 32 lanes of a warp hit 32 distinct banks with the odd pitch Wf) and combine
// with a fixed butterfly.  No dustbin (dustbin configs have narrow bands).
// ---------------------------------------------------------------------------
template <int kOp, bool kDirect, int RB, class TIn>
__global__ void __launch_bounds__(128) k_bwdS(Geo g, BT<TIn> a) {
    extern __shared__ __align__(16) float smf[];
    __shared__ __align__(8) uint64_t bar;
    constexpr int TPR = 128 / RB, GS = 32 / TPR;
    constexpr bool kRow = kOp < 10;
    constexpr bool kNeedZ = (kOp == R1 || kOp == R12);
    const int Lo = kRow ? g.Lq : g.Lk, Lx = kRow ? g.Lk : g.Lq;
    const int Lro = kRow ? g.Lrq : g.Lrk, Lrx = kRow ? g.Lrk : g.Lrq;
    const int Lpo = kRow ? g.Lqp : g.Lkp;
    const uint8_t* mo = kRow ? g.row_mask : g.col_mask;
    const uint8_t* mx = kRow ? g.col_mask : g.row_mask;
    const int bh = blockIdx.y, i0 = blockIdx.x * RB, tid = threadIdx.x, lane = tid & 31;
    const int part = lane / GS, r = (tid >> 5) * GS + lane % GS, i = i0 + r;
    const size_t bo = (size_t)bh * Lro, bx = (size_t)bh * Lrx;
    auto on_o = [&](int k) { return k < Lo && (mo == nullptr || mo[(size_t)(bh / g.H) * Lo + k] != 0); };
    auto on_x = [&](int k) { return k >= 0 && k < Lx && (mx == nullptr || mx[(size_t)(bh / g.H) * Lx + k] != 0); };
    const bool active = on_o(i);
    auto put = [&](float val) {
        if (kOp == R1 || kOp == R12) a.g_u[bo + i] = val;
        if (kOp == R2) a.u2b[bo + i] = val;
        if (kOp == R4) a.u1b[bo + i] = val;
        if (kOp == C3) a.v1b[bo + i] = val;
        if (kOp == C5) a.v0b[bo + i] = val;
    };
    if (!__syncthreads_or(active)) {
        if (part == 0 && i < Lo) put(0.f);
        return;
    }
    const int Wf = g.Wf, Nw = RB + 2 * g.w;
    float* tS = smf;
    float* tZ = tS + RB * Wf;
    float* wv = tZ + (kNeedZ ? RB * Wf : 0);
    if (tid == 0) {
        sm100::mbar_init(&bar, 1);
        sm100::fence_mbar_init();
        const uint32_t tb = (uint32_t)RB * (uint32_t)Wf * 4u;
        sm100::mbar_arrive_expect_tx(&bar, kNeedZ ? 2 * tb : tb);
        const size_t off = ((size_t)bh * Lpo + i0) * Wf;
        sm100::bulk_g2s(tS, (kRow ? a.S2 : a.S2T) + off, tb, &bar);
        if (kNeedZ) sm100::bulk_g2s(tZ, a.Z + off, tb, &bar);
    }
    for (int c = tid; c < Nw; c += 128) {
        const int x = i0 - g.w + c;
        float w0 = 0.f, w1 = 0.f, w3 = 0.f, w4 = 0.f;
        if (on_x(x)) {
            if (kRow) {
                w0 = a.v2[bx + x];
                w1 = a.v1[bx + x];
                if (kOp == R2 || kOp == R12) w3 = a.g_v[bx + x];
                if (kOp == R4) w4 = a.v1b[bx + x];
            } else {
                w0 = a.u2[bx + x];
                w1 = a.u1[bx + x];
                if (kOp == C3) w3 = a.u2b[bx + x];
                if (kOp == C5) w4 = a.u1b[bx + x];
            }
        }
        wv[c] = w0;
        wv[Nw + c] = w1;
        wv[3 * Nw + c] = w3;
        wv[4 * Nw + c] = w4;
    }
    __syncthreads();
    sm100::mbar_wait(&bar, 0);
    float o2 = 0.f, o1 = 0.f, o0 = 0.f;
    if (active) {
        o2 = kRow ? a.u2[bo + i] : a.v2[bo + i];
        o1 = kRow ? a.u1[bo + i] : a.v1[bo + i];
        if (!kRow) o0 = a.v0[bo + i];
    }
    float acc = 0.f, acc2 = 0.f;
    if (active) {
        const float* ts = tS + r * Wf;
        const float* tz = tZ + r * Wf;
        for (int k0 = part * GS; k0 < Wf; k0 += TPR * GS) {
#pragma unroll 4
            for (int kk = 0; kk < GS; ++kk) {
                const int k = k0 + kk;
                if (k >= Wf) break;
                const float s2 = ts[k];
                if (s2 == -INFINITY) continue;
                const int c = r + k;
                const float x2 = wv[c], x1 = wv[Nw + c];
                const float p = ex2(s2 + o2 + x2);
                if (kOp == R1) acc += p * tz[k];
                else if (kOp == R12) {
                    acc += p * tz[k];
                    acc2 += p * wv[3 * Nw + c];
                } else if (kOp == R2) acc += p * wv[3 * Nw + c];
                else if (kOp == R4) acc += kDirect ? ex2(s2 + o1 + x1) * wv[4 * Nw + c] : p * ex2(x1 - x2) * wv[4 * Nw + c];
                else if (kOp == C3) acc += (kDirect ? ex2(s2 + x2 + o1) : p) * wv[3 * Nw + c];
                else acc += kDirect ? ex2(s2 + x1 + o0) * wv[4 * Nw + c] : p * ex2(x1 - x2) * wv[4 * Nw + c];
            }
        }
    }
#pragma unroll
    for (int off = GS; off < 32; off <<= 1) {
        acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (kOp == R12) acc2 += __shfl_xor_sync(0xffffffffu, acc2, off);
    }
    if (kOp == R12 && part == 0 && i < Lo) a.u2b[bo + i] = active ? acc - acc2 : 0.f;
    if (part == 0 && i < Lo) {
        float val = 0.f;
        if (active) {
            if (kOp == R1 || kOp == R12) val = acc;
            if (kOp == R2) val = a.g_u[bo + i] - acc;
            if (kOp == R4) val = kDirect ? -acc : -ex2(o1 - o2) * acc;
            if (kOp == C3) val = kDirect ? -acc : -ex2(o1 - o2) * acc;
            if (kOp == C5) val = kDirect ? -acc : -ex2(o0 - o2) * acc;
        }
        put(val);
    }
}

template <class T>
__device__ __forceinline__ float4 ld4f(const T* p);
template <>
__device__ __forceinline__ float4 ld4f<float>(const float* p) {
    return *reinterpret_cast<const float4*>(p);
}
template <>
__device__ __forceinline__ float4 ld4f<__nv_bfloat16>(const __nv_bfloat16* p) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    return make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xffff0000u), __uint_as_float(u.y << 16),
                       __uint_as_float(u.y & 0xffff0000u));
}

template <int RB, int D>
struct GemmShape {
    static constexpr int OPT = RB * D / 256;          // outputs per thread
    static constexpr int RPT = OPT >= 16 ? 4 : 2;     // rows per thread
    static constexpr int CPT = OPT / RPT;             // columns per thread (multiple of 4)
    static constexpr int NCG = D / CPT;               // column groups
    static_assert(CPT % 4 == 0, "column chunks of 4");
};

template <int kOp, bool kDirect, int D, class TIn, int RB>
__global__ void __launch_bounds__(256) k_bwdG(Geo g, BT<TIn> a) {
    extern __shared__ __align__(16) float smf[];
    __shared__ __align__(8) uint64_t bar;
    using GS_ = GemmShape<RB, D>;
    constexpr int TPR = 256 / RB, GS = 32 / TPR;
    constexpr int OP = D;  // operand row pitch (elements): contiguous window rows, one bulk copy
    constexpr bool kRow = kOp < 10;
    constexpr bool kNeedZ = (kOp == R6 || kOp == C1 || kOp == C6 || kOp == RW || kOp == CW);
    const int Lo = kRow ? g.Lq : g.Lk, Lx = kRow ? g.Lk : g.Lq;
    const int Lro = kRow ? g.Lrq : g.Lrk, Lrx = kRow ? g.Lrk : g.Lrq;
    const int Lpo = kRow ? g.Lqp : g.Lkp;
    const uint8_t* mo = kRow ? g.row_mask : g.col_mask;
    const uint8_t* mx = kRow ? g.col_mask : g.row_mask;
    const int bh = blockIdx.y, i0 = blockIdx.x * RB, tid = threadIdx.x, lane = tid & 31;
    const int part = lane / GS, r = (tid >> 5) * GS + lane % GS, i = i0 + r;
    const size_t bo = (size_t)bh * Lro, bx = (size_t)bh * Lrx;
    auto on_o = [&](int k) { return k < Lo && (mo == nullptr || mo[(size_t)(bh / g.H) * Lo + k] != 0); };
    auto on_x = [&](int k) { return k >= 0 && k < Lx && (mx == nullptr || mx[(size_t)(bh / g.H) * Lx + k] != 0); };
    const bool active = on_o(i);
    float* vo = (kOp == R6 || kOp == RW) ? a.dQ : kOp == C1 ? a.dV : kOp == RO ? a.O : a.dK;
    if (!__syncthreads_or(active)) {
        if (part == 0 && i < Lo) {
            if (kOp == R6 || kOp == RW) a.deps_part[bo + i] = 0.f;
            if (kOp == C1) a.g_v[bo + i] = 0.f;
            if (kOp == C6 && a.fuse_c5) a.v0b[bo + i] = 0.f;
            for (int x = 0; x < D; ++x) vo[(bo + i) * D + x] = 0.f;
        }
        return;
    }
    const int Wf = g.Wf, Nw = RB + 2 * g.w;
    float* tS = smf;
    float* tZ = tS + RB * Wf;
    float* wv = tZ + (kNeedZ ? RB * Wf : 0);
    TIn* ops = reinterpret_cast<TIn*>(wv + ((5 * Nw + 3) & ~3));
    const TIn* osrc = (kOp == R6 || kOp == RW) ? a.K : (kOp == C1) ? a.dO : (kOp == RO) ? a.V : a.Q;
    const int xlo = max(0, i0 - g.w), xhi = min(Lx, i0 - g.w + Nw);
    const int clo = xlo - (i0 - g.w), chi = clo + max(0, xhi - xlo);
    const uint32_t obytes = chi > clo ? (uint32_t)(chi - clo) * D * (uint32_t)sizeof(TIn) : 0u;
    if (tid == 0) {
        sm100::mbar_init(&bar, 1);
        sm100::fence_mbar_init();
        const uint32_t tb = (uint32_t)RB * (uint32_t)Wf * 4u;
        sm100::mbar_arrive_expect_tx(&bar, (kNeedZ ? 2 * tb : tb) + obytes);
        const size_t off = ((size_t)bh * Lpo + i0) * Wf;
        sm100::bulk_g2s(tS, (kRow ? a.S2 : a.S2T) + off, tb, &bar);
        if (kNeedZ) sm100::bulk_g2s(tZ, (kRow ? a.Z : a.ZT) + off, tb, &bar);
        if (obytes) sm100::bulk_g2s(ops + clo * D, osrc + (bx + xlo) * D, obytes, &bar);
    }
    for (int c = tid; c < Nw; c += 256) {
        const int x = i0 - g.w + c;
        float w0 = 0.f, w1 = 0.f, w2 = 0.f, w3 = 0.f, w4 = 0.f;
        if (on_x(x)) {
            if (kRow) {
                w0 = a.v2[bx + x];
                if (kOp == R6) {
                    const float v1 = a.v1[bx + x], v0 = a.v0[bx + x];
                    w1 = kDirect ? v1 : ex2(v1 - w0);
                    w2 = kDirect ? v0 : ex2(v0 - w0);
                    w3 = a.g_v[bx + x];
                    w4 = a.v1b[bx + x];
                }
            } else {
                w0 = a.u2[bx + x];
                if (kOp == C6) {
                    const float u1 = a.u1[bx + x];
                    w1 = kDirect ? u1 : ex2(u1 - w0);
                    w3 = a.u2b[bx + x];
                    w4 = a.u1b[bx + x];
                }
            }
        }
        wv[c] = w0;
        wv[Nw + c] = w1;
        wv[2 * Nw + c] = w2;
        wv[3 * Nw + c] = w3;
        wv[4 * Nw + c] = w4;
    }
    {   // operand window rows (input dtype): the bulk copy brings the valid run, zero the rest
        const TIn z{};
        for (int e = tid; e < clo * D; e += 256) ops[e] = z;
        for (int e = chi * D + tid; e < Nw * D; e += 256) ops[e] = z;
    }
    __syncthreads();
    sm100::mbar_wait(&bar, 0);
    // ---- phase 1: weights over the cell groups of this thread, written in place
    float acc = 0.f, dacc = 0.f;
    float* ts = tS + r * Wf;
    const float* tz = tZ + r * Wf;
    if (active) {
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
        const float ma = ex2(o1 - o2), mb = kRow ? 0.f : ex2(o0 - o2);
        for (int k0 = part * GS; k0 < Wf; k0 += TPR * GS) {
#pragma unroll 4
            for (int kk = 0; kk < GS; ++kk) {
                const int k = k0 + kk;
                if (k >= Wf) break;
                const int c = r + k;
                const float s2 = ts[k];
                float wgt = 0.f;
                if (s2 != -INFINITY) {
                    const float p = (kOp == RW || kOp == CW) ? 0.f : ex2(s2 + o2 + wv[c]);
                    if (kOp == RW || kOp == CW) {  // the band already holds Sbar
                        wgt = tz[k];
                        if (kOp == RW) dacc += wgt * (s2 * kLn2);
                    } else if (kOp == RO) {
                        wgt = p;
                    } else if (kOp == C1) {
                        acc += p * tz[k];
                        wgt = p;
                    } else if (kOp == R6) {
                        const float z = tz[k];
                        if (kDirect) {
                            wgt = sbar_of(true, s2, p, z, o1, o2, wv[2 * Nw + c], wv[Nw + c], wv[c], ob2, ob1,
                                          wv[3 * Nw + c], wv[4 * Nw + c]);
                        } else {
                            const float bj = wv[Nw + c], dj = wv[2 * Nw + c];
                            wgt = p * (z - wv[3 * Nw + c] - bj * ob2 - ma * bj * wv[4 * Nw + c] - ma * dj * ob1);
                        }
                        dacc += wgt * (s2 * kLn2);
                    } else {
                        const float z = tz[k];
                        if (kDirect) {
                            wgt = sbar_of(true, s2, p, z, wv[Nw + c], wv[c], o0, o1, o2, wv[3 * Nw + c],
                                          wv[4 * Nw + c], ob2, ob1);
                            if (a.fuse_c5) acc += ex2(s2 + wv[Nw + c] + o0) * wv[4 * Nw + c];
                        } else {
                            const float ai = wv[Nw + c];
                            wgt = p * (z - ob2 - ma * wv[3 * Nw + c] - ai * ma * ob1 - ai * mb * wv[4 * Nw + c]);
                            acc += p * ai * wv[4 * Nw + c];
                        }
                    }
                }
                ts[k] = wgt;
            }
        }
    } else {
        for (int k0 = part * GS; k0 < Wf; k0 += TPR * GS)
            for (int kk = 0; kk < GS && k0 + kk < Wf; ++kk) ts[k0 + kk] = 0.f;
    }
#pragma unroll
    for (int off = GS; off < 32; off <<= 1) {
        acc += __shfl_xor_sync(0xffffffffu, acc, off);
        dacc += __shfl_xor_sync(0xffffffffu, dacc, off);
    }
    if (part == 0 && i < Lo) {
        if (kOp == C1) a.g_v[bo + i] = active ? acc : 0.f;
        if (kOp == R6 || kOp == RW) a.deps_part[bo + i] = active ? dacc : 0.f;
        if (kOp == C6 && a.fuse_c5)
            a.v0b[bo + i] = !active ? 0.f : kDirect ? -acc : -ex2(a.v0[bo + i] - a.v2[bo + i]) * acc;
    }
    __syncthreads();
    // ---- phase 2: band GEMM, thread = RPT own rows x CPT columns (chunks of 4, stride 4 NCG)
    constexpr int RPT = GS_::RPT, CPT = GS_::CPT, NCG = GS_::NCG;
    const int rg = tid / NCG, cg = tid % NCG;
    float accv[RPT][CPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q)
#pragma unroll
        for (int e = 0; e < CPT; ++e) accv[q][e] = 0.f;
    const float* wrow = tS + (RPT * rg) * Wf;
    auto step = [&](int kk, bool guard) {
        float wq[RPT];
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const int k = kk - q;
            wq[q] = (!guard || (k >= 0 && k < Wf)) ? wrow[q * Wf + k] : 0.f;
        }
        const TIn* xr = ops + (RPT * rg + kk) * OP + 4 * cg;
#pragma unroll
        for (int m = 0; m < CPT / 4; ++m) {
            const float4 x4 = ld4f<TIn>(xr + 4 * NCG * m);
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                accv[q][4 * m + 0] = fmaf(wq[q], x4.x, accv[q][4 * m + 0]);
                accv[q][4 * m + 1] = fmaf(wq[q], x4.y, accv[q][4 * m + 1]);
                accv[q][4 * m + 2] = fmaf(wq[q], x4.z, accv[q][4 * m + 2]);
                accv[q][4 * m + 3] = fmaf(wq[q], x4.w, accv[q][4 * m + 3]);
            }
        }
    };
    const int kin = min(RPT - 1, Wf + RPT - 1);
    for (int kk = 0; kk < kin; ++kk) step(kk, true);
#pragma unroll 2
    for (int kk = RPT - 1; kk < Wf; ++kk) step(kk, false);
    for (int kk = max(Wf, kin); kk < Wf + RPT - 1; ++kk) step(kk, true);
    const float sc = (kOp == C1 || kOp == RO) ? 1.f : g.inv_qk;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        const int ii = i0 + RPT * rg + q;
        if (ii >= Lo) continue;
#pragma unroll
        for (int m = 0; m < CPT / 4; ++m) {
            const int col = 4 * cg + 4 * NCG * m;
            *reinterpret_cast<float4*>(vo + (bo + ii) * D + col) =
                make_float4(accv[q][4 * m] * sc, accv[q][4 * m + 1] * sc, accv[q][4 * m + 2] * sc,
                            accv[q][4 * m + 3] * sc);
        }
    }
}

// ---------------------------------------------------------------------------
// Window-chunked vector stages (R6 dQ, C6 dK (+C5), C1 dV, RO output, RW / CW) for dustbin-free
// bands with w % 16 == 0.  The band tile is read in its sheared view: cell (row i0 + r, window
// column c = r + k) sits at base + r (Wf - 1) + c, so 32 consecutive window columns of one row are
// 128 contiguous, 16-byte aligned bytes, and one chunk of the window is a [128][32] strip.  Per
// chunk of kWC = 32 window columns (NSTG-deep cp.async ring of S / Z strips + the chunk's 32
// operand rows; NSTG = 2 and one WT buffer keep two CTAs per SM):
//   phase 1 (2 threads per row, rotated column order: bank-conflict free) the weight W of every cell
//           (0 off the band), stored transposed WT[c][r]; row partials (g_v, d_eps, v0b) in registers
//   phase 2 dense tile GEMM out[128][D] += W X over the chunk: thread = 4 rows x D/8 columns, per
//           window column one LDS.128 of W and D/32 LDS.128 of X feed 4 D/8 FMAs; warps whose 16
//           rows miss the chunk skip it
// Every operand row is read once per block (no per-row window redundancy), every reduction has a
// fixed order (increasing window column), and the kernel is independent of the band width beyond
// the chunk count.
// ---------------------------------------------------------------------------
constexpr int kWC = 16;  // window columns per chunk

// 16-byte global -> shared async copy (LDGSTS); src_bytes = 0 zero-fills the destination
__device__ __forceinline__ void cp_async16(void* dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sm100::smem_u32(dst)), "l"(src), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int D, class TIn>
__host__ __device__ constexpr size_t bwdW_stage_floats(bool z) {
    return (size_t)(z ? 2 : 1) * 128 * kWC + (size_t)kWC * D * sizeof(TIn) / 4;
}
template <int D, class TIn>
static size_t bwdW_smem_bytes(const Geo& g, bool z, int nstg) {
    const int Nw = 128 + 2 * g.w;
    const size_t xf = sizeof(TIn) == 4 ? 0 : (size_t)kWC * D;  // f32 copy of a bf16 operand chunk
    return ((size_t)nstg * bwdW_stage_floats<D, TIn>(z) + kWC * 128 + xf + 5 * (size_t)Nw) * 4 + 128;
}
bool bwdW_supported(const Geo& g) {
    return !g.dustbin && g.w >= 16 && g.w % 16 == 0 && (g.d == 32 || g.d == 64 || g.d == 128) &&
           !getenv("ST_NO_BWDW");
}

template <int kOp, bool kDirect, int D, class TIn, int NSTG>
__global__ void __launch_bounds__(256, (D <= 64 ? 3 : 2)) k_bwdW(Geo g, BT<TIn> a) {
    extern __shared__ __align__(128) float smw[];
    __shared__ float sacc[2][128], sdacc[2][128];
    constexpr bool kRow = kOp < 10;
    constexpr bool kNeedZ = (kOp == R6 || kOp == C1 || kOp == C6 || kOp == RW || kOp == CW);
    constexpr int CPT = D / 8;  // output columns per thread
    const int Lo = kRow ? g.Lq : g.Lk, Lx = kRow ? g.Lk : g.Lq;
    const int Lro = kRow ? g.Lrq : g.Lrk, Lrx = kRow ? g.Lrk : g.Lrq;
    const int Lpo = kRow ? g.Lqp : g.Lkp;
    const uint8_t* mo = kRow ? g.row_mask : g.col_mask;
    const uint8_t* mx = kRow ? g.col_mask : g.row_mask;
    const int bh = blockIdx.y, i0 = blockIdx.x * 128, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const size_t bo = (size_t)bh * Lro, bx = (size_t)bh * Lrx;
    auto on_o = [&](int k) { return k < Lo && (mo == nullptr || mo[(size_t)(bh / g.H) * Lo + k] != 0); };
    auto on_x = [&](int k) { return k >= 0 && k < Lx && (mx == nullptr || mx[(size_t)(bh / g.H) * Lx + k] != 0); };
    const int r = tid & 127, hh = tid >> 7, i = i0 + r;
    const bool active = on_o(i);
    float* vo = (kOp == R6 || kOp == RW) ? a.dQ : kOp == C1 ? a.dV : kOp == RO ? a.O : a.dK;
    if (!__syncthreads_or(active)) {
        if (hh == 0 && i < Lo) {
            if (kOp == R6 || kOp == RW) a.deps_part[bo + i] = 0.f;
            if (kOp == C1) a.g_v[bo + i] = 0.f;
            if (kOp == C6 && a.fuse_c5) a.v0b[bo + i] = 0.f;
            for (int x = 0; x < D; ++x) vo[(bo + i) * D + x] = 0.f;
        }
        return;
    }
    const int Wf = g.Wf, Nw = 128 + 2 * g.w, NCH = Nw / kWC;
    const size_t stf = bwdW_stage_floats<D, TIn>(kNeedZ);
    float* WT = smw + NSTG * stf;     // [kWC][128]
    float* Xf = WT + kWC * 128;       // [kWC][D] f32 operand chunk (bf16 inputs: converted once per chunk)
    float* wv = Xf + (sizeof(TIn) == 4 ? 0 : kWC * D);  // [5][Nw]
    const float* Sb = (kRow ? a.S2 : a.S2T) + ((size_t)bh * Lpo + i0) * Wf;
    const float* Zb = kNeedZ ? (kRow ? a.Z : a.ZT) + ((size_t)bh * Lpo + i0) * Wf : nullptr;
    const TIn* osrc = (kOp == R6 || kOp == RW) ? a.K : (kOp == C1) ? a.dO : (kOp == RO) ? a.V : a.Q;
    auto stS = [&](int s) { return smw + (size_t)s * stf; };
    auto stZ = [&](int s) { return smw + (size_t)s * stf + 128 * kWC; };
    auto stX = [&](int s) { return reinterpret_cast<TIn*>(smw + (size_t)s * stf + (kNeedZ ? 2 : 1) * 128 * kWC); };
    auto issue = [&](int j) {  // all threads: one chunk's strips (8 x 16 B per row and band) + operand rows
        const int s = j % NSTG, c0 = j * kWC;
        float* S = stS(s);
        float* Z = stZ(s);
        for (int e = tid; e < 128 * (kWC / 4); e += 256) {
            const int rr = e / (kWC / 4), sg = (e % (kWC / 4)) * 4;
            cp_async16(S + rr * kWC + sg, Sb + (size_t)rr * (Wf - 1) + c0 + sg, 16u);
            if (kNeedZ) cp_async16(Z + rr * kWC + sg, Zb + (size_t)rr * (Wf - 1) + c0 + sg, 16u);
        }
        constexpr int SPR = D * (int)sizeof(TIn) / 16;  // 16-byte segments per operand row
        const int xb0 = i0 - g.w + c0;
        TIn* X = stX(s);
        for (int e = tid; e < kWC * SPR; e += 256) {
            const int row = e / SPR, sg = e % SPR, x = xb0 + row;
            const bool ok = x >= 0 && x < Lx;  // rows outside the sequence: zero-filled
            cp_async16(reinterpret_cast<uint8_t*>(X) + (size_t)row * D * sizeof(TIn) + sg * 16,
                       reinterpret_cast<const uint8_t*>(osrc + (bx + (ok ? x : 0)) * D) + sg * 16, ok ? 16u : 0u);
        }
        cp_async_commit();
    };
    for (int j = 0; j < NSTG - 1; ++j) {  // prologue (empty groups past the end keep the count uniform)
        if (j < NCH) issue(j);
        else cp_async_commit();
    }
    // window vectors (other side), c <-> x = i0 - w + c; 0 where invalid (the band carries -inf there)
    //   R6: v2, beta|v1, delta|v0, v2b(=g_v), v1b     C6: u2, alpha|u1, -, u2b, u1b     C1 / RO: u2 / v2
    for (int c = tid; c < Nw; c += 256) {
        const int x = i0 - g.w + c;
        float w0 = 0.f, w1 = 0.f, w2 = 0.f, w3 = 0.f, w4 = 0.f;
        if (on_x(x)) {
            if (kRow) {
                w0 = a.v2[bx + x];
                if (kOp == R6) {
                    const float v1 = a.v1[bx + x], v0 = a.v0[bx + x];
                    w1 = kDirect ? v1 : ex2(v1 - w0);
                    w2 = kDirect ? v0 : ex2(v0 - w0);
                    w3 = a.g_v[bx + x];
                    w4 = a.v1b[bx + x];
                }
            } else {
                w0 = a.u2[bx + x];
                if (kOp == C6) {
                    const float u1 = a.u1[bx + x];
                    w1 = kDirect ? u1 : ex2(u1 - w0);
                    w3 = a.u2b[bx + x];
                    w4 = a.u1b[bx + x];
                }
            }
        }
        wv[c] = w0;
        wv[Nw + c] = w1;
        wv[2 * Nw + c] = w2;
        wv[3 * Nw + c] = w3;
        wv[4 * Nw + c] = w4;
    }
    float o2 = 0.f, o1 = 0.f, o0 = 0.f, ob2 = 0.f, ob1 = 0.f;
    if (active) {
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
    }
    // one-reference modifiers of the own index: R6 alpha_i; C6 beta_j, delta_j
    const float ma = active ? ex2(o1 - o2) : 0.f, mb = (active && !kRow) ? ex2(o0 - o2) : 0.f;
    __syncthreads();  // window vectors visible
    float acc = 0.f, dacc = 0.f;
    const int rg = tid >> 3, cg = tid & 7;
    const int wr0 = warp * 16;  // phase-2 rows of this warp: [wr0, wr0 + 16)
    float2 accv[4][CPT / 2];  // column pairs (FFMA2: half the issue slots of the chunk GEMM)
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int e = 0; e < CPT / 2; ++e) accv[q][e] = make_float2(0.f, 0.f);
    for (int j = 0; j < NCH; ++j) {
        const int s = j % NSTG, c0 = j * kWC;
        cp_async_wait<NSTG - 2>();  // this thread's copies of chunk j landed
        __syncthreads();            // everyone's; and every thread is past the previous chunk's phase 2
        if (j + NSTG - 1 < NCH) issue(j + NSTG - 1);  // into the stage the previous chunk used
        else cp_async_commit();
        const float* S = stS(s);
        const float* Z = stZ(s);
        const float* X;  // the chunk's operand rows as f32
        if constexpr (sizeof(TIn) == 4) {
            X = reinterpret_cast<const float*>(stX(s));
        } else {  // one conversion per element instead of one per row group (read again after phase 1's barrier)
            const TIn* Xb = stX(s);
            for (int e = 4 * tid; e < kWC * D; e += 4 * 256)
                *reinterpret_cast<float4*>(Xf + e) = ld4f<TIn>(Xb + e);
            X = Xf;
        }
        // ---- phase 1: weights of this thread's 16 columns of row r (rotated: conflict-free)
        float* wt = WT;  // single buffer: every thread finished the previous chunk's phase 2 (barrier above)
#pragma unroll 4
        for (int jj = 0; jj < kWC / 2; ++jj) {
            const int cl = (r + (kWC / 2) * hh + jj + (r >> 4)) & (kWC - 1);  // conflict-free (kWC = 16)
            const int c = c0 + cl;
            const float s2 = S[r * kWC + cl];
            float wgt = 0.f;
            if (active && (unsigned)(c - r) < (unsigned)Wf && s2 != -INFINITY) {
                const float p = (kOp == RW || kOp == CW) ? 0.f : ex2(s2 + o2 + wv[c]);
                if (kOp == RW || kOp == CW) {  // the band already holds Sbar
                    wgt = Z[r * kWC + cl];
                    if (kOp == RW) dacc += wgt * (s2 * kLn2);
                } else if (kOp == RO) {
                    wgt = p;
                } else if (kOp == C1) {
                    acc += p * Z[r * kWC + cl];
                    wgt = p;
                } else if (kOp == R6) {
                    const float z = Z[r * kWC + cl];
                    if (kDirect) {
                        wgt = sbar_of(true, s2, p, z, o1, o2, wv[2 * Nw + c], wv[Nw + c], wv[c], ob2, ob1,
                                      wv[3 * Nw + c], wv[4 * Nw + c]);
                    } else {  // Sbar = P22 (Z - v2b_j - beta_j u2b_i - alpha_i beta_j v1b_j - alpha_i delta_j u1b_i)
                        const float bj = wv[Nw + c], dj = wv[2 * Nw + c];
                        wgt = p * (z - wv[3 * Nw + c] - bj * ob2 - ma * bj * wv[4 * Nw + c] - ma * dj * ob1);
                    }
                    dacc += wgt * (s2 * kLn2);
                } else {  // C6: own = column j, window = rows i
                    const float z = Z[r * kWC + cl];
                    if (kDirect) {
                        wgt = sbar_of(true, s2, p, z, wv[Nw + c], wv[c], o0, o1, o2, wv[3 * Nw + c], wv[4 * Nw + c],
                                      ob2, ob1);
                        if (a.fuse_c5) acc += ex2(s2 + wv[Nw + c] + o0) * wv[4 * Nw + c];  // C5: P10 u1b
                    } else {  // alpha_i = wv[Nw + c], beta_j = ma, delta_j = mb
                        const float ai = wv[Nw + c];
                        wgt = p * (z - ob2 - ma * wv[3 * Nw + c] - ai * ma * ob1 - ai * mb * wv[4 * Nw + c]);
                        acc += p * ai * wv[4 * Nw + c];  // C5: P22 alpha_i u1b_i (used when fuse_c5)
                    }
                }
            }
            wt[cl * 128 + r] = wgt;
        }
        __syncthreads();  // WT of this chunk complete
        // ---- phase 2: out[4 rg + q][4 cg + 32 m ..] += sum_c W[row][c] X[c][..]
        if (c0 <= wr0 + 15 + 2 * g.w && c0 + kWC - 1 >= wr0) {
            const float* wrow = wt + 4 * rg;
            const float* xr = X + 4 * cg;
#pragma unroll 4
            for (int cl = 0; cl < kWC; ++cl) {
                const float4 w4 = *reinterpret_cast<const float4*>(wrow + cl * 128);
                const float2 wq[4] = {make_float2(w4.x, w4.x), make_float2(w4.y, w4.y), make_float2(w4.z, w4.z),
                                      make_float2(w4.w, w4.w)};
#pragma unroll
                for (int m = 0; m < CPT / 4; ++m) {
                    const float4 x4 = *reinterpret_cast<const float4*>(xr + cl * D + 32 * m);
                    const float2 xa = make_float2(x4.x, x4.y), xb = make_float2(x4.z, x4.w);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        accv[q][2 * m + 0] = ffma2w(xa, wq[q], accv[q][2 * m + 0]);
                        accv[q][2 * m + 1] = ffma2w(xb, wq[q], accv[q][2 * m + 1]);
                    }
                }
            }
        }
    }
    sacc[hh][r] = acc;
    sdacc[hh][r] = dacc;
    __syncthreads();
    if (hh == 0 && i < Lo) {
        if (kOp == C1) a.g_v[bo + i] = active ? sacc[0][r] + sacc[1][r] : 0.f;
        if (kOp == R6 || kOp == RW) a.deps_part[bo + i] = active ? sdacc[0][r] + sdacc[1][r] : 0.f;
        if (kOp == C6 && a.fuse_c5) {  // v0b_j = -delta_j sum_i P22 alpha_i u1b_i  (direct: -sum P10 u1b)
            const float s5 = sacc[0][r] + sacc[1][r];
            a.v0b[bo + i] = !active ? 0.f : kDirect ? -s5 : -ex2(a.v0[bo + i] - a.v2[bo + i]) * s5;
        }
    }
    const float sc = (kOp == C1 || kOp == RO) ? 1.f : g.inv_qk;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int ii = i0 + 4 * rg + q;
        if (ii >= Lo) continue;
#pragma unroll
        for (int m = 0; m < CPT / 4; ++m) {
            const int col = 4 * cg + 32 * m;
            *reinterpret_cast<float4*>(vo + (bo + ii) * D + col) =
                make_float4(accv[q][2 * m].x * sc, accv[q][2 * m].y * sc, accv[q][2 * m + 1].x * sc,
                            accv[q][2 * m + 1].y * sc);
        }
    }
}


// 8 bf16 packed in 4 words (element e in word e >> 1, half e & 1): out[(rot + e) & 7] = in[e]
__device__ __forceinline__ void rot8_bf16(uint32_t (&w)[4], int rot) {
    if (rot & 1) {  // by one element: out[e + 1] = in[e]
        const uint32_t t3 = w[3];
        w[3] = __byte_perm(w[2], w[3], 0x5432);
        w[2] = __byte_perm(w[1], w[2], 0x5432);
        w[1] = __byte_perm(w[0], w[1], 0x5432);
        w[0] = __byte_perm(t3, w[0], 0x5432);
    }
    if (rot & 2) {  // by one word
        const uint32_t t = w[3];
        w[3] = w[2];
        w[2] = w[1];
        w[1] = w[0];
        w[0] = t;
    }
    if (rot & 4) {  // by two words
        uint32_t t = w[0];
        w[0] = w[2];
        w[2] = t;
        t = w[1];
        w[1] = w[3];
        w[3] = t;
    }
}
// ---------------------------------------------------------------------------
// bf16 operands: the window-chunked vector stages with the chunk GEMM on tcgen05.  Per 16-column
// window chunk: phase 1 (as k_bwdW) writes the weights as two bf16 planes W = hi + lo (16 bits of
// mantissa: the split costs <= 2^-17 relative per weight, far inside the bf16 parity bound) in the
// UMMA K-major core-matrix layout, the chunk's 16 operand rows are transposed into the B operand,
// and one elected thread issues two kind::f16 MMAs (M = 128 rows, N = D, K = 16) accumulating
// out[128][D] in TMEM (fp32).  A / B are double-buffered against the MMA (commit -> mbarrier).
// ---------------------------------------------------------------------------
// fp32 operands: W and X both split into three bf16 planes (hi, mid, lo) and the six products of
// order <= 2^-16 (hh, hm, mh, hl, mm, lh), i.e. fp32-accurate products at bf16 tensor rate.
// C1 / RO read one window vector: smaller SMEM, three CTAs per SM
template <int kOp, bool kDirect, int D, int NSTG, class TIn = __nv_bfloat16>
__global__ void __launch_bounds__(256, (kOp == C1 || kOp == RO) ? 3 : 2) k_bwdM(Geo g, BT<TIn> a) {
    constexpr bool kF32 = sizeof(TIn) == 4;
    constexpr int WP = kF32 ? 3 : 2;   // weight planes
    constexpr int XP = kF32 ? 3 : 1;   // operand planes
    constexpr int KC = 16;  // NSTG: cp.async ring depth
    extern __shared__ __align__(1024) uint8_t smm[];
    __shared__ __align__(8) uint64_t mma_bar[2];
    __shared__ uint32_t tmem_sh;
    __shared__ float sacc[2][128], sdacc[2][128];
    constexpr bool kRow = kOp < 10;
    constexpr bool kNeedZ = (kOp == R6 || kOp == C1 || kOp == C6);
    const int Lo = kRow ? g.Lq : g.Lk, Lx = kRow ? g.Lk : g.Lq;
    const int Lro = kRow ? g.Lrq : g.Lrk, Lrx = kRow ? g.Lrk : g.Lrq;
    const int Lpo = kRow ? g.Lqp : g.Lkp;
    const uint8_t* mo = kRow ? g.row_mask : g.col_mask;
    const uint8_t* mx = kRow ? g.col_mask : g.row_mask;
    const int bh = blockIdx.y, i0 = blockIdx.x * 128, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const size_t bo = (size_t)bh * Lro, bx = (size_t)bh * Lrx;
    auto on_o = [&](int k) { return k < Lo && (mo == nullptr || mo[(size_t)(bh / g.H) * Lo + k] != 0); };
    auto on_x = [&](int k) { return k >= 0 && k < Lx && (mx == nullptr || mx[(size_t)(bh / g.H) * Lx + k] != 0); };
    const int r = tid & 127, hh = tid >> 7, i = i0 + r;
    const bool active = on_o(i);
    float* vo = kOp == R6 ? a.dQ : kOp == C1 ? a.dV : kOp == RO ? a.O : a.dK;
    if (!__syncthreads_or(active)) {
        if (hh == 0 && i < Lo) {
            if (kOp == R6) a.deps_part[bo + i] = 0.f;
            if (kOp == C1) a.g_v[bo + i] = 0.f;
            if (kOp == C6 && a.fuse_c5) a.v0b[bo + i] = 0.f;
            for (int x = 0; x < D; ++x) vo[(bo + i) * D + x] = 0.f;
        }
        return;
    }
    const int Wf = g.Wf, Nw = 128 + 2 * g.w, NCH = Nw / KC;
    // SMEM: NSTG stages {S [128][16] f32 | Z [128][16] f32 | X [16][D] bf16}, then A [2][2 planes][128 x 16]
    // bf16, B [2][D x 16] bf16 (K-major core matrices), then the window vectors [5][Nw]
    constexpr int SP = KC + 4;  // strip row pitch (floats): with the rotation below, conflict-free phase-1 reads
    constexpr int STB = (kNeedZ ? 2 : 1) * 128 * SP * 4 + KC * D * (int)sizeof(TIn);  // stage bytes
    constexpr int AB = 128 * KC * 2, BB = D * KC * 2;  // one bf16 plane of A / B
    uint8_t* Abuf = smm + NSTG * STB;                  // [2][WP][AB]
    uint8_t* Bbuf = Abuf + 2 * WP * AB;                // [2][XP][BB]
    float* wv = reinterpret_cast<float*>(Bbuf + 2 * XP * BB);
    const float* Sb = (kRow ? a.S2 : a.S2T) + ((size_t)bh * Lpo + i0) * Wf;
    const float* Zb = kNeedZ ? (kRow ? a.Z : a.ZT) + ((size_t)bh * Lpo + i0) * Wf : nullptr;
    const TIn* osrc = kOp == R6 ? a.K : (kOp == C1) ? a.dO : (kOp == RO) ? a.V : a.Q;
    auto stS = [&](int s) { return reinterpret_cast<float*>(smm + (size_t)s * STB); };
    auto stZ = [&](int s) { return reinterpret_cast<float*>(smm + (size_t)s * STB) + 128 * SP; };
    auto stX = [&](int s) { return reinterpret_cast<TIn*>(smm + (size_t)s * STB + (kNeedZ ? 2 : 1) * 128 * SP * 4); };
    auto issue = [&](int j) {
        const int s = j % NSTG, c0 = j * KC;
        float* S = stS(s);
        float* Z = stZ(s);
        for (int e = tid; e < 128 * (KC / 4); e += 256) {
            const int rr = e / (KC / 4), sg = (e % (KC / 4)) * 4;
            cp_async16(S + rr * SP + sg, Sb + (size_t)rr * (Wf - 1) + c0 + sg, 16u);
            if (kNeedZ) cp_async16(Z + rr * SP + sg, Zb + (size_t)rr * (Wf - 1) + c0 + sg, 16u);
        }
        constexpr int SPR = D * (int)sizeof(TIn) / 16;
        const int xb0 = i0 - g.w + c0;
        TIn* X = stX(s);
        for (int e = tid; e < KC * SPR; e += 256) {
            const int row = e / SPR, sg = e % SPR, x = xb0 + row;
            const bool ok = x >= 0 && x < Lx;
            cp_async16(reinterpret_cast<uint8_t*>(X) + (size_t)row * D * sizeof(TIn) + sg * 16,
                       reinterpret_cast<const uint8_t*>(osrc + (bx + (ok ? x : 0)) * D) + sg * 16, ok ? 16u : 0u);
        }
        cp_async_commit();
    };
    if (warp == 0) {
        sm100::tc_alloc(&tmem_sh, D < 32 ? 32 : D);
        sm100::tc_relinquish();
    }
    if (tid == 0) {
        sm100::mbar_init(&mma_bar[0], 1);
        sm100::mbar_init(&mma_bar[1], 1);
        sm100::fence_mbar_init();
    }
    for (int j = 0; j < NSTG - 1; ++j) {
        if (j < NCH) issue(j);
        else cp_async_commit();
    }
    for (int c = tid; c < Nw; c += 256) {
        const int x = i0 - g.w + c;
        float w0 = 0.f, w1 = 0.f, w2 = 0.f, w3 = 0.f, w4 = 0.f;
        if (on_x(x)) {
            if (kRow) {
                w0 = a.v2[bx + x];
                if (kOp == R6) {
                    const float v1 = a.v1[bx + x], v0 = a.v0[bx + x];
                    w1 = kDirect ? v1 : ex2(v1 - w0);
                    w2 = kDirect ? v0 : ex2(v0 - w0);
                    w3 = a.g_v[bx + x];
                    w4 = a.v1b[bx + x];
                }
            } else {
                w0 = a.u2[bx + x];
                if (kOp == C6) {
                    const float u1 = a.u1[bx + x];
                    w1 = kDirect ? u1 : ex2(u1 - w0);
                    w3 = a.u2b[bx + x];
                    w4 = a.u1b[bx + x];
                }
            }
        }
        wv[c] = w0;
        if (kOp == R6 || kOp == C6) {
            wv[Nw + c] = w1;
            wv[2 * Nw + c] = w2;
            wv[3 * Nw + c] = w3;
            wv[4 * Nw + c] = w4;
        }
    }
    float o2 = 0.f, o1 = 0.f, o0 = 0.f, ob2 = 0.f, ob1 = 0.f;
    if (active) {
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
    }
    const float ma = active ? ex2(o1 - o2) : 0.f, mb = (active && !kRow) ? ex2(o0 - o2) : 0.f;
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const uint32_t tmem = tmem_sh;
    const uint32_t idesc = sm100::make_idesc(128, D, 1u);
    float acc = 0.f, dacc = 0.f;
    // this thread's 16-byte core-matrix row of the A planes: row r, K half hh
    const uint32_t a_off = (uint32_t)((r & ~7) * (KC * 2) + hh * 128 + (r & 7) * 16);
    for (int j = 0; j < NCH; ++j) {
        const int s = j % NSTG, c0 = j * KC, ab = j & 1;
        cp_async_wait<NSTG - 2>();
        __syncthreads();  // chunk j landed everywhere; the previous chunk's phase 1 / B build are done
        if (j + NSTG - 1 < NCH) issue(j + NSTG - 1);
        else cp_async_commit();
        if (j >= 2) sm100::mbar_wait(&mma_bar[ab], (uint32_t)((j - 2) >> 1) & 1u);  // A / B[ab] free again
        const float* S = stS(s);
        const float* Z = stZ(s);
        const TIn* X = stX(s);
        uint8_t* Ap = Abuf + ab * WP * AB;
        uint8_t* Bt = Bbuf + ab * XP * BB;
        // ---- phase 1: 8 weights of row r (columns 8 hh .. 8 hh + 7), rotated reads (conflict-free strip
        // reads), bf16 hi / lo planes; the 8 values are rotated back into column order in registers and
        // stored as ONE 16-byte core-matrix row per plane (2-byte stores were 4-way bank-conflicted)
        const int rot = (r + 2 * (r >> 3)) & 7;
        uint32_t hw[4], mw[4], lw[4];  // bf16 pairs in rotated order: element jj = column (rot + jj) & 7
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
            const int pos = (rot + jj) & 7, cl = 8 * hh + pos;
            const int c = c0 + cl;
            const float s2 = S[r * SP + cl];
            float wgt = 0.f;
            if (active && (unsigned)(c - r) < (unsigned)Wf && s2 != -INFINITY) {
                const float p = ex2(s2 + o2 + wv[c]);
                if (kOp == RO) {
                    wgt = p;
                } else if (kOp == C1) {
                    acc += p * Z[r * SP + cl];
                    wgt = p;
                } else if (kOp == R6) {
                    const float z = Z[r * SP + cl];
                    if (kDirect) {
                        wgt = sbar_of(true, s2, p, z, o1, o2, wv[2 * Nw + c], wv[Nw + c], wv[c], ob2, ob1,
                                      wv[3 * Nw + c], wv[4 * Nw + c]);
                    } else {
                        const float bj = wv[Nw + c], dj = wv[2 * Nw + c];
                        wgt = p * (z - wv[3 * Nw + c] - bj * ob2 - ma * bj * wv[4 * Nw + c] - ma * dj * ob1);
                    }
                    dacc += wgt * (s2 * kLn2);
                } else {  // C6
                    const float z = Z[r * SP + cl];
                    if (kDirect) {
                        wgt = sbar_of(true, s2, p, z, wv[Nw + c], wv[c], o0, o1, o2, wv[3 * Nw + c], wv[4 * Nw + c],
                                      ob2, ob1);
                        if (a.fuse_c5) acc += ex2(s2 + wv[Nw + c] + o0) * wv[4 * Nw + c];
                    } else {
                        const float ai = wv[Nw + c];
                        wgt = p * (z - ob2 - ma * wv[3 * Nw + c] - ai * ma * ob1 - ai * mb * wv[4 * Nw + c]);
                        acc += p * ai * wv[4 * Nw + c];
                    }
                }
            }
            const __nv_bfloat16 hi = __float2bfloat16_rn(wgt);
            const float r1 = wgt - __bfloat162float(hi);  // exact in fp32
            const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
            const uint32_t hb = __bfloat16_as_ushort(hi), mb16 = __bfloat16_as_ushort(mid);
            const uint32_t lb = WP == 3 ? __bfloat16_as_ushort(__float2bfloat16_rn(r1 - __bfloat162float(mid))) : 0u;
            if (jj & 1) {
                hw[jj >> 1] |= hb << 16;
                mw[jj >> 1] |= mb16 << 16;
                lw[jj >> 1] |= lb << 16;
            } else {
                hw[jj >> 1] = hb;
                mw[jj >> 1] = mb16;
                lw[jj >> 1] = lb;
            }
        }
        rot8_bf16(hw, rot);
        rot8_bf16(mw, rot);
        *reinterpret_cast<uint4*>(Ap + a_off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        *reinterpret_cast<uint4*>(Ap + AB + a_off) = make_uint4(mw[0], mw[1], mw[2], mw[3]);
        if (WP == 3) {
            rot8_bf16(lw, rot);
            *reinterpret_cast<uint4*>(Ap + 2 * AB + a_off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
        }
        // ---- B operand: X^T of the chunk, K-major core matrices (n = output column, k = window column)
        for (int u = tid; u < D * 2; u += 256) {
            const int n = u >> 1, kc = u & 1;
            const uint32_t boff = (n & ~7) * (KC * 2) + kc * 128 + (n & 7) * 16;
            if constexpr (!kF32) {
                __align__(16) __nv_bfloat16 e8[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) e8[e] = X[(kc * 8 + e) * D + n];
                *reinterpret_cast<uint4*>(Bt + boff) = *reinterpret_cast<const uint4*>(e8);
            } else {
                __align__(16) __nv_bfloat16 h8[8], m8[8], l8[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const float x = X[(kc * 8 + e) * D + n];
                    h8[e] = __float2bfloat16_rn(x);
                    const float r1 = x - __bfloat162float(h8[e]);
                    m8[e] = __float2bfloat16_rn(r1);
                    l8[e] = __float2bfloat16_rn(r1 - __bfloat162float(m8[e]));
                }
                *reinterpret_cast<uint4*>(Bt + boff) = *reinterpret_cast<const uint4*>(h8);
                *reinterpret_cast<uint4*>(Bt + BB + boff) = *reinterpret_cast<const uint4*>(m8);
                *reinterpret_cast<uint4*>(Bt + 2 * BB + boff) = *reinterpret_cast<const uint4*>(l8);
            }
        }
        sm100::fence_proxy_async_smem();  // generic SMEM writes -> visible to the tensor core
        __syncthreads();
        if (warp == 0) {
            sm100::tc_fence_after();
            if (sm100::elect_one()) {
                // (A plane, B plane) products: bf16 operands (hi, lo) x X; fp32 the six of order <= 2^-16
                constexpr int NP = kF32 ? 6 : 2;
                constexpr int pa_[6] = {0, 0, 1, 0, 1, 2};
                constexpr int pb_[6] = {0, 1, 0, 2, 1, 0};
                constexpr int qa_[2] = {0, 1};
#pragma unroll
                for (int pr = 0; pr < NP; ++pr) {
                    const int pa = kF32 ? pa_[pr] : qa_[pr], pb = kF32 ? pb_[pr] : 0;
                    sm100::mma_bf16(tmem, sm100::make_desc(sm100::smem_u32(Ap + pa * AB), 128, 8 * KC * 2),
                                    sm100::make_desc(sm100::smem_u32(Bt + pb * BB), 128, 8 * KC * 2), idesc,
                                    (j > 0 || pr > 0) ? 1u : 0u);
                }
                sm100::tc_commit(&mma_bar[ab]);
            }
            __syncwarp();
        }
    }
    // the last commit covers every earlier MMA
    sm100::mbar_wait(&mma_bar[(NCH - 1) & 1], (uint32_t)((NCH - 1) >> 1) & 1u);
    sm100::tc_fence_after();
    sacc[hh][r] = acc;
    sdacc[hh][r] = dacc;
    __syncthreads();
    if (hh == 0 && i < Lo) {
        if (kOp == C1) a.g_v[bo + i] = active ? sacc[0][r] + sacc[1][r] : 0.f;
        if (kOp == R6) a.deps_part[bo + i] = active ? sdacc[0][r] + sdacc[1][r] : 0.f;
        if (kOp == C6 && a.fuse_c5) {
            const float s5 = sacc[0][r] + sacc[1][r];
            a.v0b[bo + i] = !active ? 0.f : kDirect ? -s5 : -ex2(a.v0[bo + i] - a.v2[bo + i]) * s5;
        }
    }
    if (warp < 4) {  // TMEM lane quadrant = warp: thread r holds output row r
        const float sc = (kOp == C1 || kOp == RO) ? 1.f : g.inv_qk;
#pragma unroll
        for (int h = 0; h < D / 32; ++h) {
            float v[32];
            sm100::tc_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(32 * h), v);
            sm100::tc_wait_ld();
            if (i < Lo) {
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    *reinterpret_cast<float4*>(vo + (bo + i) * D + 32 * h + 4 * q) =
                        make_float4(v[4 * q] * sc, v[4 * q + 1] * sc, v[4 * q + 2] * sc, v[4 * q + 3] * sc);
            }
        }
    }
    sm100::tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        sm100::tc_fence_after();
        sm100::tc_dealloc(tmem, D < 32 ? 32 : D);
    }
}

template <int D, class TIn>
static size_t bwdM_smem_bytes(const Geo& g, bool z, int nstg, int nvec) {
    const int Nw = 128 + 2 * g.w;
    const int wp = sizeof(TIn) == 4 ? 3 : 2, xp = sizeof(TIn) == 4 ? 3 : 1;
    return (size_t)nstg * ((z ? 2 : 1) * 128 * 20 * 4 + 16 * D * sizeof(TIn)) + (size_t)2 * wp * 128 * 16 * 2 +
           (size_t)2 * xp * D * 16 * 2 + (size_t)nvec * Nw * 4 + 1024;
}

// Window-chunked scalar sweeps (R1, R12, R2, R4, C3, C5) over the sheared band strips, for the bands
// whose 128-row tile does not fit SMEM: 2 threads per row (rotated columns), NSTG-deep cp.async ring
// of [128][32] S (and Z) strips, one barrier per chunk, 2-3 CTAs per SM.
template <int kOp, bool kDirect, class TIn, int NSTG>
__global__ void __launch_bounds__(256, 4) k_sweepW(Geo g, BT<TIn> a) {
    extern __shared__ __align__(128) float smw[];
    __shared__ float sacc[2][128], sacc2[2][128];
    constexpr bool kRow = kOp < 10;
    constexpr bool kNeedZ = (kOp == R1 || kOp == R12);
    const int Lo = kRow ? g.Lq : g.Lk, Lx = kRow ? g.Lk : g.Lq;
    const int Lro = kRow ? g.Lrq : g.Lrk, Lrx = kRow ? g.Lrk : g.Lrq;
    const int Lpo = kRow ? g.Lqp : g.Lkp;
    const uint8_t* mo = kRow ? g.row_mask : g.col_mask;
    const uint8_t* mx = kRow ? g.col_mask : g.row_mask;
    const int bh = blockIdx.y, i0 = blockIdx.x * 128, tid = threadIdx.x;
    const size_t bo = (size_t)bh * Lro, bx = (size_t)bh * Lrx;
    auto on_o = [&](int k) { return k < Lo && (mo == nullptr || mo[(size_t)(bh / g.H) * Lo + k] != 0); };
    auto on_x = [&](int k) { return k >= 0 && k < Lx && (mx == nullptr || mx[(size_t)(bh / g.H) * Lx + k] != 0); };
    const int r = tid & 127, hh = tid >> 7, i = i0 + r;
    const bool active = on_o(i);
    auto put = [&](float val) {
        if (kOp == R1 || kOp == R12) a.g_u[bo + i] = val;
        if (kOp == R2) a.u2b[bo + i] = val;
        if (kOp == R4) a.u1b[bo + i] = val;
        if (kOp == C3) a.v1b[bo + i] = val;
        if (kOp == C5) a.v0b[bo + i] = val;
    };
    if (!__syncthreads_or(active)) {
        if (hh == 0 && i < Lo) {
            put(0.f);
            if (kOp == R12) a.u2b[bo + i] = 0.f;
        }
        return;
    }
    const int Wf = g.Wf, Nw = 128 + 2 * g.w, NCH = Nw / kWC;
    constexpr int STF = (kNeedZ ? 2 : 1) * 128 * kWC;
    float* wv = smw + NSTG * STF;  // [4][Nw]: x2, x1, g_v|u2b, v1b|u1b
    const float* Sb = (kRow ? a.S2 : a.S2T) + ((size_t)bh * Lpo + i0) * Wf;
    const float* Zb = kNeedZ ? a.Z + ((size_t)bh * Lpo + i0) * Wf : nullptr;
    auto issue = [&](int j) {
        float* S = smw + (size_t)(j % NSTG) * STF;
        const int c0 = j * kWC;
        for (int e = tid; e < 128 * (kWC / 4); e += 256) {
            const int rr = e / (kWC / 4), sg = (e % (kWC / 4)) * 4;
            cp_async16(S + rr * kWC + sg, Sb + (size_t)rr * (Wf - 1) + c0 + sg, 16u);
            if (kNeedZ) cp_async16(S + 128 * kWC + rr * kWC + sg, Zb + (size_t)rr * (Wf - 1) + c0 + sg, 16u);
        }
        cp_async_commit();
    };
    for (int j = 0; j < NSTG - 1; ++j) {
        if (j < NCH) issue(j);
        else cp_async_commit();
    }
    for (int c = tid; c < Nw; c += 256) {
        const int x = i0 - g.w + c;
        float w0 = 0.f, w1 = 0.f, w3 = 0.f, w4 = 0.f;
        if (on_x(x)) {
            if (kRow) {
                w0 = a.v2[bx + x];
                w1 = a.v1[bx + x];
                if (kOp == R2 || kOp == R12) w3 = a.g_v[bx + x];
                if (kOp == R4) w4 = a.v1b[bx + x];
            } else {
                w0 = a.u2[bx + x];
                w1 = a.u1[bx + x];
                if (kOp == C3) w3 = a.u2b[bx + x];
                if (kOp == C5) w4 = a.u1b[bx + x];
            }
            // one-reference R4 / C5: the window side's modifier beta_j / alpha_i folded in once per column
            if (!kDirect && (kOp == R4 || kOp == C5)) w4 *= ex2(w1 - w0);
        }
        wv[c] = w0;
        wv[Nw + c] = w1;
        wv[2 * Nw + c] = w3;
        wv[3 * Nw + c] = w4;
    }
    float o2 = 0.f, o1 = 0.f, o0 = 0.f;
    if (active) {
        o2 = kRow ? a.u2[bo + i] : a.v2[bo + i];
        o1 = kRow ? a.u1[bo + i] : a.v1[bo + i];
        if (!kRow) o0 = a.v0[bo + i];
    }
    float acc = 0.f, acc2 = 0.f;
    for (int j = 0; j < NCH; ++j) {
        cp_async_wait<NSTG - 2>();
        __syncthreads();  // chunk j visible (and the window vectors, j = 0); chunk j - 1 fully consumed
        if (j + NSTG - 1 < NCH) issue(j + NSTG - 1);
        else cp_async_commit();
        const float* S = smw + (size_t)(j % NSTG) * STF;
        const float* Z = S + 128 * kWC;
        const int c0 = j * kWC;
        if (!active || c0 > r + 2 * g.w || c0 + kWC - 1 < r) continue;  // this row's band misses the chunk
#pragma unroll 4
        for (int jj = 0; jj < kWC / 2; ++jj) {
            const int cl = (r + (kWC / 2) * hh + jj + (r >> 4)) & (kWC - 1);  // conflict-free (kWC = 16)
            const int c = c0 + cl;
            const float s2 = S[r * kWC + cl];
            if ((unsigned)(c - r) >= (unsigned)Wf || s2 == -INFINITY) continue;
            const float x2 = wv[c], x1 = wv[Nw + c];
            const float p = ex2(s2 + o2 + x2);
            if (kOp == R1) acc += p * Z[r * kWC + cl];
            else if (kOp == R12) {
                acc += p * Z[r * kWC + cl];
                acc2 += p * wv[2 * Nw + c];
            } else if (kOp == R2) acc += p * wv[2 * Nw + c];
            else if (kOp == R4) acc += kDirect ? ex2(s2 + o1 + x1) * wv[3 * Nw + c] : p * wv[3 * Nw + c];
            else if (kOp == C3) acc += (kDirect ? ex2(s2 + x2 + o1) : p) * wv[2 * Nw + c];
            else acc += kDirect ? ex2(s2 + x1 + o0) * wv[3 * Nw + c] : p * wv[3 * Nw + c];
        }
    }
    sacc[hh][r] = acc;
    sacc2[hh][r] = acc2;
    __syncthreads();
    if (hh == 0 && i < Lo) {
        acc = sacc[0][r] + sacc[1][r];
        acc2 = sacc2[0][r] + sacc2[1][r];
        if (kOp == R12) a.u2b[bo + i] = active ? acc - acc2 : 0.f;
        float val = 0.f;
        if (active) {
            if (kOp == R1 || kOp == R12) val = acc;
            if (kOp == R2) val = a.g_u[bo + i] - acc;
            if (kOp == R4) val = kDirect ? -acc : -ex2(o1 - o2) * acc;
            if (kOp == C3) val = kDirect ? -acc : -ex2(o1 - o2) * acc;
            if (kOp == C5) val = kDirect ? -acc : -ex2(o0 - o2) * acc;
        }
        put(val);
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
    return (size_t)2 * 128 * g.Wf * 4 + (size_t)((5 * Nw + 3) & ~3) * 4 + (size_t)Nw * D * 4 + 64;
}

// SMEM of one k_bwdT stage: S tile, Z tile (R1 / C1 / R6 / C6), window vectors, operand rows (vector stages)
static size_t bwdT_op_smem(const Geo& g, int op, int D) {
    const int Nw = 128 + 2 * g.w;
    const bool z = (op == R1 || op == R12 || op == R6 || op == C1 || op == C6);
    const bool vec = (op == R6 || op == C1 || op == C6 || op == RO);
    return (size_t)(z ? 2 : 1) * 128 * g.Wf * 4 + (size_t)((5 * Nw + 3) & ~3) * 4 + (vec ? (size_t)Nw * (D + 4) * 4 : 0) + 64;
}

// SMEM of the wide-band kernels (k_bwdS scalar stages, k_bwdG vector stages) at RB rows per CTA
static size_t wide_smem(const Geo& g, int op, int D, int esz, int RB) {
    const int Nw = RB + 2 * g.w;
    const bool vec = (op == R6 || op == C1 || op == C6 || op == RO || op == RW || op == CW);
    const bool z = vec ? (op != RO) : (op == R1 || op == R12);
    return (size_t)(z ? 2 : 1) * RB * g.Wf * 4 + (size_t)((5 * Nw + 3) & ~3) * 4 + (vec ? (size_t)Nw * D * esz : 0) + 64;
}

// rows per CTA for a stage: 128 (the k_bwdT / k_bwdV tiles or k_bwdG<128>), else 64 / 32; 0 = none fits
static int pick_rb(const Geo& g, int op, int D, int esz) {
    constexpr size_t kMax = 227 * 1024;
    const bool vec = (op == R6 || op == C1 || op == C6 || op == RO || op == RW || op == CW);
    if (!vec && bwdT_op_smem(g, op, D) <= kMax) return 128;
    for (int RB : {128, 64, 32}) {
        if (vec && D == 32 && RB == 32) continue;
        if (g.dustbin && RB < 128) continue;  // the spoke cells live in the 128-row kernels
        if (!vec && RB == 128) continue;      // covered above
        if (wide_smem(g, op, D, esz, RB) <= kMax) return RB;
    }
    return 0;
}

bool bwdT_supported(const Geo& g) {
    if (!(g.d == 32 || g.d == 64 || g.d == 128)) return false;
    const int esz = g.esz ? g.esz : 4;
    const bool narrow = g.d <= 64 && bwdT_smem_bytes(g) <= 227 * 1024;  // k_bwdV path for the vector stages
    for (int op : {R12, R4, C3, C5})
        if (!pick_rb(g, op, g.d, esz)) return false;
    if (!narrow)
        for (int op : {R6, C6, C1, RO})
            if (!pick_rb(g, op, g.d, esz)) return false;
    return true;
}

template <int kOp, bool kDirect, int D, class TIn, int RB>
static cudaError_t run_wide(const Geo& g, const BT<TIn>& a, cudaStream_t s) {
    constexpr bool kVec = (kOp == R6 || kOp == C1 || kOp == C6 || kOp == RO || kOp == RW || kOp == CW);
    const bool row = kOp < 10;
    const int n = row ? g.Lq : g.Lk;
    const size_t smem = wide_smem(g, kOp, D, (int)sizeof(TIn), RB);
    if constexpr (kVec) {
        if constexpr (D == 32 && RB == 32) {
            return cudaErrorNotSupported;
        } else {
            auto k = k_bwdG<kOp, kDirect, D, TIn, RB>;
            cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
            k<<<dim3((n + RB - 1) / RB, g.BH), 256, smem, s>>>(g, a);
        }
    } else {
        auto k = k_bwdS<kOp, kDirect, RB, TIn>;
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        k<<<dim3((n + RB - 1) / RB, g.BH), 128, smem, s>>>(g, a);
    }
    return cudaGetLastError();
}

template <int kOp, bool kDirect, int D, class TIn>
static cudaError_t run_op(const Geo& g, const BT<TIn>& a, cudaStream_t s) {
    const bool row = kOp < 10;
    constexpr bool kVec = (kOp == R6 || kOp == C1 || kOp == C6 || kOp == RO || kOp == RW || kOp == CW);
    const bool narrow_ok = kVec && D <= 64 && bwdT_smem_bytes(g) <= 227 * 1024 && !getenv("ST_NO_BWDV");
    if constexpr (kVec) {
        // wide bands (no 128-row band tile in SMEM): the window-chunked vector stage over sheared band
        // strips; narrow bands keep the 128-row tile kernel (the strips would read the 2x wider window)
        if constexpr (kOp == R6 || kOp == C1 || kOp == C6 || kOp == RO) {
            // chunk GEMM on tcgen05 for bf16 operands on wide bands.  The fp32 variant (3-plane split,
            // six products) passes parity but measured slower than the CUDA-core kernels on config 2
            // (0.368 vs 0.288 ms backward), so it is opt-in (ST_BWDM_F32=1)
            const bool f32 = std::is_same<TIn, float>::value;
            static const bool f32_on = getenv("ST_BWDM_F32") != nullptr;
            if ((f32 ? f32_on : !narrow_ok) && bwdW_supported(g) && !getenv("ST_NO_BWDM")) {
                constexpr bool kZ = (kOp == R6 || kOp == C1 || kOp == C6);
                static const int nsm = getenv("ST_BWDM_NSTG") ? atoi(getenv("ST_BWDM_NSTG")) : 2;
                const int ns = nsm >= 6 ? 6 : nsm >= 4 ? 4 : 2;
                const size_t smem = bwdM_smem_bytes<D, TIn>(g, kZ, ns, (kOp == R6 || kOp == C6) ? 5 : 1);
                auto k = ns == 6 ? k_bwdM<kOp, kDirect, D, 6, TIn>
                                 : ns == 4 ? k_bwdM<kOp, kDirect, D, 4, TIn> : k_bwdM<kOp, kDirect, D, 2, TIn>;
                cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                if (e != cudaSuccess) return e;
                const int n = row ? g.Lq : g.Lk;
                k<<<dim3((n + 127) / 128, g.BH), 256, smem, s>>>(g, a);
                return cudaGetLastError();
            }
        }
        if (!narrow_ok && bwdW_supported(g)) {
            constexpr bool kZ = (kOp == R6 || kOp == C1 || kOp == C6 || kOp == RW || kOp == CW);
            static const int nstg = getenv("ST_BWDW_NSTG") ? atoi(getenv("ST_BWDW_NSTG")) : 2;
            const int ns = nstg >= 4 ? 4 : nstg == 3 ? 3 : 2;
            const size_t smem = bwdW_smem_bytes<D, TIn>(g, kZ, ns);
            if (smem <= 227 * 1024) {
                auto k = ns == 4 ? k_bwdW<kOp, kDirect, D, TIn, 4>
                                 : ns == 3 ? k_bwdW<kOp, kDirect, D, TIn, 3> : k_bwdW<kOp, kDirect, D, TIn, 2>;
                cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                if (e != cudaSuccess) return e;
                const int n = row ? g.Lq : g.Lk;
                k<<<dim3((n + 127) / 128, g.BH), 256, smem, s>>>(g, a);
                return cudaGetLastError();
            }
        }
    }
    if (narrow_ok) {
        // 128-row weights + register-tiled band GEMM (operands as f32)
        const size_t smem = bwdT_smem_bytes(g);
        auto k = k_bwdV<kOp, kDirect, D, TIn>;
        // set on every launch: the attribute is per device, and callers may drive several devices / threads
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        const int n = row ? g.Lq : g.Lk;
        k<<<dim3((n + 127) / 128, g.BH), 256, smem, s>>>(g, a);
        return cudaGetLastError();
    }
    if constexpr (!kVec) {
        // scalar sweeps over bands whose 128-row tile does not fit SMEM: window-chunked strips
        if ((bwdT_op_smem(g, kOp, D) > 227 * 1024 || g.Wf > 129) && bwdW_supported(g)) {
            constexpr bool kZ = (kOp == R1 || kOp == R12);
            static const int ns_env = getenv("ST_SWEEPW_NSTG") ? atoi(getenv("ST_SWEEPW_NSTG")) : 3;
            const int NS = ns_env >= 4 ? 4 : ns_env == 2 ? 2 : 3;
            const size_t smem = ((size_t)NS * (kZ ? 2 : 1) * 128 * kWC + 4 * (size_t)(128 + 2 * g.w)) * 4 + 128;
            auto k = NS == 4 ? k_sweepW<kOp, kDirect, TIn, 4> : NS == 2 ? k_sweepW<kOp, kDirect, TIn, 2> : k_sweepW<kOp, kDirect, TIn, 3>;
            cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
            const int n = row ? g.Lq : g.Lk;
            k<<<dim3((n + 127) / 128, g.BH), 256, smem, s>>>(g, a);
            return cudaGetLastError();
        }
    }
    const int rb = pick_rb(g, kOp, D, (int)sizeof(TIn));
    if (rb == 0) return cudaErrorNotSupported;
    if (kVec || rb != 128) {
        if (rb == 128) return run_wide<kOp, kDirect, D, TIn, 128>(g, a, s);
        if (rb == 64) return run_wide<kOp, kDirect, D, TIn, 64>(g, a, s);
        return run_wide<kOp, kDirect, D, TIn, 32>(g, a, s);
    }
    const size_t smem = bwdT_op_smem(g, kOp, D);
    auto k = k_bwdT<kOp, kDirect, D, TIn>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int n = row ? g.Lq : g.Lk;
    k<<<dim3((n + 127) / 128, g.BH), 128, smem, s>>>(g, a);
    return cudaGetLastError();
}

template <bool kDirect, int D, class TIn>
static cudaError_t run_all(const Geo& g, const BwdPtrs& p, const BwdTPtrs& t, int dtype, cudaStream_t s,
                           long long& launches, const BwdHook* hook) {
    auto halo = [&](int kind, float* vec) {  // let the caller complete the vector's halo (sequence sharding)
        if (hook && hook->fn) hook->fn(hook->user, kind, vec, kind == 0 ? hook->nq : hook->nk, (void*)s);
    };
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
    a.fuse_c5 = 0;
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
    if (g.dustbin) {  // the dustbin row/column stages interleave with R1 / R2
        ST_RUN(R1);
        ST_RUN(C1);
        ST_DUST(0);
        ST_RUN(R2);
        ST_DUST(1);
    } else {  // C1 first, then R1 + R2 in one sweep
        ST_RUN(C1);
        halo(1, a.g_v);
        ST_RUN(R12);
        halo(0, a.u2b);
    }
    ST_RUN(C3);
    ST_DUST(2);
    halo(1, a.v1b);
    ST_RUN(R4);
    ST_DUST(3);
    halo(0, a.u1b);
    a.fuse_c5 = g.dustbin ? 0 : 1;  // the C5 sweep rides in C6 (same tiles and window vectors)
    if (!a.fuse_c5) {
        ST_RUN(C5);
        ST_DUST(4);
    }
    if (!g.dustbin && !getenv("ST_NO_FORK")) {
        // R6 (dQ, d_eps) and C6 (dK, v0b) read the same finished vectors and write disjoint outputs:
        // run them on two streams so each fills the other's partial last wave (event fork / join,
        // captured as graph dependencies)
        // side stream and events per (thread, device): a process may drive several GPUs
        constexpr int kMaxDev = 64;
        static thread_local cudaStream_t sides[kMaxDev] = {};
        static thread_local cudaEvent_t forks[kMaxDev] = {}, joins[kMaxDev] = {};
        int dev = 0;
        if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
        if (dev < 0 || dev >= kMaxDev) return cudaErrorInvalidDevice;
        if (!sides[dev]) {
            if ((e = cudaStreamCreateWithFlags(&sides[dev], cudaStreamNonBlocking)) != cudaSuccess) return e;
            if ((e = cudaEventCreateWithFlags(&forks[dev], cudaEventDisableTiming)) != cudaSuccess) return e;
            if ((e = cudaEventCreateWithFlags(&joins[dev], cudaEventDisableTiming)) != cudaSuccess) return e;
        }
        cudaStream_t side = sides[dev];
        cudaEvent_t ev_fork = forks[dev], ev_join = joins[dev];
        if ((e = cudaEventRecord(ev_fork, s)) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(side, ev_fork, 0)) != cudaSuccess) return e;
        if ((e = run_op<C6, kDirect, D, TIn>(g, a, side)) != cudaSuccess) return e;
        ++launches;
        ST_RUN(R6);
        if ((e = cudaEventRecord(ev_join, side)) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(s, ev_join, 0)) != cudaSuccess) return e;
    } else {
        ST_RUN(R6);
        ST_RUN(C6);
        ST_DUST(5);
    }
#undef ST_RUN
#undef ST_DUST
    return cudaSuccess;
}

// ---------------------------------------------------------------------------
// Generic-R tail adjoint (adjoint.hpp:132-200).  The R=2 path never materialises the score
// cotangent; for any other depth it is built once in place over the Z band:
//   Sbar = P^(RR) (.) Z - sum_{t=1..R} [ P^(h,h) (.) vb_t,j + P^(h,h-1) (.) ub_t,i ],  h = T+t,
// then transposed and contracted by the RW (dQ, d_eps) / CW (dK) band GEMMs.  2R+1 exps per cell.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_sbar_band(Geo g, TailPtrs tp, const float* __restrict__ S2,
                                                   float* __restrict__ Z) {
    const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const long total = (long)g.BH * g.Lqp * g.Wf;
    if (t >= total) return;
    const int k = (int)(t % g.Wf);
    const long ri = t / g.Wf;
    const int i = (int)(ri % g.Lqp), bh = (int)(ri / g.Lqp);
    const int j = i - g.w + k;
    const float s2 = S2[t];
    float out = 0.f;
    if (i < g.Lq && j >= 0 && j < g.Lk && s2 != -INFINITY) {
        const size_t oi = (size_t)bh * g.Lrq + i, oj = (size_t)bh * g.Lrk + j;
        const int R = tp.R;
        const float uR = tp.u[R][oi];
        float acc = ex2(s2 + uR + tp.v[R][oj]) * Z[t];
        for (int q = R; q >= 1; --q) {
            const float uq = tp.u[q][oi];
            acc -= ex2(s2 + uq + tp.v[q][oj]) * tp.vb[q][oj];
            acc -= ex2(s2 + uq + tp.v[q - 1][oj]) * tp.ub[q][oi];
        }
        out = acc;
    }
    Z[t] = out;
}

template <int D, class TIn>
static cudaError_t run_tail(const Geo& g, const TailPtrs& tp, const float* S2, const float* S2T, float* Z, float* ZT,
                            const void* Q, const void* K, const void* V, const void* dO, float* dQ, float* dK,
                            float* dV, float* deps_part, cudaStream_t s, long long& launches) {
    const int R = tp.R;
    BT<TIn> a{};
    a.S2 = S2;
    a.S2T = S2T;
    a.Z = Z;
    a.ZT = ZT;
    a.Q = (const TIn*)Q;
    a.K = (const TIn*)K;
    a.V = (const TIn*)V;
    a.dO = (const TIn*)dO;
    a.dQ = dQ;
    a.dK = dK;
    a.dV = dV;
    a.deps_part = deps_part;
    a.fuse_c5 = 0;
    // a stage that reads one plan P^(hu,hv) binds every dual slot of its side to that step, so the
    // one-reference ratios alpha / beta / delta are exactly 1
    auto bind = [&](int hu, int hv) {
        a.u1 = a.u2 = tp.u[hu];
        a.v0 = a.v1 = a.v2 = tp.v[hv];
    };
    cudaError_t e;
#define ST_RUN(op)                                                                           do {                                                                                         if ((e = run_op<op, false, D, TIn>(g, a, s)) != cudaSuccess) return e;                   ++launches;                                                                          } while (0)
    // C1: vb_R = g_v = colsum(P^(RR) (.) Z), dV = P^(RR)^T dO
    bind(R, R);
    a.g_v = tp.vb[R];
    ST_RUN(C1);
    if (R == 0 && tp.eta_u) {  // base cotangent u part: g_u = rowsum(P^(TT) (.) Z)
        a.g_u = tp.eta_u;
        ST_RUN(R1);
    }
    if (R >= 1) {  // ub_R = g_u - P^(RR) vb_R
        a.g_u = tp.g_u;
        a.u2b = tp.ub[R];
        ST_RUN(R12);
        for (int q = R; q >= 1; --q) {
            bind(q, q - 1);  // vb_{q-1} = -P^(h,h-1)^T ub_q
            a.u2b = tp.ub[q];
            a.v1b = tp.vb[q - 1];
            ST_RUN(C3);
            if (q >= 2) {  // ub_{q-1} = -P^(h-1,h-1) vb_{q-1}
                bind(q - 1, q - 1);
                a.v1b = tp.vb[q - 1];
                a.u1b = tp.ub[q - 1];
                ST_RUN(R4);
            }
        }
    }
    const long total = (long)g.BH * g.Lqp * g.Wf;
    k_sbar_band<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(g, tp, S2, Z);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    ++launches;
    if ((e = launch_transpose_band(g, Z, ZT, s, 0.f)) != cudaSuccess) return e;
    bind(R, R);
    ST_RUN(RW);
    ST_RUN(CW);
#undef ST_RUN
    return cudaSuccess;
}

cudaError_t launch_tail_adjoint(const Geo& g, int dtype, const TailPtrs& tp, const float* S2, const float* S2T,
                                float* Z, float* ZT, const void* Q, const void* K, const void* V, const void* dO,
                                float* dQ, float* dK, float* dV, float* deps_part, cudaStream_t s,
                                long long& launches) {
    if (tp.R < 0 || tp.R > kMaxTailSteps || g.dustbin) return cudaErrorNotSupported;
#define ST_TAIL(D)                                                                                              return dtype == 0 ? run_tail<D, float>(g, tp, S2, S2T, Z, ZT, Q, K, V, dO, dQ, dK, dV, deps_part, s, launches)                       : run_tail<D, __nv_bfloat16>(g, tp, S2, S2T, Z, ZT, Q, K, V, dO, dQ, dK, dV, deps_part, s, launches);
    if (g.d == 32) { ST_TAIL(32) }
    if (g.d == 64) { ST_TAIL(64) }
    ST_TAIL(128)
#undef ST_TAIL
}

// ---------------------------------------------------------------------------
// base_solve_vjp (certificates.hpp:25-70): the reverse recurrences through the T base steps.  Step h
// (band at eps_h): abar = ubar - P^(h,h) vbar (row stage), vbar <- -P^(h,h-1)^T abar (column stage),
// and the raw-score cotangent band gains -(eps/eps_h) [P^(h,h) (.) vbar_j + P^(h,h-1) (.) abar_i]
// (k_base_acc; stored times eps so the RW / CW contraction's 1/(sqrt(d) eps) gives grad = raw_bar K/sqrt(d)).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_base_acc(Geo g, const float* __restrict__ S2, float* __restrict__ A,
                                                  const float* __restrict__ uh, const float* __restrict__ vh,
                                                  const float* __restrict__ vhm1, const float* __restrict__ vb,
                                                  const float* __restrict__ ab, float coef, int init) {
    const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const long total = (long)g.BH * g.Lqp * g.Wf;
    if (t >= total) return;
    const int k = (int)(t % g.Wf);
    const long ri = t / g.Wf;
    const int i = (int)(ri % g.Lqp), bh = (int)(ri / g.Lqp);
    const int j = i - g.w + k;
    const float s2 = S2[t];
    float acc = init ? 0.f : A[t];
    if (i < g.Lq && j >= 0 && j < g.Lk && s2 != -INFINITY) {
        const size_t oi = (size_t)bh * g.Lrq + i, oj = (size_t)bh * g.Lrk + j;
        const float u = uh[oi];
        acc -= coef * (ex2(s2 + u + vh[oj]) * vb[oj] + ex2(s2 + u + vhm1[oj]) * ab[oi]);
    }
    A[t] = acc;
}

template <int D, class TIn>
static cudaError_t run_base_vjp(const Geo& g, int dtype, const BaseVjpPtrs& p, cudaStream_t s, long long& launches) {
    const size_t nq = (size_t)g.BH * g.Lrq, nk = (size_t)g.BH * g.Lrk;
    auto hu = [&](int h) { return p.hu + (size_t)h * nq; };
    auto hv = [&](int h) { return p.hv + (size_t)h * nk; };
    BT<TIn> a{};
    a.Q = (const TIn*)p.Q;
    a.K = (const TIn*)p.K;
    a.dQ = p.dQ;
    a.dK = p.dK;
    a.deps_part = p.deps_part;
    a.fuse_c5 = 0;
    cudaError_t e;
#define ST_RUN(op)                                                              \
    do {                                                                        \
        if ((e = run_op<op, false, D, TIn>(g, a, s)) != cudaSuccess) return e; \
        ++launches;                                                             \
    } while (0)
    float band_lam = 0.f;
    const float* vcur = p.eta_v;
    const long total = (long)g.BH * g.Lqp * g.Wf;
    for (int h = p.T; h >= 1; --h) {
        const float lam = p.lam[h];
        Geo gs = g;
        gs.c2 = g.c2 * lam;
        if (lam != band_lam) {  // scores at this step's stage temperature
            if (band_dual_supported(g)) {
                if ((e = launch_band_dual(gs, dtype, false, p.Q, p.K, p.S2, p.S2T, s)) != cudaSuccess) return e;
            } else {
                if ((e = launch_scores(gs, dtype, p.Q, p.K, p.S2, s)) != cudaSuccess) return e;
                if ((e = launch_transpose_band(g, p.S2, p.S2T, s, -INFINITY)) != cudaSuccess) return e;
            }
            band_lam = lam;
        }
        a.S2 = p.S2;
        a.S2T = p.S2T;
        // abar = ubar - P^(h,h) vbar: R2 with g_u = ubar (step T: eta_u) ...
        a.u1 = a.u2 = hu(h);
        a.v0 = a.v1 = a.v2 = hv(h);
        a.g_v = const_cast<float*>(vcur);
        a.g_u = (h == p.T && p.eta_u) ? const_cast<float*>(p.eta_u) : p.zero_u;
        a.u2b = p.ab;
        ST_RUN(R2);
        float* vnext = p.vb[h & 1];
        k_base_acc<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(gs, p.S2, p.A, hu(h), hv(h), hv(h - 1), vcur, p.ab,
                                                                   lam, h == p.T);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        ++launches;
        // ... vbar <- -P^(h,h-1)^T abar: C3 on the plan (u_h, v_{h-1})
        a.v0 = a.v1 = a.v2 = hv(h - 1);
        a.u2b = p.ab;
        a.v1b = vnext;
        ST_RUN(C3);
        vcur = vnext;
    }
    if ((e = launch_transpose_band(g, p.A, p.AT, s, 0.f)) != cudaSuccess) return e;
    a.S2 = p.S2;
    a.S2T = p.S2T;
    a.Z = p.A;
    a.ZT = p.AT;
    a.u1 = a.u2 = hu(p.T);
    a.v0 = a.v1 = a.v2 = hv(p.T);
    ST_RUN(RW);
    ST_RUN(CW);
#undef ST_RUN
    return cudaSuccess;
}

cudaError_t launch_base_vjp(const Geo& g, int dtype, const BaseVjpPtrs& p, cudaStream_t s, long long& launches) {
    if (g.dustbin || p.T < 1) return cudaErrorNotSupported;
#define ST_BV(D) \
    return dtype == 0 ? run_base_vjp<D, float>(g, dtype, p, s, launches) : run_base_vjp<D, __nv_bfloat16>(g, dtype, p, s, launches);
    if (g.d == 32) { ST_BV(32) }
    if (g.d == 64) { ST_BV(64) }
    ST_BV(128)
#undef ST_BV
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
                                 cudaStream_t s, long long& launches, const BwdHook* hook) {
    if (g.dustbin) {
        const long n = (long)g.BH * (g.Lq + g.Lk);
        if (dtype == 0) k_dust_dots<float><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(g, (const float*)p.dO, (const float*)p.V, t.Zd, t.ZdT);
        else k_dust_dots<__nv_bfloat16><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(g, (const __nv_bfloat16*)p.dO, (const __nv_bfloat16*)p.V, t.Zd, t.ZdT);
        ++launches;
    }
#define ST_DISPATCH(D)                                                                                 \
    if (dtype == 0) return direct ? run_all<true, D, float>(g, p, t, dtype, s, launches, hook)         \
                                  : run_all<false, D, float>(g, p, t, dtype, s, launches, hook);      \
    return direct ? run_all<true, D, __nv_bfloat16>(g, p, t, dtype, s, launches, hook)                \
                  : run_all<false, D, __nv_bfloat16>(g, p, t, dtype, s, launches, hook);
    if (g.d == 32) { ST_DISPATCH(32) }
    if (g.d == 64) { ST_DISPATCH(64) }
    ST_DISPATCH(128)
#undef ST_DISPATCH
}

}  // namespace st
