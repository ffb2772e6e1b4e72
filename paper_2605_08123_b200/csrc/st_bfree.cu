// st_bfree.cu -- band-free tcgen05 sweeps for bf16 inputs: the transport output O = P V
// (apply_transport, sinkhorn.hpp:257-277) and the exact R=2 adjoint (r2_backward,
// adjoint.hpp:232-373; one-reference form adjoint.hpp:202-226, direct four-plan form
// adjoint.hpp:311-368) without any stored L x W band.
//
// One kernel, k_bsweep<MODE>, streams the band of a 128-row block ("own" side, one TMEM lane
// per row) through its 64-column window chunks ("other" side):
//   tile   S_c = A1_blk B1_c^T  (and Z_c = A2_blk B2_c^T where the stage needs the cotangent
//          tile) on tcgen05 (kind::f16, fp32 accumulation in TMEM); the operand tiles are tensor-map
//          TMA boxes of the raw [B, H, L, d] tensors (128B-swizzled), or packed planes as a fallback
//   cell   p = ex2(c2 S + a_i + b_j) on the band (a, b = -inf padded duals), then per stage
//            PV    weight = p                      -> Y += W X_c       (O = P V; dV = P^T dO, g_v)
//            R12   acc_i += p (z - g_v_j)                              (u2_bar)
//            PX    acc_i += p x_j                                      (v1_bar, u1_bar)
//            SBAR  weight = Sbar (one-reference modifier field or the four-plan form)
//                                                  -> Y += W X_c       (dQ + d_eps;  dK + v0_bar)
//   GEMM   the weights go back to TMEM over the score tile, as two bf16 planes (hi + lo: 16 mantissa
//          bits, two K elements per 32-bit column), and are the A operand of a TS-form tcgen05.mma;
//          the chunk's operand rows X_c are the packed plane itself read MN-major (the same 8 x 16-byte
//          core matrices), so Y[128][d] (+)= W X_c is two tcgen05.mma per 16 window columns into a
//          TMEM accumulator -- no SMEM staging of the weights.
// Column stages are the same kernel on the transposed geometry (own = keys: A1 = K, B1 = Q).
// Nothing of size L x W is written or read: beyond the caller's tensors HBM holds only the padded
// dual / cotangent vectors (O(L)) and the outputs.
//
// Roles (persistent CTA, one per SM):
//   warp 0      producer: 1-D bulk async copies (TMA engine) of the block operands, the window
//               chunks and the window / own vectors
//   warp 1      issues the S / Z tiles; warp 18 issues the Y accumulations (tcgen05.mma issue rate is
//               the scarce resource: two issuing threads)
//   warps 2-17  epilogue: TMEM lane quadrant x column half x chunk parity; a thread owns one row
//               and 32 columns of every other chunk, so every row reduction is in-thread and the
//               four parts of a row combine in a fixed order.
#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "st_bfree.cuh"
#include "st_common.cuh"
#include "st_phase.cuh"
#include "st_sm100.cuh"

namespace st {

using namespace sm100;

namespace {

constexpr int kCR = 64;   // window chunk columns (MMA N of the score / cotangent tiles)
constexpr int kEW = 16;   // epilogue warps
constexpr int kNV = 2;    // vector ring slots

enum { M_PV = 0, M_R12 = 1, M_PX = 2, M_SROW = 3, M_SCOL = 4 };

struct alignas(64) SweepArgs {
    // tensor maps of the raw [BH][L][d] bf16 tensors behind the A2 / B2 streams (V and dO): boxes of
    // 64 rows x 64 columns, SWIZZLE_128B (tma2 = 1; else A2 / B2 point at packed planes)
    CUtensorMap tmA2, tmB2;
    int tma2;
    CUtensorMap tmA1, tmB1;  // the same for the A1 / B1 streams (Q and K): tma1
    int tma1;
    int NA, NS0, NS1, row_bytes, maxwin;  // A buffers; ring slots of the B1 / B2 window chunks
    int H, NB, nblk;
    int L_own, L_other, Lr_own, Lp_own, Lp_other, w;
    int wl_cap;
    int dbg;  // development ablations (ST_BF_DBG): 1 = no Y MMAs, 2 = one S / Z K-step, 4 = no cell math, 8 = no chunk loads (results invalid)
    float c2, scale;
    const uint8_t *A1, *B1, *A2, *B2;
    const void *rawA1, *rawB1, *rawA2, *rawB2;  // raw [BH][Lr][D] bf16 tensors behind the streams (host side: tensor maps)
    int Lr_other;
    const float* wv[5];  // window vectors [BH][Lp_other]; wv[0] = exponent offsets (-inf when inactive)
    const float* ov[5];  // own vectors [BH][Lp_own]; ov[0] = exponent offsets
    float* out_mat;      // [BH][Lr_own][D]
    float* out1;         // [BH][Lp_own]
    float* out2;         // [BH][Lp_own] or null
    float* out_api;      // [BH][Lr_own] or null
    const float* fvec;   // PX: own-side factor [BH][Lp_own] (null = 1)
    const __nv_bfloat16* dot_src;  // PV: raw rows [BH][Lr_own][D] for <Y_i, src_i> (null = none)
    unsigned long long* trace;     // development timeline (ST_BF_TRACE), null in production
};

template <int MODE, bool kDirect>
struct ModeTraits {
    static constexpr bool kZ = MODE == M_R12 || MODE == M_SROW || MODE == M_SCOL;
    static constexpr bool kGemm = MODE == M_PV || MODE == M_SROW || MODE == M_SCOL;
    static constexpr bool kB2 = kZ || MODE == M_PV;
    static constexpr int NW = MODE == M_PV ? 1 : (MODE == M_R12 || MODE == M_PX) ? 2 : MODE == M_SROW ? 5 : 4;
    static constexpr int NO = (MODE == M_PV || MODE == M_R12 || MODE == M_PX) ? 1 : MODE == M_SROW ? 4 : 5;
};

struct BSmem {
    uint8_t* A;    // [NA][(1 + Z) * 128 * row_bytes]
    uint8_t* B0;   // [NS0][64 * row_bytes]  B1 window chunks
    uint8_t* B1;   // [NS1][64 * row_bytes]  B2 window chunks
    float* vw;     // [kNV][NW][maxwin]
    float* vo;     // [kNV][NO][128]
    float* rowx;   // [2][4][128]
    uint64_t *v_full, *v_empty, *a_full, *a_empty, *k_full, *k_empty, *k2_full, *k2_empty, *t_full, *t_empty, *w_full, *y_full, *y_empty;
    uint32_t* tmem_base;
    int4* bd;
};

template <int MODE, bool kDirect>
__host__ __device__ inline size_t bs_bytes(int NA, int NS0, int NS1, int row_bytes, int maxwin, int wl_cap) {
    using T = ModeTraits<MODE, kDirect>;
    size_t n = (size_t)NA * (T::kZ ? 2 : 1) * 128 * row_bytes + (size_t)(NS0 + (T::kB2 ? NS1 : 0)) * kCR * row_bytes;
    n += (size_t)kNV * (T::NW * maxwin + T::NO * 128) * 4 + 2 * 4 * 128 * 4;
    n += (size_t)(2 * kNV + 2 * NA + 2 * NS0 + 2 * NS1 + 16) * 8 + 16 + (size_t)wl_cap * 16;
    return n;
}

template <int MODE, bool kDirect>
__device__ __forceinline__ BSmem bcarve(uint8_t* base, const SweepArgs& a) {
    using T = ModeTraits<MODE, kDirect>;
    BSmem s;
    s.A = base;
    s.B0 = s.A + (size_t)a.NA * (T::kZ ? 2 : 1) * 128 * a.row_bytes;
    s.B1 = s.B0 + (size_t)a.NS0 * kCR * a.row_bytes;
    s.vw = (float*)(s.B1 + (size_t)(T::kB2 ? a.NS1 : 0) * kCR * a.row_bytes);
    s.vo = s.vw + kNV * T::NW * a.maxwin;
    s.rowx = s.vo + kNV * T::NO * 128;
    uint64_t* b = (uint64_t*)(s.rowx + 2 * 4 * 128);
    s.v_full = b; b += kNV;
    s.v_empty = b; b += kNV;
    s.a_full = b; b += a.NA;
    s.a_empty = b; b += a.NA;
    s.k_full = b; b += a.NS0;
    s.k_empty = b; b += a.NS0;
    s.k2_full = b; b += a.NS1;
    s.k2_empty = b; b += a.NS1;
    s.t_full = b; b += 4;
    s.t_empty = b; b += 4;
    s.w_full = b; b += 4;
    s.y_full = b; b += 2;
    s.y_empty = b; b += 2;
    s.tmem_base = (uint32_t*)b;
    s.bd = (int4*)(s.tmem_base + 4);
    return s;
}

// B operand read MN-major: N = head dim (8 elements = the 16 contiguous bytes of a core-matrix row),
// K = packed rows (8 rows of a core matrix 16 bytes apart): SBO = step between 8-element groups
// along N (128 B), LBO = step between 8-row groups along K (8 * row_bytes).
__host__ __device__ constexpr uint32_t make_idesc_bmn(uint32_t M, uint32_t N) {
    return make_idesc(M, N, 1u) | (1u << 16);
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&v);
}

template <int N>
__device__ __forceinline__ void tc_ldn(uint32_t taddr, float (&v)[N]) {
    if constexpr (N == 32) tc_ld32(taddr, v);
    else tc_ld16(taddr, v);
}

}  // namespace

// One 16-column half of a warp's slice: thread = one row.  sv / zv: the score / cotangent tile values,
// W: the window vectors at these columns, O: the row's own scalars.  Packed (two-cell) FP32 math; the
// band test (kEdge: slices the band boundary crosses) is the only per-cell select.  Weights leave as
// bf16 hi / lo pairs (hw, lw: two K elements per word); row partial sums accumulate in acc2.
template <int MODE, bool kDirect, bool kEdge, int NW, int NO>
__device__ __forceinline__ void slice_half(const float (&sv)[16], const float (&zv)[16], const float* __restrict__ vwp,
                                           int maxwin, int cc0, int lo, unsigned bw, const float (&O)[NO], float c2,
                                           float2& acc2, uint32_t (&hw)[8], uint32_t (&lw)[8]) {
    constexpr bool kGemm = MODE == M_PV || MODE == M_SROW || MODE == M_SCOL;
    const float2 c2v = make_float2(c2, c2), a2v = make_float2(O[0], O[0]), neg1 = make_float2(-1.f, -1.f);
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
        float2 W[NW][2];
#pragma unroll
        for (int k = 0; k < NW; ++k) {
            const float4 t4 = *reinterpret_cast<const float4*>(vwp + (size_t)k * maxwin + cc0 + 4 * q4);
            W[k][0] = make_float2(t4.x, t4.y);
            W[k][1] = make_float2(t4.z, t4.w);
        }
#pragma unroll
        for (int e2 = 0; e2 < 2; ++e2) {
            const int kx = 4 * q4 + 2 * e2;
            const float2 s2 = make_float2(sv[kx], sv[kx + 1]);
            bool in0 = true, in1 = true;
            if (kEdge) {
                in0 = (unsigned)(cc0 + kx - lo) <= bw;
                in1 = (unsigned)(cc0 + kx + 1 - lo) <= bw;
            }
            float2 e0 = __fmul2_rn(s2, c2v);  // direct mode: the bare scaled score (masked)
            float2 zz = __fadd2_rn(__ffma2_rn(s2, c2v, W[0][e2]), a2v);
            if (kEdge) {
                zz.x = in0 ? zz.x : -INFINITY;
                zz.y = in1 ? zz.y : -INFINITY;
            }
            const float2 p = make_float2(ex2(zz.x), ex2(zz.y));
            float2 wgt = p;
            if constexpr (MODE == M_R12) {
                const float2 z2 = make_float2(zv[kx], zv[kx + 1]);
                acc2 = __ffma2_rn(p, __ffma2_rn(W[1][e2], neg1, z2), acc2);
            } else if constexpr (MODE == M_PX) {
                acc2 = __ffma2_rn(p, W[1][e2], acc2);
            } else if constexpr (MODE == M_SROW) {
                const float2 z2 = make_float2(zv[kx], zv[kx + 1]);
                if constexpr (!kDirect) {
                    // O = (a, u2b, alpha, au1); W = (b, v2b, beta, bv1, delta)
                    const float2 m = __ffma2_rn(W[4][e2], make_float2(O[3], O[3]),
                                                __ffma2_rn(W[3][e2], make_float2(O[2], O[2]),
                                                           __ffma2_rn(W[2][e2], make_float2(O[1], O[1]), W[1][e2])));
                    wgt = __fmul2_rn(p, __ffma2_rn(m, neg1, z2));
                } else {
                    // O = (u2, u1, u2b, u1b); W = (v2, v1, v0, v2b, v1b)
                    if (kEdge) {
                        e0.x = in0 ? e0.x : -INFINITY;
                        e0.y = in1 ? e0.y : -INFINITY;
                    }
                    const float2 t21 = __fadd2_rn(e0, __fadd2_rn(W[1][e2], a2v));
                    const float2 t11 = __fadd2_rn(e0, __fadd2_rn(W[1][e2], make_float2(O[1], O[1])));
                    const float2 t10 = __fadd2_rn(e0, __fadd2_rn(W[2][e2], make_float2(O[1], O[1])));
                    const float2 p21 = make_float2(ex2(t21.x), ex2(t21.y)), p11 = make_float2(ex2(t11.x), ex2(t11.y)),
                                 p10 = make_float2(ex2(t10.x), ex2(t10.y));
                    wgt = __fmul2_rn(p, __ffma2_rn(W[3][e2], neg1, z2));
                    wgt = __ffma2_rn(p21, make_float2(-O[2], -O[2]), wgt);
                    wgt = __ffma2_rn(__fmul2_rn(p11, neg1), W[4][e2], wgt);
                    wgt = __ffma2_rn(p10, make_float2(-O[3], -O[3]), wgt);
                }
                acc2 = __ffma2_rn(wgt, s2, acc2);  // d_eps partial, scaled by c2 ln 2 at the end
            } else if constexpr (MODE == M_SCOL) {
                const float2 z2 = make_float2(zv[kx], zv[kx + 1]);
                if constexpr (!kDirect) {
                    // O = (a = v2, v2b, beta, bv1, delta); W = (b = u2, u2b, alpha, au1)
                    const float2 m = __ffma2_rn(make_float2(O[4], O[4]), W[3][e2],
                                                __ffma2_rn(make_float2(O[3], O[3]), W[2][e2],
                                                           __ffma2_rn(make_float2(O[2], O[2]), W[1][e2], make_float2(O[1], O[1]))));
                    wgt = __fmul2_rn(p, __ffma2_rn(m, neg1, z2));
                    acc2 = __ffma2_rn(p, W[3][e2], acc2);
                } else {
                    // O = (v2, v1, v0, v2b, v1b); W = (u2, u1, u2b, u1b)
                    if (kEdge) {
                        e0.x = in0 ? e0.x : -INFINITY;
                        e0.y = in1 ? e0.y : -INFINITY;
                    }
                    const float2 t21 = __fadd2_rn(e0, __fadd2_rn(W[0][e2], make_float2(O[1], O[1])));
                    const float2 t11 = __fadd2_rn(e0, __fadd2_rn(W[1][e2], make_float2(O[1], O[1])));
                    const float2 t10 = __fadd2_rn(e0, __fadd2_rn(W[1][e2], make_float2(O[2], O[2])));
                    const float2 p21 = make_float2(ex2(t21.x), ex2(t21.y)), p11 = make_float2(ex2(t11.x), ex2(t11.y)),
                                 p10 = make_float2(ex2(t10.x), ex2(t10.y));
                    wgt = __fmul2_rn(p, __fadd2_rn(z2, make_float2(-O[3], -O[3])));
                    wgt = __ffma2_rn(__fmul2_rn(p21, neg1), W[2][e2], wgt);
                    wgt = __ffma2_rn(p11, make_float2(-O[4], -O[4]), wgt);
                    wgt = __ffma2_rn(__fmul2_rn(p10, neg1), W[3][e2], wgt);
                    acc2 = __ffma2_rn(p10, W[3][e2], acc2);
                }
            }
            if constexpr (kGemm) {
                const __nv_bfloat162 h2 = __floats2bfloat162_rn(wgt.x, wgt.y);  // one cvt.rn.bf16x2.f32
                const uint32_t hb = *reinterpret_cast<const uint32_t*>(&h2);
                const float2 hf2 = make_float2(__uint_as_float(hb << 16), __uint_as_float(hb & 0xffff0000u));
                const float2 r2 = __ffma2_rn(hf2, neg1, wgt);  // exact residual
                hw[2 * q4 + e2] = hb;
                lw[2 * q4 + e2] = pack_bf16(r2.x, r2.y);
            }
        }
    }
}

__device__ __forceinline__ unsigned long long bf_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// development timeline of CTA 0, blocks kTrB .. kTrB + 1 (build with -DST_BF_TRACE): slot layout in bf_trace_dump
#ifdef ST_BF_TRACE
#define BF_TRACE(cond, slot)                                                    \
    do {                                                                        \
        if (a.trace && blockIdx.x == 0 && (cond)) a.trace[(slot)] = bf_gtimer(); \
    } while (0)
#else
#define BF_TRACE(cond, slot) \
    do {                     \
    } while (0)
#endif
constexpr int kTrB = 4;

template <int MODE, bool kDirect, int D>
__global__ void __launch_bounds__(96 + 32 * kEW, 1) k_bsweep(const __grid_constant__ SweepArgs a) {
    using T = ModeTraits<MODE, kDirect>;
    constexpr bool kZ = T::kZ, kGemm = T::kGemm, kB2 = T::kB2;
    constexpr int NW = T::NW, NO = T::NO;
    constexpr int TCOLS = kCR * (kZ ? 2 : 1);  // TMEM columns of one chunk buffer (S | Z)
    // Y accumulators ahead of the chunk buffers: two (the drain of a block overlaps the next block's
    // accumulation), or one where a third chunk buffer is worth more (d = 128 with a cotangent tile)
    constexpr int kYB = !kGemm ? 0 : (kZ && D == 128) ? 1 : 2;
    constexpr int YC = kYB * D;
    constexpr int NBUF = (512 - YC) / TCOLS < 4 ? (512 - YC) / TCOLS : 4;  // chunk buffers in flight
    constexpr int NE = 32 * kEW;
    static_assert(NBUF >= 2 && YC + NBUF * TCOLS <= 512, "TMEM budget");
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const BSmem s = bcarve<MODE, kDirect>(smem_raw, a);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t blk_bytes = 128u * a.row_bytes, chk_bytes = (uint32_t)kCR * a.row_bytes;
    const uint32_t a_stride = blk_bytes * (kZ ? 2 : 1);
    // the ring whose chunk is also the Y operand X_c is released by the Y accumulation (long-lived)
    constexpr bool kLong0 = MODE == M_SROW || MODE == M_SCOL, kLong1 = MODE == M_PV;

    if (threadIdx.x == 0) {
        for (int k = 0; k < kNV; ++k) {
            mbar_init(&s.v_full[k], 1);
            mbar_init(&s.v_empty[k], kEW);
        }
        for (int k = 0; k < a.NA; ++k) {
            mbar_init(&s.a_full[k], 1);
            mbar_init(&s.a_empty[k], 1);
        }
        for (int k = 0; k < a.NS0; ++k) {
            mbar_init(&s.k_full[k], 1);
            mbar_init(&s.k_empty[k], 1);
        }
        for (int k = 0; k < a.NS1; ++k) {
            mbar_init(&s.k2_full[k], 1);
            mbar_init(&s.k2_empty[k], 1);
        }
        for (int k = 0; k < 4; ++k) {
            mbar_init(&s.t_full[k], 1);
            mbar_init(&s.t_empty[k], kGemm ? 1 : kEW / 2);  // gemm: freed by the Y accumulation's commit
            mbar_init(&s.w_full[k], kEW / 2);
        }
        for (int k = 0; k < 2; ++k) {
            mbar_init(&s.y_full[k], 1);
            mbar_init(&s.y_empty[k], kEW);
        }
        fence_mbar_init();
    }
    if (warp == 1) {
        tc_alloc(s.tmem_base, 512);
        tc_relinquish();
    }
    const int g_begin = (int)((long long)a.nblk * blockIdx.x / gridDim.x);
    const int g_end = (int)((long long)a.nblk * (blockIdx.x + 1) / gridDim.x);
    const int nb = min(g_end - g_begin, a.wl_cap);
    const int nq = a.Lp_other / kCR;
    for (int k = threadIdx.x; k < nb; k += blockDim.x) {
        const int g = g_begin + k;
        const int bh = g / a.NB, blk = g % a.NB, i0 = blk * 128;
        const int q0 = max(0, i0 - a.w) / kCR;
        const int q1 = min(nq - 1, (i0 + 127 + a.w) / kCR);
        s.bd[k] = make_int4(bh, blk, q0, q1);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *s.tmem_base;

    if (warp == 0) {
        // ------------------------------------------------------------ producer (one thread)
        if (lane == 0) {
        // three independent cursors over the CTA's (block, chunk) sequence, each advancing as soon as
        // its buffer is free: block operands + vectors, B1 chunks (ring 0), B2 chunks (ring 1)
        int pb = 0;                       // block cursor
        int b0 = 0, c0 = 0, b1 = 0, c1 = 0;  // ring cursors: block, chunk within the block
        uint32_t s0 = 0, s1 = 0;          // running chunk numbers
        if (!kB2) b1 = nb;
        while (pb < nb || b0 < nb || b1 < nb) {
            bool moved = false;
            if (pb < nb) {
                const int vs = pb % kNV, ab = pb % a.NA;
                bool ok = mbar_test(&s.v_empty[vs], ((pb / kNV) & 1) ^ 1) && mbar_test(&s.a_empty[ab], ((pb / a.NA) & 1) ^ 1);
                if (ok) {
                    {
                        const int4 b = s.bd[pb];
                        const int i0 = b.y * 128, nwin = (b.w - b.z + 1) * kCR, wbase = b.z * kCR;
                        mbar_arrive_expect_tx(&s.v_full[vs], (uint32_t)(NW * nwin + NO * 128) * 4u);
#pragma unroll
                        for (int k = 0; k < NW; ++k)
                            bulk_g2s(s.vw + ((size_t)vs * NW + k) * a.maxwin, a.wv[k] + (size_t)b.x * a.Lp_other + wbase,
                                     (uint32_t)nwin * 4u, &s.v_full[vs]);
#pragma unroll
                        for (int k = 0; k < NO; ++k)
                            bulk_g2s(s.vo + ((size_t)vs * NO + k) * 128, a.ov[k] + (size_t)b.x * a.Lp_own + i0, 512u,
                                     &s.v_full[vs]);
                        mbar_arrive_expect_tx(&s.a_full[ab], a_stride);
                        const size_t off = ((size_t)b.x * a.Lp_own + i0) * a.row_bytes;
                        if (a.tma1) {  // [d half][128 rows][128 B], two 64-row boxes per half
#pragma unroll
                            for (int kb = 0; kb < D / 64; ++kb)
#pragma unroll
                                for (int h = 0; h < 2; ++h)
                                    tma_load_3d(s.A + (size_t)ab * a_stride + kb * 16384 + h * 8192, &a.tmA1, kb * 64, i0 + 64 * h, b.x, &s.a_full[ab]);
                        } else {
                            bulk_g2s(s.A + (size_t)ab * a_stride, a.A1 + off, blk_bytes, &s.a_full[ab]);
                        }
                        if (kZ) {
                            uint8_t* dst = s.A + (size_t)ab * a_stride + blk_bytes;
                            if (a.tma2) {  // [d half][128 rows][128 B], two 64-row boxes per half
#pragma unroll
                                for (int kb = 0; kb < D / 64; ++kb)
#pragma unroll
                                    for (int h = 0; h < 2; ++h)
                                        tma_load_3d(dst + kb * 16384 + h * 8192, &a.tmA2, kb * 64, i0 + 64 * h, b.x, &s.a_full[ab]);
                            } else {
                                bulk_g2s(dst, a.A2 + off, blk_bytes, &s.a_full[ab]);
                            }
                        }
                    }
                    ++pb;
                    moved = true;
                }
            }
#pragma unroll
            for (int ring = 0; ring < (kB2 ? 2 : 1); ++ring) {
                int& rb = ring ? b1 : b0;
                int& rc = ring ? c1 : c0;
                uint32_t& rs = ring ? s1 : s0;
                if (rb >= nb) continue;
                const int ns = ring ? a.NS1 : a.NS0;
                uint64_t* full = ring ? s.k2_full : s.k_full;
                uint64_t* empty = ring ? s.k2_empty : s.k_empty;
                const int sl = rs % ns;
                bool ok = mbar_test(&empty[sl], ((rs / ns) & 1) ^ 1);
                if (!ok) continue;
                const int4 b = s.bd[rb];
                if (a.dbg & 8) {  // ablation: no window-chunk loads (stale operands)
                    mbar_arrive(&full[sl]);
                } else {
                    mbar_arrive_expect_tx(&full[sl], chk_bytes);
                    const size_t off = ((size_t)b.x * a.Lp_other + (size_t)(b.z + rc) * kCR) * a.row_bytes;
                    if (ring ? a.tma2 : a.tma1) {  // [d half][64 rows][128 B]
#pragma unroll
                        for (int kb = 0; kb < D / 64; ++kb)
                            tma_load_3d((ring ? s.B1 : s.B0) + (size_t)sl * chk_bytes + kb * 8192, ring ? &a.tmB2 : &a.tmB1, kb * 64,
                                        (b.z + rc) * kCR, b.x, &full[sl]);
                    } else {
                        bulk_g2s((ring ? s.B1 : s.B0) + (size_t)sl * chk_bytes, (ring ? a.B2 : a.B1) + off, chk_bytes, &full[sl]);
                    }
                }
                moved = true;
                ++rs;
                if (++rc == b.w - b.z + 1) {
                    rc = 0;
                    ++rb;
                }
            }
            if (!moved) __nanosleep(64);  // leave the issue slots of this SMSP to its epilogue warps
        }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ S / Z tile issuer
        const uint32_t idesc_s = make_idesc(128, kCR, 1u);
        const uint32_t sbo = (uint32_t)a.row_bytes * 8u;
        constexpr int ksteps = D / 16;
        uint32_t scs = 0;
        for (int sb = 0; sb < nb; ++sb) {
            const int ab = sb % a.NA;
            const int s_nch = s.bd[sb].w - s.bd[sb].z + 1;
            mbar_wait(&s.a_full[ab], (sb / a.NA) & 1);
            const uint64_t ad = make_desc(smem_u32(s.A + (size_t)ab * a_stride), 128, sbo);
            const uint64_t ad2 = make_desc(smem_u32(s.A + (size_t)ab * a_stride + blk_bytes), 128, sbo);
            for (int sc = 0; sc < s_nch; ++sc, ++scs) {
                const uint32_t sl = scs % a.NS0, sl2 = kB2 ? scs % a.NS1 : 0, tb = scs % NBUF;
                mbar_wait(&s.k_full[sl], (scs / a.NS0) & 1);
                if (kZ) mbar_wait(&s.k2_full[sl2], (scs / a.NS1) & 1);
                mbar_wait(&s.t_empty[tb], ((scs / NBUF) & 1) ^ 1);
                BF_TRACE(lane == 0 && sb == kTrB, sc);
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t a1s = smem_u32(s.A + (size_t)ab * a_stride), b1s = smem_u32(s.B0 + (size_t)sl * chk_bytes);
                    const uint64_t bd = make_desc(b1s, 128, sbo);
                    const uint32_t dt = tbase + YC + tb * TCOLS;
                    // score tile K step kk: packed planes (core-matrix order) or 128B-swizzled tensor-map tiles
                    auto s_mma = [&](int kk) {
                        if (a.tma1)
                            mma_bf16(dt, make_desc_sw128(a1s + (kk / 4) * 16384 + (kk % 4) * 32, 16, 1024),
                                     make_desc_sw128(b1s + (kk / 4) * 8192 + (kk % 4) * 32, 16, 1024), idesc_s, kk > 0);
                        else
                            mma_bf16(dt, ad + (uint64_t)(kk * 16), bd + (uint64_t)(kk * 16), idesc_s, kk > 0);
                    };
                    if (kZ) {  // the score and cotangent chains interleave (independent accumulators)
                        const uint32_t a2s = smem_u32(s.A + (size_t)ab * a_stride + blk_bytes);
                        const uint32_t b2s = smem_u32(s.B1 + (size_t)sl2 * chk_bytes);
                        const uint64_t bd2 = make_desc(b2s, 128, sbo);
#pragma unroll
                        for (int kk = 0; kk < ksteps; ++kk) {
                            if (kk > 0 && (a.dbg & 2)) break;
                            s_mma(kk);
                            if (a.tma2)  // swizzled tiles: d half kk / 4, 32 bytes per K step inside the 128-byte row
                                mma_bf16(dt + kCR, make_desc_sw128(a2s + (kk / 4) * 16384 + (kk % 4) * 32, 16, 1024),
                                         make_desc_sw128(b2s + (kk / 4) * 8192 + (kk % 4) * 32, 16, 1024), idesc_s, kk > 0);
                            else
                                mma_bf16(dt + kCR, ad2 + (uint64_t)(kk * 16), bd2 + (uint64_t)(kk * 16), idesc_s, kk > 0);
                        }
                    } else {
#pragma unroll
                        for (int kk = 0; kk < ksteps; ++kk) {
                            if (kk > 0 && (a.dbg & 2)) break;
                            s_mma(kk);
                        }
                    }
                    tc_commit(&s.t_full[tb]);
                    if (sc == s_nch - 1) tc_commit(&s.a_empty[ab]);
                    if (!kLong0) tc_commit(&s.k_empty[sl]);
                    if (kZ) tc_commit(&s.k2_empty[sl2]);
                }
                __syncwarp();
                BF_TRACE(lane == 0 && sb == kTrB, 56 + sc);
            }
        }
    } else if (warp == 2 + kEW) {
        // ------------------------------------------------------------ Y accumulation issuer (its own warp:
        // tcgen05.mma issue is the scarce resource of the sweep, two issuers double it)
        if (kGemm) {
            const uint32_t idesc_y = make_idesc_bmn(128, D);
            const uint32_t sbo = (uint32_t)a.row_bytes * 8u;
            uint32_t ycs = 0;
            for (int yb = 0; yb < nb; ++yb) {
                const int y_nch = s.bd[yb].w - s.bd[yb].z + 1;
                const uint32_t ybuf = kYB == 2 ? (yb & 1) : 0;
                mbar_wait(&s.y_empty[ybuf], ((yb / (kYB == 2 ? 2 : 1)) & 1) ^ 1);
                for (int yc = 0; yc < y_nch; ++yc, ++ycs) {
                    const uint32_t wb = ycs % NBUF, sl = kLong1 ? ycs % a.NS1 : ycs % a.NS0;
                    if (kLong1) mbar_wait(&s.k2_full[sl], (ycs / a.NS1) & 1);  // the V chunk (X_c)
                    mbar_wait(&s.w_full[wb], (ycs / NBUF) & 1);
                    BF_TRACE(lane == 0 && yb == kTrB, 8 + yc);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t dy = tbase + ybuf * D;
                        const uint8_t* xs = (kLong1 ? s.B1 : s.B0) + (size_t)sl * chk_bytes;
                        const uint64_t xd = make_desc(smem_u32(xs), sbo, 128);
                        // weights: warp half hf of the chunk left plane p of its K = 16 kk .. 16 kk + 15 at
                        // columns 32 hf + 16 p + 8 kk of the score tile (two bf16 per column)
                        const uint32_t wa = tbase + YC + wb * TCOLS;
                        if (!(a.dbg & 1)) {
#pragma unroll
                            for (int hf = 0; hf < 2; ++hf)
#pragma unroll
                                for (int p = 0; p < 2; ++p)
#pragma unroll
                                    for (int kk = 0; kk < 2; ++kk)
                                        mma_bf16_ts(dy, wa + 32 * hf + 16 * p + 8 * kk,
                                                    (kLong1 ? a.tma2 : a.tma1)
                                                        // swizzled operand chunk read MN-major: 64-column halves 8192 B
                                                        // apart, 8-row K groups 1024 B apart, 16 rows per K step
                                                        ? make_desc_sw128(smem_u32(xs) + (2 * hf + kk) * 2048, 8192, 1024)
                                                        : xd + (uint64_t)((2 * hf + kk) * a.row_bytes),
                                                    idesc_y, (yc > 0 || hf > 0 || p > 0 || kk > 0) ? 1u : 0u);
                        }
                        tc_commit(&s.t_empty[wb]);
                        tc_commit(kLong1 ? &s.k2_empty[sl] : &s.k_empty[sl]);
                        if (yc == y_nch - 1) tc_commit(&s.y_full[ybuf]);
                    }
                    __syncwarp();
                    BF_TRACE(lane == 0 && yb == kTrB, 48 + yc);
                }
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const int qd = warp & 3, gidx = ((warp - 2) >> 2) & 1, hf = (warp - 2) >> 3;
        const int part = gidx * 2 + hf;
        const int r = qd * 32 + lane;
        const uint32_t tl = tbase + ((uint32_t)(qd * 32) << 16);
        const unsigned bw = 2u * (unsigned)a.w;
        const float c2ln2 = a.c2 * kLn2;
        uint32_t cs = 0;
        for (int bi = 0; bi < nb; ++bi) {
            const int4 b = s.bd[bi];
            const int i0 = b.y * 128, nch = b.w - b.z + 1, wbase = b.z * kCR;
            const int vs = bi % kNV, par = bi & 1;
            const int i = i0 + r;
            const int lo = i - a.w - wbase;                  // band start of this row, window coordinates
            const int lo_min = i0 + qd * 32 - a.w - wbase;   // of the warp's first row
            BF_TRACE(lane == 0 && warp == 2 && bi == kTrB, 44);
            mbar_wait(&s.v_full[vs], (bi / kNV) & 1);
            BF_TRACE(lane == 0 && warp == 2 && bi == kTrB, 45);
            const float* vwp = s.vw + (size_t)vs * NW * a.maxwin;
            float O[NO];
#pragma unroll
            for (int k = 0; k < NO; ++k) O[k] = s.vo[((size_t)vs * NO + k) * 128 + r];
            float fown = 1.f;  // PX: the own-side factor, fetched ahead of the block-end combine
            if (MODE == M_PX && part == 0 && a.fvec) fown = a.fvec[(size_t)b.x * a.Lp_own + i];
            float2 acc2 = make_float2(0.f, 0.f);
            for (int c = 0; c < nch; ++c, ++cs) {
                if ((int)(cs & 1) != gidx) continue;
                const uint32_t tb = cs % NBUF, tpar = (cs / NBUF) & 1;
                const int c0 = c * kCR + 32 * hf;  // first window column of this warp's slice
                const bool outside = c0 + 31 < lo_min || c0 > lo_min + 31 + (int)bw || (a.dbg & 4);
                const bool edge = !(c0 >= lo_min + 31 && c0 + 31 <= lo_min + (int)bw);
                const uint32_t ta = tl + YC + tb * TCOLS + 32 * hf;
                mbar_wait(&s.t_full[tb], tpar);
                BF_TRACE(lane == 0 && (warp == 2 || warp == 6) && bi == kTrB, 16 + c);
                BF_TRACE(lane == 0 && bi == kTrB && (c == 2 || c == 3), 64 + (warp - 2) * 3);
                if (outside) {
                    if (kGemm) {
                        tc_fence_after();
                        const uint32_t zero8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
                        for (int q = 0; q < 4; ++q) tc_st8(ta + 8 * q, zero8);
                        tc_wait_st();
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&s.w_full[tb]);
                    } else {
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&s.t_empty[tb]);
                    }
                    continue;
                }
                tc_fence_after();
                float sv[2][16], zv[2][16];
                tc_ld16(ta, sv[0]);
                tc_ld16(ta + 16, sv[1]);
                if (kZ) {
                    tc_ld16(ta + kCR, zv[0]);
                    tc_ld16(ta + kCR + 16, zv[1]);
                }
                tc_wait_ld();
                BF_TRACE(lane == 0 && (warp == 2 || warp == 6) && bi == kTrB, 24 + c);
                BF_TRACE(lane == 0 && bi == kTrB && (c == 2 || c == 3), 64 + (warp - 2) * 3 + 1);
                if (!kGemm) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&s.t_empty[tb]);
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    uint32_t hw[8], lw[8];
                    if (edge)
                        slice_half<MODE, kDirect, true, NW, NO>(sv[h], zv[h], vwp, a.maxwin, c0 + 16 * h, lo, bw, O, a.c2, acc2, hw, lw);
                    else
                        slice_half<MODE, kDirect, false, NW, NO>(sv[h], zv[h], vwp, a.maxwin, c0 + 16 * h, lo, bw, O, a.c2, acc2, hw, lw);
                    if (kGemm) {  // K = 16 h .. 16 h + 15 of this warp's slice: hi plane, lo plane
                        tc_st8(ta + 8 * h, hw);
                        tc_st8(ta + 16 + 8 * h, lw);
                    }
                }
                if (kGemm) {
                    tc_wait_st();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&s.w_full[tb]);
                }
                BF_TRACE(lane == 0 && (warp == 2 || warp == 6) && bi == kTrB, 32 + c);
                BF_TRACE(lane == 0 && bi == kTrB && (c == 2 || c == 3), 64 + (warp - 2) * 3 + 2);
            }
            const float acc = (acc2.x + acc2.y) * (MODE == M_SROW ? c2ln2 : 1.f);
            __syncwarp();
            BF_TRACE(lane == 0 && warp == 2 && bi == kTrB, 40);
            if (lane == 0) mbar_arrive(&s.v_empty[vs]);
            const size_t orow = (size_t)b.x * a.Lr_own + i;
            if (kGemm) {
                // ---- drain this block's accumulator with 16x256b loads: thread (t0, t1) holds rows t1, t1 + 8
                // of a 16-row half and columns 8 m + 2 t0 + {0, 1} of a 32-column group, so the 4 threads of
                // a row write one full 32-byte sector per store (D = 128: the warp's column quarter, both
                // halves; D = 64: one column half of one row half)
                constexpr int NH = D == 128 ? 2 : 1;
                const int cg = D == 128 ? part : (part & 1);
                const uint32_t ybuf = kYB == 2 ? (bi & 1) : 0;
                const int t0 = lane & 3, t1 = lane >> 2;
                const bool dot = MODE == M_PV && a.dot_src != nullptr;
                // <Y_i, src_i> operands (C1: the raw V rows) fetched before the accumulator is waited for
                uint32_t dsrc[NH][2][4];
                if (dot) {
#pragma unroll
                    for (int hh = 0; hh < NH; ++hh) {
                        const int rh = D == 128 ? hh : (part >> 1);
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int ig = i0 + qd * 32 + 16 * rh + t1 + 8 * h;
                            const uint32_t* src = reinterpret_cast<const uint32_t*>(
                                a.dot_src + ((size_t)b.x * a.Lr_own + min(ig, a.L_own - 1)) * D + cg * 32 + 2 * t0);
#pragma unroll
                            for (int m = 0; m < 4; ++m) dsrc[hh][h][m] = src[4 * m];
                        }
                    }
                }
                mbar_wait(&s.y_full[ybuf], (bi / (kYB == 2 ? 2 : 1)) & 1);
                BF_TRACE(lane == 0 && warp == 2 && bi == kTrB, 41);
                tc_fence_after();
                float y[NH][16];
#pragma unroll
                for (int hh = 0; hh < NH; ++hh) {
                    const int rh = D == 128 ? hh : (part >> 1);
                    tc_ld16x256(tbase + ((uint32_t)(qd * 32 + 16 * rh) << 16) + ybuf * D + cg * 32, y[hh]);
                }
                tc_wait_ld();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&s.y_empty[ybuf]);
                float* rxd = s.rowx + (size_t)par * 4 * 128 + part * 128;
#pragma unroll
                for (int hh = 0; hh < NH; ++hh) {
                    const int rh = D == 128 ? hh : (part >> 1);
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int rloc = qd * 32 + 16 * rh + t1 + 8 * h;
                        const int ig = i0 + rloc;
                        float dsum = 0.f;
                        if (ig < a.L_own) {
                            const size_t eo = ((size_t)b.x * a.Lr_own + ig) * D + cg * 32 + 2 * t0;
                            float* dst = a.out_mat + eo;
#pragma unroll
                            for (int m = 0; m < 4; ++m)
                                *reinterpret_cast<float2*>(dst + 8 * m) =
                                    make_float2(y[hh][4 * m + 2 * h] * a.scale, y[hh][4 * m + 2 * h + 1] * a.scale);
                            if (dot) {
#pragma unroll
                                for (int m = 0; m < 4; ++m) {
                                    const uint32_t ww = dsrc[hh][h][m];
                                    dsum = fmaf(y[hh][4 * m + 2 * h], __uint_as_float(ww << 16), dsum);
                                    dsum = fmaf(y[hh][4 * m + 2 * h + 1], __uint_as_float(ww & 0xffff0000u), dsum);
                                }
                            }
                        }
                        if (dot) {  // <Y_i, src_i> over this warp's 32 columns
                            dsum += __shfl_xor_sync(0xffffffffu, dsum, 1);
                            dsum += __shfl_xor_sync(0xffffffffu, dsum, 2);
                            if (t0 == 0) rxd[rloc] = dsum;
                            if (D == 64 && t0 == 1) rxd[qd * 32 + 16 * (1 - rh) + t1 + 8 * h] = 0.f;
                        }
                    }
                }
            }
            if (MODE != M_PV || a.dot_src) {
                // ---- the four parts of a row combine in a fixed order
                float* rx = s.rowx + (size_t)par * 4 * 128;
                if (MODE != M_PV) rx[part * 128 + r] = acc;
                BF_TRACE(lane == 0 && warp == 2 && bi == kTrB, 42);
                named_bar(1, NE);
                BF_TRACE(lane == 0 && warp == 2 && bi == kTrB, 43);
                if (part == 0) {
                    const float tot = (rx[r] + rx[128 + r]) + (rx[256 + r] + rx[384 + r]);
                    const size_t prow = (size_t)b.x * a.Lp_own + i;
                    if constexpr (MODE == M_PV || MODE == M_R12) {
                        a.out1[prow] = tot;
                    } else if constexpr (MODE == M_PX) {
                        const float f = fown;
                        const float o = -f * tot;
                        a.out1[prow] = o;
                        if (a.out2) a.out2[prow] = f * o;
                    } else if constexpr (MODE == M_SROW) {
                        if (i < a.L_own) a.out_api[orow] = tot;
                    } else {
                        if (i < a.L_own) a.out_api[orow] = kDirect ? -tot : -O[4] * tot;
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tc_dealloc(tbase, 512);
    }
}

// ---------------------------------------------------------------------------
// Padded vectors of the sweeps: duals with -inf on inactive / padding entries, step ratios.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_bf_prep(int BH, int H, int L, int Lr, int Lp, const uint8_t* __restrict__ mask,
                                                 const float* __restrict__ d2, const float* __restrict__ d1,
                                                 const float* __restrict__ d0, float* __restrict__ P2,
                                                 float* __restrict__ P1, float* __restrict__ P0,
                                                 float* __restrict__ R21, float* __restrict__ R20) {
    // P2 / P1 / P0 = padded d2 / d1 / d0; R21 = ex2(d1 - d2), R20 = ex2(d0 - d2) (0 off the support)
    const int bh = blockIdx.y;
    const int j = blockIdx.x * 256 + threadIdx.x;
    if (j >= Lp) return;
    const bool act = j < L && (mask == nullptr || mask[(size_t)(bh / H) * L + j] != 0);
    const size_t src = (size_t)bh * Lr + j, dst = (size_t)bh * Lp + j;
    const float x2 = act ? d2[src] : -INFINITY;
    P2[dst] = x2;
    if (P1) P1[dst] = act ? d1[src] : -INFINITY;
    if (P0) P0[dst] = act ? d0[src] : -INFINITY;
    if (R21) R21[dst] = act ? ex2(d1[src] - x2) : 0.f;
    if (R20) R20[dst] = act ? ex2(d0[src] - x2) : 0.f;
}

static thread_local long long g_bf_launches = 0;
long long bfree_launch_count(bool reset) {
    const long long c = g_bf_launches;
    if (reset) g_bf_launches = 0;
    return c;
}

bool bfree_supported(int d, int w, int dustbin, int esz) {
    static const bool off = getenv("ST_NO_BFREE") != nullptr;
    if (off) return false;
    return esz == 2 && !dustbin && (d == 64 || d == 128) && w >= 64 && w % kCR == 0;
}

namespace {

int bf_num_sms() {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                  const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {  // the driver entry point through the runtime (no -lcuda)
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (getenv("ST_BF_NO_TMA") || cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return (EncodeTiledFn)p;
    }();
    return fn;
}
// [BH][Lr][d] bf16 (raw API tensor) -> boxes of 64 rows x 64 columns (128 bytes), SWIZZLE_128B, zeros past Lr
bool make_tmap(CUtensorMap* m, const void* base, int BH, int Lr, int d, int box_rows = 64) {
    EncodeTiledFn fn = encode_fn();
    if (!fn || !base) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)Lr, (cuuint64_t)BH};
    const cuuint64_t strides[2] = {(cuuint64_t)d * 2, (cuuint64_t)Lr * d * 2};
    const cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1}, es[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int MODE, bool kDirect, int D>
cudaError_t run_sweep(SweepArgs a, cudaStream_t st) {
    const int grid = std::min(bf_num_sms(), a.nblk);
    a.wl_cap = (a.nblk + grid - 1) / grid;
    a.row_bytes = D * 2;
    {   // the V / dO streams straight from the raw tensors through tensor maps (no packed copy) when the driver has them
        using T0 = ModeTraits<MODE, kDirect>;
        const int BH = a.nblk / a.NB;
        a.tma2 = 0;
        if (T0::kB2 && a.rawB2 && (!T0::kZ || a.rawA2)) {
            bool okm = make_tmap(&a.tmB2, a.rawB2, BH, a.Lr_other, D);
            if (okm && T0::kZ) okm = make_tmap(&a.tmA2, a.rawA2, BH, a.Lr_own, D);
            a.tma2 = okm ? 1 : 0;
        }
        if (T0::kB2 && !a.tma2 && !a.B2) return cudaErrorNotSupported;
        a.tma1 = (a.rawA1 && a.rawB1 && make_tmap(&a.tmA1, a.rawA1, BH, a.Lr_own, D) && make_tmap(&a.tmB1, a.rawB1, BH, a.Lr_other, D)) ? 1 : 0;
        if (!a.tma1 && (!a.A1 || !a.B1)) return cudaErrorNotSupported;
    }
    static const int env_dbg = getenv("ST_BF_DBG") ? atoi(getenv("ST_BF_DBG")) : 0;
    static const int env_na = getenv("ST_BF_NA") ? atoi(getenv("ST_BF_NA")) : 0;
    static const int env_ns0 = getenv("ST_BF_NS0") ? atoi(getenv("ST_BF_NS0")) : 0;
    static const int env_ns1 = getenv("ST_BF_NS1") ? atoi(getenv("ST_BF_NS1")) : 0;
    a.dbg = env_dbg;
    const size_t kMax = 227 * 1024;
    using T = ModeTraits<MODE, kDirect>;
    constexpr bool kLong0 = MODE == M_SROW || MODE == M_SCOL, kLong1 = MODE == M_PV;
    // (A buffers, long-ring slots, short-ring slots): the ring whose chunk is also the Y operand lives until
    // the Y accumulation retires it and needs the depth; the other is freed by the S / Z tiles
    static const int plans[][3] = {{2, 8, 3}, {2, 6, 3}, {2, 5, 3}, {1, 6, 3}, {1, 5, 3}, {2, 4, 3}, {1, 4, 3}, {2, 4, 2}, {1, 4, 2}, {1, 3, 2}, {1, 2, 2}};
    bool ok = false;
    for (const auto& pl : plans) {
        const int lng = pl[1], sht = T::kGemm ? pl[2] : std::max(pl[1], pl[2]);
        const int ns0 = kLong0 ? lng : sht, ns1 = !T::kB2 ? 0 : kLong1 ? lng : pl[2];
        if (bs_bytes<MODE, kDirect>(pl[0], ns0, ns1, a.row_bytes, a.maxwin, a.wl_cap) <= kMax) {
            a.NA = pl[0];
            a.NS0 = ns0;
            a.NS1 = ns1;
            ok = true;
            break;
        }
    }
    if (!ok) return cudaErrorNotSupported;
    if (env_na) a.NA = env_na;
    if (env_ns0) a.NS0 = env_ns0;
    if (env_ns1 && T::kB2) a.NS1 = env_ns1;
    const size_t smem = bs_bytes<MODE, kDirect>(a.NA, a.NS0, a.NS1, a.row_bytes, a.maxwin, a.wl_cap);
    if (smem > kMax) return cudaErrorNotSupported;
    auto k = k_bsweep<MODE, kDirect, D>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
#ifdef ST_BF_TRACE
    static unsigned long long* tbuf = nullptr;
    if (getenv("ST_BF_TRACE")) {
        if (!tbuf) cudaMalloc(&tbuf, 128 * 8);
        cudaMemsetAsync(tbuf, 0, 128 * 8, st);
        a.trace = tbuf;
    }
#endif
    k<<<grid, 96 + 32 * kEW, smem, st>>>(a);
    ++g_bf_launches;
#ifdef ST_BF_TRACE
    if (a.trace) {
        unsigned long long h[128];
        cudaStreamSynchronize(st);
        cudaMemcpy(h, tbuf, sizeof(h), cudaMemcpyDeviceToHost);
        const unsigned long long t0 = h[44];
        auto rel = [&](int k2) { return h[k2] ? (long long)(h[k2] - t0) : -1LL; };
        fprintf(stderr, "k_bsweep<%d,%d,%d> NA %d NS0 %d NS1 %d (ns rel. to block %d start of epilogue warp 2)\n", MODE, (int)kDirect, D, a.NA, a.NS0, a.NS1, kTrB);
        {
            const int o = 0;
            fprintf(stderr, " blk %d: start %lld vfull %lld | chunks-end %lld yfull %lld pre-bar %lld post-bar %lld\n", kTrB, rel(o + 44),
                    rel(o + 45), rel(o + 40), rel(o + 41), rel(o + 42), rel(o + 43));
            for (int c = 0; c < 8; ++c)
                fprintf(stderr, "   c%d: S-issue %6lld-%6lld Y-issue %6lld-%6lld | epi tfull %6lld loaded %6lld done %6lld\n", c, rel(o + c), rel(o + 56 + c),
                        rel(o + 8 + c), rel(o + 48 + c), rel(o + 16 + c), rel(o + 24 + c), rel(o + 32 + c));
            for (int w2 = 0; w2 < 16; ++w2)
                fprintf(stderr, "   warp %2d (qd %d grp %d hf %d) chunk %d: tfull %6lld loaded %6lld done %6lld\n", w2 + 2, (w2 + 2) & 3, (w2 >> 2) & 1,
                        w2 >> 3, 2 + ((w2 >> 2) & 1), rel(64 + w2 * 3), rel(64 + w2 * 3 + 1), rel(64 + w2 * 3 + 2));
        }
    }
#endif
    return cudaGetLastError();
}

struct Vecs {
    float *U2, *U1, *ALPHA, *U2B, *AU1, *U1B;
    float *V2, *V1, *V0, *BETA, *DELTA, *GV, *BV1, *V1B;
};
Vecs carve_vecs(const BfGeo& g, float* vec) {
    Vecs v;
    const size_t nq = (size_t)g.BH * g.Lpq, nk = (size_t)g.BH * g.Lpk;
    float* p = vec;
    v.U2 = p; p += nq;
    v.U1 = p; p += nq;
    v.ALPHA = p; p += nq;
    v.U2B = p; p += nq;
    v.AU1 = p; p += nq;
    v.U1B = p; p += nq;
    v.V2 = p; p += nk;
    v.V1 = p; p += nk;
    v.V0 = p; p += nk;
    v.BETA = p; p += nk;
    v.DELTA = p; p += nk;
    v.GV = p; p += nk;
    v.BV1 = p; p += nk;
    v.V1B = p;
    return v;
}

// own = rows (queries) or, transposed, columns (keys)
SweepArgs base_args(const BfGeo& g, bool col) {
    SweepArgs a{};
    a.H = g.H;
    a.w = g.w;
    a.c2 = g.c2;
    a.scale = 1.f;
    a.maxwin = (128 + 2 * g.w + kCR - 1) / kCR * kCR;
    a.L_own = col ? g.Lk : g.Lq;
    a.L_other = col ? g.Lq : g.Lk;
    a.Lr_own = col ? g.Lrk : g.Lrq;
    a.Lr_other = col ? g.Lrq : g.Lrk;
    a.Lp_own = col ? g.Lpk : g.Lpq;
    a.Lp_other = col ? g.Lpq : g.Lpk;
    a.NB = a.Lp_own / 128;
    a.nblk = g.BH * a.NB;
    return a;
}

cudaError_t prep(const BfGeo& g, bool col, const float* d2, const float* d1, const float* d0, float* P2, float* P1,
                 float* P0, float* R21, float* R20, cudaStream_t st) {
    const int L = col ? g.Lk : g.Lq, Lr = col ? g.Lrk : g.Lrq, Lp = col ? g.Lpk : g.Lpq;
    k_bf_prep<<<dim3((Lp + 255) / 256, g.BH), 256, 0, st>>>(g.BH, g.H, L, Lr, Lp, col ? g.col_mask : g.row_mask, d2, d1,
                                                            d0, P2, P1, P0, R21, R20);
    ++g_bf_launches;
    return cudaGetLastError();
}

template <int D>
cudaError_t output_t(const BfGeo& g, const uint8_t* qp, const uint8_t* kp, const uint8_t* vp, const void* Qraw,
                     const void* Kraw, const void* Vraw, const float* u, const float* v, float* vec, float* O, cudaStream_t st) {
    const Vecs V = carve_vecs(g, vec);
    cudaError_t e;
    if ((e = prep(g, false, u, nullptr, nullptr, V.U2, nullptr, nullptr, nullptr, nullptr, st)) != cudaSuccess) return e;
    if ((e = prep(g, true, v, nullptr, nullptr, V.V2, nullptr, nullptr, nullptr, nullptr, st)) != cudaSuccess) return e;
    SweepArgs a = base_args(g, false);
    a.A1 = qp;
    a.B1 = kp;
    a.B2 = vp;
    a.rawB2 = Vraw;
    a.rawA1 = Qraw;
    a.rawB1 = Kraw;
    a.wv[0] = V.V2;
    a.ov[0] = V.U2;
    a.out_mat = O;
    return run_sweep<M_PV, false, D>(a, st);
}

template <bool kDirect, int D>
cudaError_t backward_t(const BfGeo& g, const BfBwd& p, cudaStream_t st) {
    const Vecs V = carve_vecs(g, p.vec);
    cudaError_t e;
#define BF(call) \
    if ((e = (call)) != cudaSuccess) return e
    BF(prep(g, false, p.u2, p.u1, nullptr, V.U2, V.U1, nullptr, V.ALPHA, nullptr, st));
    BF(prep(g, true, p.v2, p.v1, p.v0, V.V2, V.V1, V.V0, V.BETA, V.DELTA, st));
    {   // C1: dV_j = sum_i P22 dO_i;  g_v_j = <V_j, dV_j> = sum_i P22 Z   (own = keys)
        SweepArgs a = base_args(g, true);
        a.A1 = p.kp; a.B1 = p.qp; a.B2 = p.gp; a.rawB2 = p.dO; a.rawA1 = p.K; a.rawB1 = p.Q;
        a.wv[0] = V.U2; a.ov[0] = V.V2;
        a.out_mat = p.dV;
        a.out1 = V.GV;
        a.dot_src = (const __nv_bfloat16*)p.V;
        BF((run_sweep<M_PV, false, D>(a, st)));
    }
    {   // R12: u2b_i = sum_j P22 (Z - g_v_j)
        SweepArgs a = base_args(g, false);
        a.A1 = p.qp; a.B1 = p.kp; a.A2 = p.gp; a.B2 = p.vp; a.rawA2 = p.dO; a.rawB2 = p.V; a.rawA1 = p.Q; a.rawB1 = p.K;
        a.wv[0] = V.V2; a.wv[1] = V.GV; a.ov[0] = V.U2;
        a.out1 = V.U2B;
        BF((run_sweep<M_R12, false, D>(a, st)));
    }
    {   // C3: v1b_j = -beta_j sum_i P22 u2b_i   (direct: -sum_i P21 u2b_i, P21 = ex2(s + u2_i + v1_j))
        SweepArgs a = base_args(g, true);
        a.A1 = p.kp; a.B1 = p.qp; a.rawA1 = p.K; a.rawB1 = p.Q;
        a.wv[0] = V.U2; a.wv[1] = V.U2B; a.ov[0] = kDirect ? V.V1 : V.V2;
        a.fvec = kDirect ? nullptr : V.BETA;
        a.out1 = V.V1B;
        a.out2 = kDirect ? nullptr : V.BV1;
        BF((run_sweep<M_PX, false, D>(a, st)));
    }
    {   // R4: u1b_i = -alpha_i sum_j P22 beta_j v1b_j   (direct: -sum_j P11 v1b_j)
        SweepArgs a = base_args(g, false);
        a.A1 = p.qp; a.B1 = p.kp; a.rawA1 = p.Q; a.rawB1 = p.K;
        a.wv[0] = kDirect ? V.V1 : V.V2; a.wv[1] = kDirect ? V.V1B : V.BV1; a.ov[0] = kDirect ? V.U1 : V.U2;
        a.fvec = kDirect ? nullptr : V.ALPHA;
        a.out1 = V.U1B;
        a.out2 = kDirect ? nullptr : V.AU1;
        BF((run_sweep<M_PX, false, D>(a, st)));
    }
    {   // R6: dQ_i = inv sum_j Sbar K_j, d_eps partials
        SweepArgs a = base_args(g, false);
        a.A1 = p.qp; a.B1 = p.kp; a.A2 = p.gp; a.B2 = p.vp; a.rawA2 = p.dO; a.rawB2 = p.V; a.rawA1 = p.Q; a.rawB1 = p.K;
        if (kDirect) {
            a.ov[0] = V.U2; a.ov[1] = V.U1; a.ov[2] = V.U2B; a.ov[3] = V.U1B;
            a.wv[0] = V.V2; a.wv[1] = V.V1; a.wv[2] = V.V0; a.wv[3] = V.GV; a.wv[4] = V.V1B;
        } else {
            a.ov[0] = V.U2; a.ov[1] = V.U2B; a.ov[2] = V.ALPHA; a.ov[3] = V.AU1;
            a.wv[0] = V.V2; a.wv[1] = V.GV; a.wv[2] = V.BETA; a.wv[3] = V.BV1; a.wv[4] = V.DELTA;
        }
        a.out_mat = p.dQ;
        a.scale = g.inv_qk;
        a.out_api = p.deps_part;
        BF((run_sweep<M_SROW, kDirect, D>(a, st)));
    }
    {   // C6 (+ C5): dK_j = inv sum_i Sbar Q_i;  v0b_j = -delta_j sum_i P22 alpha_i u1b_i
        SweepArgs a = base_args(g, true);
        a.A1 = p.kp; a.B1 = p.qp; a.A2 = p.vp; a.B2 = p.gp; a.rawA2 = p.V; a.rawB2 = p.dO; a.rawA1 = p.K; a.rawB1 = p.Q;
        if (kDirect) {
            a.ov[0] = V.V2; a.ov[1] = V.V1; a.ov[2] = V.V0; a.ov[3] = V.GV; a.ov[4] = V.V1B;
            a.wv[0] = V.U2; a.wv[1] = V.U1; a.wv[2] = V.U2B; a.wv[3] = V.U1B;
        } else {
            a.ov[0] = V.V2; a.ov[1] = V.GV; a.ov[2] = V.BETA; a.ov[3] = V.BV1; a.ov[4] = V.DELTA;
            a.wv[0] = V.U2; a.wv[1] = V.U2B; a.wv[2] = V.ALPHA; a.wv[3] = V.AU1;
        }
        a.out_mat = p.dK;
        a.scale = g.inv_qk;
        a.out_api = p.eta_v;
        BF((run_sweep<M_SCOL, kDirect, D>(a, st)));
    }
#undef BF
    return cudaSuccess;
}

}  // namespace

bool bfree_tma_available() { return encode_fn() != nullptr; }
bool bfree_make_tmap(CUtensorMap* m, const void* base, int BH, int Lr, int d, int box_rows) {
    return make_tmap(m, base, BH, Lr, d, box_rows);
}

cudaError_t launch_bfree_output(const BfGeo& g, const uint8_t* qp, const uint8_t* kp, const uint8_t* vp, const void* Qraw,
                                const void* Kraw, const void* Vraw, const float* u, const float* v, float* vec, float* O,
                                cudaStream_t s) {
    if (g.d == 128) return output_t<128>(g, qp, kp, vp, Qraw, Kraw, Vraw, u, v, vec, O, s);
    if (g.d == 64) return output_t<64>(g, qp, kp, vp, Qraw, Kraw, Vraw, u, v, vec, O, s);
    return cudaErrorNotSupported;
}

cudaError_t launch_bfree_backward(const BfGeo& g, const BfBwd& p, bool direct, cudaStream_t s) {
    if (g.d == 128) return direct ? backward_t<true, 128>(g, p, s) : backward_t<false, 128>(g, p, s);
    if (g.d == 64) return direct ? backward_t<true, 64>(g, p, s) : backward_t<false, 64>(g, p, s);
    return cudaErrorNotSupported;
}

}  // namespace st
