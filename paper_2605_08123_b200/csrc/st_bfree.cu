// st_bfree.cu -- band-free tcgen05 sweeps for bf16 inputs: the transport output O = P V
// (apply_transport, sinkhorn.hpp:257-277) and the exact R=2 adjoint (r2_backward,
// adjoint.hpp:232-373; one-reference form adjoint.hpp:202-226, direct four-plan form
// adjoint.hpp:311-368) without any stored L x W band.
//
// One kernel, k_bsweep<MODE>, streams the band of a 128-row block ("own" side, one TMEM lane
// per row) through its 64-column window chunks ("other" side):
//   tile   S_c = A1_blk B1_c^T  (and Z_c = A2_blk B2_c^T where the stage needs the cotangent
//          tile) on tcgen05 (kind::f16, fp32 accumulation in TMEM) from the packed operand planes
//   cell   p = ex2(c2 S + a_i + b_j) on the band (a, b = -inf padded duals), then per stage
//            PV    weight = p                      -> Y += W X_c       (O = P V; dV = P^T dO, g_v)
//            R12   acc_i += p (z - g_v_j)                              (u2_bar)
//            PX    acc_i += p x_j                                      (v1_bar, u1_bar)
//            SBAR  weight = Sbar (one-reference modifier field or the four-plan form)
//                                                  -> Y += W X_c       (dQ + d_eps;  dK + v0_bar)
//   GEMM   the weights go to SMEM as two bf16 planes (hi + lo: 16 mantissa bits) in the UMMA
//          K-major core-matrix layout; the chunk's operand rows X_c are the packed plane itself
//          read MN-major (the same 8 x 16-byte core matrices), so Y[128][d] (+)= W X_c is two
//          tcgen05.mma per 16 window columns into a TMEM accumulator.
// Column stages are the same kernel on the transposed geometry (own = keys: A1 = K, B1 = Q).
// Nothing of size L x W is written or read: HBM holds the packed planes (O(L d)), the padded
// dual / cotangent vectors (O(L)) and the outputs.
//
// Roles (persistent CTA, one per SM):
//   warp 0      producer: 1-D bulk async copies (TMA engine) of the block operands, the window
//               chunks and the window / own vectors
//   warp 1      MMA issuer: polls the tile and weight barriers, issues S / Z tiles one chunk ahead
//               of the Y accumulation
//   warps 2-17  epilogue: TMEM lane quadrant x column half x chunk parity; a thread owns one row
//               and 32 columns of every other chunk, so every row reduction is in-thread and the
//               four parts of a row combine in a fixed order.
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
constexpr int kWPlane = 128 * kCR * 2;  // bytes of one bf16 weight plane of a chunk

enum { M_PV = 0, M_R12 = 1, M_PX = 2, M_SROW = 3, M_SCOL = 4 };

struct SweepArgs {
    int NA, NSK, row_bytes, maxwin;
    int H, NB, nblk;
    int L_own, L_other, Lr_own, Lp_own, Lp_other, w;
    int wl_cap;
    float c2, scale;
    const uint8_t *A1, *B1, *A2, *B2;
    const float* wv[5];  // window vectors [BH][Lp_other]; wv[0] = exponent offsets (-inf when inactive)
    const float* ov[5];  // own vectors [BH][Lp_own]; ov[0] = exponent offsets
    float* out_mat;      // [BH][Lr_own][D]
    float* out1;         // [BH][Lp_own]
    float* out2;         // [BH][Lp_own] or null
    float* out_api;      // [BH][Lr_own] or null
    const float* fvec;   // PX: own-side factor [BH][Lp_own] (null = 1)
    const __nv_bfloat16* dot_src;  // PV: raw rows [BH][Lr_own][D] for <Y_i, src_i> (null = none)
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
    uint8_t* B;    // [NSK][(1 + B2) * 64 * row_bytes]
    uint8_t* W;    // [2][2 planes][128 * 64 * 2]
    float* vw;     // [kNV][NW][maxwin]
    float* vo;     // [kNV][NO][128]
    float* rowx;   // [2][4][128]
    uint64_t *v_full, *v_empty, *a_full, *a_empty, *k_full, *k_empty, *t_full, *t_empty, *w_full, *w_empty, *y_full,
        *y_empty;
    uint32_t* tmem_base;
    int4* bd;
};

template <int MODE, bool kDirect>
__host__ __device__ inline size_t bs_bytes(int NA, int NSK, int row_bytes, int maxwin, int wl_cap) {
    using T = ModeTraits<MODE, kDirect>;
    size_t n = (size_t)NA * (T::kZ ? 2 : 1) * 128 * row_bytes + (size_t)NSK * (T::kB2 ? 2 : 1) * kCR * row_bytes;
    if (T::kGemm) n += 2 * 2 * kWPlane;
    n += (size_t)kNV * (T::NW * maxwin + T::NO * 128) * 4 + 2 * 4 * 128 * 4;
    n += (size_t)(2 * kNV + 2 * NA + 2 * NSK + 12) * 8 + 16 + (size_t)wl_cap * 16;
    return n;
}

template <int MODE, bool kDirect>
__device__ __forceinline__ BSmem bcarve(uint8_t* base, const SweepArgs& a) {
    using T = ModeTraits<MODE, kDirect>;
    BSmem s;
    s.A = base;
    s.B = s.A + (size_t)a.NA * (T::kZ ? 2 : 1) * 128 * a.row_bytes;
    s.W = s.B + (size_t)a.NSK * (T::kB2 ? 2 : 1) * kCR * a.row_bytes;
    s.vw = (float*)(s.W + (T::kGemm ? 2 * 2 * kWPlane : 0));
    s.vo = s.vw + kNV * T::NW * a.maxwin;
    s.rowx = s.vo + kNV * T::NO * 128;
    uint64_t* b = (uint64_t*)(s.rowx + 2 * 4 * 128);
    s.v_full = b; b += kNV;
    s.v_empty = b; b += kNV;
    s.a_full = b; b += a.NA;
    s.a_empty = b; b += a.NA;
    s.k_full = b; b += a.NSK;
    s.k_empty = b; b += a.NSK;
    s.t_full = b; b += 2;
    s.t_empty = b; b += 2;
    s.w_full = b; b += 2;
    s.w_empty = b; b += 2;
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

template <int MODE, bool kDirect, int D>
__global__ void __launch_bounds__(64 + 32 * kEW, 1) k_bsweep(SweepArgs a) {
    using T = ModeTraits<MODE, kDirect>;
    constexpr bool kZ = T::kZ, kGemm = T::kGemm, kB2 = T::kB2;
    constexpr int NW = T::NW, NO = T::NO;
    constexpr int TCOLS = kCR * (kZ ? 2 : 1);  // TMEM columns of one chunk buffer (S | Z)
    constexpr int YC = kGemm ? 2 * D : 0;      // two Y accumulators ahead of the chunk buffers
    constexpr int NE = 32 * kEW;
    static_assert(YC + 2 * TCOLS <= 512, "TMEM budget");
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const BSmem s = bcarve<MODE, kDirect>(smem_raw, a);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t blk_bytes = 128u * a.row_bytes, chk_bytes = (uint32_t)kCR * a.row_bytes;
    const uint32_t a_stride = blk_bytes * (kZ ? 2 : 1), b_stride = chk_bytes * (kB2 ? 2 : 1);

    if (threadIdx.x == 0) {
        for (int k = 0; k < kNV; ++k) {
            mbar_init(&s.v_full[k], 1);
            mbar_init(&s.v_empty[k], kEW);
        }
        for (int k = 0; k < a.NA; ++k) {
            mbar_init(&s.a_full[k], 1);
            mbar_init(&s.a_empty[k], 1);
        }
        for (int k = 0; k < a.NSK; ++k) {
            mbar_init(&s.k_full[k], 1);
            mbar_init(&s.k_empty[k], 1);
        }
        for (int k = 0; k < 2; ++k) {
            mbar_init(&s.t_full[k], 1);
            mbar_init(&s.t_empty[k], kEW / 2);
            mbar_init(&s.w_full[k], kEW / 2);
            mbar_init(&s.w_empty[k], 1);
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
        // ------------------------------------------------------------ producer
        uint32_t cs = 0;
        for (int bi = 0; bi < nb; ++bi) {
            const int4 b = s.bd[bi];
            const int i0 = b.y * 128, nch = b.w - b.z + 1, wbase = b.z * kCR, nwin = nch * kCR;
            {
                const int vs = bi % kNV;
                mbar_wait(&s.v_empty[vs], ((bi / kNV) & 1) ^ 1);
                if (elect_one()) {
                    mbar_arrive_expect_tx(&s.v_full[vs], (uint32_t)(NW * nwin + NO * 128) * 4u);
#pragma unroll
                    for (int k = 0; k < NW; ++k)
                        bulk_g2s(s.vw + ((size_t)vs * NW + k) * a.maxwin, a.wv[k] + (size_t)b.x * a.Lp_other + wbase,
                                 (uint32_t)nwin * 4u, &s.v_full[vs]);
#pragma unroll
                    for (int k = 0; k < NO; ++k)
                        bulk_g2s(s.vo + ((size_t)vs * NO + k) * 128, a.ov[k] + (size_t)b.x * a.Lp_own + i0, 512u,
                                 &s.v_full[vs]);
                }
                __syncwarp();
            }
            const int ab = bi % a.NA;
            mbar_wait(&s.a_empty[ab], ((bi / a.NA) & 1) ^ 1);
            if (elect_one()) {
                mbar_arrive_expect_tx(&s.a_full[ab], a_stride);
                const size_t off = ((size_t)b.x * a.Lp_own + i0) * a.row_bytes;
                bulk_g2s(s.A + (size_t)ab * a_stride, a.A1 + off, blk_bytes, &s.a_full[ab]);
                if (kZ) bulk_g2s(s.A + (size_t)ab * a_stride + blk_bytes, a.A2 + off, blk_bytes, &s.a_full[ab]);
            }
            __syncwarp();
            for (int q = b.z; q <= b.w; ++q, ++cs) {
                const int sl = cs % a.NSK;
                mbar_wait(&s.k_empty[sl], ((cs / a.NSK) & 1) ^ 1);
                if (elect_one()) {
                    mbar_arrive_expect_tx(&s.k_full[sl], b_stride);
                    const size_t off = ((size_t)b.x * a.Lp_other + (size_t)q * kCR) * a.row_bytes;
                    bulk_g2s(s.B + (size_t)sl * b_stride, a.B1 + off, chk_bytes, &s.k_full[sl]);
                    if (kB2) bulk_g2s(s.B + (size_t)sl * b_stride + chk_bytes, a.B2 + off, chk_bytes, &s.k_full[sl]);
                }
                __syncwarp();
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        const uint32_t idesc_s = make_idesc(128, kCR, 1u);
        const uint32_t idesc_y = make_idesc_bmn(128, D);
        const uint32_t sbo = (uint32_t)a.row_bytes * 8u;
        const int ksteps = a.row_bytes / 32;
        // S / Z cursor and Y cursor over (block, chunk); cs = running chunk number
        int sb = 0, sc = 0, yb = 0, yc = 0;
        uint32_t scs = 0, ycs = 0;
        int s_nch = nb > 0 ? s.bd[0].w - s.bd[0].z + 1 : 0;
        int y_nch = s_nch;
        while (sb < nb || (kGemm && yb < nb)) {
            if (sb < nb) {
                const int ab = sb % a.NA;
                const uint32_t sl = scs % a.NSK, tb = scs & 1;
                bool ok = (sc > 0 || mbar_test(&s.a_full[ab], (sb / a.NA) & 1)) &&
                          mbar_test(&s.k_full[sl], (scs / a.NSK) & 1) && mbar_test(&s.t_empty[tb], ((scs >> 1) & 1) ^ 1);
                ok = __shfl_sync(0xffffffffu, ok ? 1 : 0, 0) != 0;
                if (ok) {
                    tc_fence_after();
                    if (elect_one()) {
                        const uint64_t ad = make_desc(smem_u32(s.A + (size_t)ab * a_stride), 128, sbo);
                        const uint64_t bd = make_desc(smem_u32(s.B + (size_t)sl * b_stride), 128, sbo);
                        const uint32_t dt = tbase + YC + tb * TCOLS;
                        for (int kk = 0; kk < ksteps; ++kk)
                            mma_bf16(dt, ad + (uint64_t)(kk * 16), bd + (uint64_t)(kk * 16), idesc_s, kk > 0);
                        if (kZ) {
                            const uint64_t ad2 = make_desc(smem_u32(s.A + (size_t)ab * a_stride + blk_bytes), 128, sbo);
                            const uint64_t bd2 = make_desc(smem_u32(s.B + (size_t)sl * b_stride + chk_bytes), 128, sbo);
                            for (int kk = 0; kk < ksteps; ++kk)
                                mma_bf16(dt + kCR, ad2 + (uint64_t)(kk * 16), bd2 + (uint64_t)(kk * 16), idesc_s, kk > 0);
                        }
                        tc_commit(&s.t_full[tb]);
                        if (sc == s_nch - 1) tc_commit(&s.a_empty[ab]);
                        if (!kGemm) tc_commit(&s.k_empty[sl]);
                    }
                    __syncwarp();
                    ++scs;
                    if (++sc == s_nch) {
                        sc = 0;
                        ++sb;
                        if (sb < nb) s_nch = s.bd[sb].w - s.bd[sb].z + 1;
                    }
                }
            }
            if (kGemm && yb < nb && ycs < scs) {
                const uint32_t wb = ycs & 1, sl = ycs % a.NSK, ybuf = yb & 1;
                bool ok = mbar_test(&s.w_full[wb], (ycs >> 1) & 1) &&
                          (yc > 0 || mbar_test(&s.y_empty[ybuf], ((yb >> 1) & 1) ^ 1));
                ok = __shfl_sync(0xffffffffu, ok ? 1 : 0, 0) != 0;
                if (ok) {
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t dy = tbase + ybuf * D;
                        const uint8_t* xs = s.B + (size_t)sl * b_stride + (MODE == M_PV ? chk_bytes : 0);
                        const uint64_t xd = make_desc(smem_u32(xs), sbo, 128);
#pragma unroll
                        for (int p = 0; p < 2; ++p) {
                            const uint64_t wd = make_desc(smem_u32(s.W + (size_t)(wb * 2 + p) * kWPlane), 2048, 128);
#pragma unroll
                            for (int kk = 0; kk < kCR / 16; ++kk)
                                mma_bf16(dy, wd + (uint64_t)(kk * 256), xd + (uint64_t)(kk * a.row_bytes), idesc_y,
                                         (yc > 0 || p > 0 || kk > 0) ? 1u : 0u);
                        }
                        tc_commit(&s.w_empty[wb]);
                        tc_commit(&s.k_empty[sl]);
                        if (yc == y_nch - 1) tc_commit(&s.y_full[ybuf]);
                    }
                    __syncwarp();
                    ++ycs;
                    if (++yc == y_nch) {
                        yc = 0;
                        ++yb;
                        if (yb < nb) y_nch = s.bd[yb].w - s.bd[yb].z + 1;
                    }
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
            mbar_wait(&s.v_full[vs], (bi / kNV) & 1);
            const float* vwp = s.vw + (size_t)vs * NW * a.maxwin;
            float O[NO];
#pragma unroll
            for (int k = 0; k < NO; ++k) O[k] = s.vo[((size_t)vs * NO + k) * 128 + r];
            float acc = 0.f;
            for (int c = 0; c < nch; ++c, ++cs) {
                if ((int)(cs & 1) != gidx) continue;
                const uint32_t tb = cs & 1;
                const int c0 = c * kCR + 32 * hf;  // first window column of this warp's slice
                const bool outside = c0 + 31 < lo_min || c0 > lo_min + 31 + (int)bw;
                const bool edge = !(c0 >= lo_min + 31 && c0 + 31 <= lo_min + (int)bw);
                uint8_t* wrow = s.W + (size_t)(tb * 2) * kWPlane + (size_t)(4 * hf) * 2048 + (size_t)r * 16;
                mbar_wait(&s.t_full[tb], (cs >> 1) & 1);
                if (outside) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&s.t_empty[tb]);
                    if (kGemm) {
                        mbar_wait(&s.w_empty[tb], ((cs >> 1) & 1) ^ 1);
#pragma unroll
                        for (int kg = 0; kg < 4; ++kg) {
                            *reinterpret_cast<uint4*>(wrow + kg * 2048) = make_uint4(0, 0, 0, 0);
                            *reinterpret_cast<uint4*>(wrow + kWPlane + kg * 2048) = make_uint4(0, 0, 0, 0);
                        }
                        fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&s.w_full[tb]);
                    }
                    continue;
                }
                tc_fence_after();
                float sv[2][16], zv[2][16];
                const uint32_t ta = tl + YC + tb * TCOLS + 32 * hf;
                tc_ld16(ta, sv[0]);
                tc_ld16(ta + 16, sv[1]);
                if (kZ) {
                    tc_ld16(ta + kCR, zv[0]);
                    tc_ld16(ta + kCR + 16, zv[1]);
                }
                tc_wait_ld();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&s.t_empty[tb]);
                if (kGemm) mbar_wait(&s.w_empty[tb], ((cs >> 1) & 1) ^ 1);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
#pragma unroll
                    for (int g8 = 0; g8 < 2; ++g8) {
                        float wg[8];
#pragma unroll
                        for (int q4 = 0; q4 < 2; ++q4) {
                            const int cc = c0 + 16 * h + 8 * g8 + 4 * q4;
                            float wvv[NW][4];
#pragma unroll
                            for (int k = 0; k < NW; ++k) {
                                const float4 t4 = *reinterpret_cast<const float4*>(vwp + (size_t)k * a.maxwin + cc);
                                wvv[k][0] = t4.x;
                                wvv[k][1] = t4.y;
                                wvv[k][2] = t4.z;
                                wvv[k][3] = t4.w;
                            }
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const int kx = 8 * g8 + 4 * q4 + e;
                                const float sc_ = sv[h][kx];
                                const bool inb = !edge || (unsigned)(cc + e - lo) <= bw;
                                const float e0 = sc_ * a.c2;
                                float zz = e0 + wvv[0][e] + O[0];
                                zz = inb ? zz : -INFINITY;
                                const float p = ex2(zz);
                                float wgt = p;
                                if constexpr (MODE == M_R12) {
                                    acc = fmaf(p, zv[h][kx] - wvv[1][e], acc);
                                } else if constexpr (MODE == M_PX) {
                                    acc = fmaf(p, wvv[1][e], acc);
                                } else if constexpr (MODE == M_SROW) {
                                    const float z = zv[h][kx];
                                    if constexpr (!kDirect) {
                                        // O = (a, u2b, alpha, au1); W = (b, v2b, beta, bv1, delta)
                                        const float m = fmaf(wvv[4][e], O[3], fmaf(wvv[3][e], O[2], fmaf(wvv[2][e], O[1], wvv[1][e])));
                                        wgt = p * (z - m);
                                    } else {
                                        // O = (u2, u1, u2b, u1b); W = (v2, v1, v0, v2b, v1b)
                                        const float em = inb ? e0 : -INFINITY;
                                        const float p21 = ex2(em + O[0] + wvv[1][e]);
                                        const float p11 = ex2(em + O[1] + wvv[1][e]);
                                        const float p10 = ex2(em + O[1] + wvv[2][e]);
                                        wgt = p * (z - wvv[3][e]) - O[2] * p21 - p11 * wvv[4][e] - O[3] * p10;
                                    }
                                    acc = fmaf(wgt, sc_ * c2ln2, acc);
                                } else if constexpr (MODE == M_SCOL) {
                                    const float z = zv[h][kx];
                                    if constexpr (!kDirect) {
                                        // O = (a = v2, v2b, beta, bv1, delta); W = (b = u2, u2b, alpha, au1)
                                        const float m = fmaf(O[4], wvv[3][e], fmaf(O[3], wvv[2][e], fmaf(O[2], wvv[1][e], O[1])));
                                        wgt = p * (z - m);
                                        acc = fmaf(p, wvv[3][e], acc);
                                    } else {
                                        // O = (v2, v1, v0, v2b, v1b); W = (u2, u1, u2b, u1b)
                                        const float em = inb ? e0 : -INFINITY;
                                        const float p21 = ex2(em + wvv[0][e] + O[1]);
                                        const float p11 = ex2(em + wvv[1][e] + O[1]);
                                        const float p10 = ex2(em + wvv[1][e] + O[2]);
                                        wgt = p * (z - O[3]) - wvv[2][e] * p21 - p11 * O[4] - wvv[3][e] * p10;
                                        acc = fmaf(p10, wvv[3][e], acc);
                                    }
                                }
                                wg[4 * q4 + e] = wgt;
                            }
                        }
                        if (kGemm) {
                            uint32_t hw[4], lw[4];
#pragma unroll
                            for (int k2 = 0; k2 < 4; ++k2) {
                                const __nv_bfloat16 h0 = __float2bfloat16_rn(wg[2 * k2]), h1 = __float2bfloat16_rn(wg[2 * k2 + 1]);
                                hw[k2] = (uint32_t)__bfloat16_as_ushort(h0) | ((uint32_t)__bfloat16_as_ushort(h1) << 16);
                                lw[k2] = pack_bf16(wg[2 * k2] - __bfloat162float(h0), wg[2 * k2 + 1] - __bfloat162float(h1));
                            }
                            const int kg = 2 * h + g8;
                            *reinterpret_cast<uint4*>(wrow + kg * 2048) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
                            *reinterpret_cast<uint4*>(wrow + kWPlane + kg * 2048) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
                        }
                    }
                }
                if (kGemm) {
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&s.w_full[tb]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.v_empty[vs]);
            const size_t orow = (size_t)b.x * a.Lr_own + i;
            if (kGemm) {
                // ---- drain this block's accumulator: the warp's quarter of the D output columns
                constexpr int QC = D / 4;
                const uint32_t ybuf = bi & 1;
                mbar_wait(&s.y_full[ybuf], (bi >> 1) & 1);
                tc_fence_after();
                float y[QC];
                tc_ldn<QC>(tl + ybuf * D + part * QC, y);
                tc_wait_ld();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&s.y_empty[ybuf]);
                if (i < a.L_own) {
                    float* dst = a.out_mat + orow * D + part * QC;
#pragma unroll
                    for (int q = 0; q < QC / 4; ++q)
                        *reinterpret_cast<float4*>(dst + 4 * q) =
                            make_float4(y[4 * q] * a.scale, y[4 * q + 1] * a.scale, y[4 * q + 2] * a.scale, y[4 * q + 3] * a.scale);
                    if (MODE == M_PV && a.dot_src) {
                        const uint4* src = reinterpret_cast<const uint4*>(a.dot_src + orow * D + part * QC);
                        float dsum = 0.f;
#pragma unroll
                        for (int q = 0; q < QC / 8; ++q) {
                            const uint4 v8 = src[q];
                            const uint32_t ww[4] = {v8.x, v8.y, v8.z, v8.w};
#pragma unroll
                            for (int k2 = 0; k2 < 4; ++k2) {
                                dsum = fmaf(y[8 * q + 2 * k2], __uint_as_float(ww[k2] << 16), dsum);
                                dsum = fmaf(y[8 * q + 2 * k2 + 1], __uint_as_float(ww[k2] & 0xffff0000u), dsum);
                            }
                        }
                        acc = dsum;
                    }
                }
            }
            if (MODE != M_PV || a.dot_src) {
                // ---- the four parts of a row combine in a fixed order
                float* rx = s.rowx + (size_t)par * 4 * 128;
                rx[part * 128 + r] = acc;
                named_bar(1, NE);
                if (part == 0) {
                    const float tot = (rx[r] + rx[128 + r]) + (rx[256 + r] + rx[384 + r]);
                    const size_t prow = (size_t)b.x * a.Lp_own + i;
                    if constexpr (MODE == M_PV || MODE == M_R12) {
                        a.out1[prow] = tot;
                    } else if constexpr (MODE == M_PX) {
                        const float f = a.fvec ? a.fvec[prow] : 1.f;
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
    if (getenv("ST_NO_BFREE")) return false;
    return esz == 2 && !dustbin && (d == 64 || d == 128) && w >= 64 && w % kCR == 0;
}

namespace {

int bf_num_sms() {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
}

template <int MODE, bool kDirect, int D>
cudaError_t run_sweep(SweepArgs a, cudaStream_t st) {
    const int grid = std::min(bf_num_sms(), a.nblk);
    a.wl_cap = (a.nblk + grid - 1) / grid;
    a.row_bytes = D * 2;
    const size_t kMax = 227 * 1024;
    bool ok = false;
    for (int NA = 2; NA >= 1 && !ok; --NA)
        for (int NSK = 4; NSK >= 2 && !ok; --NSK)
            if (bs_bytes<MODE, kDirect>(NA, NSK, a.row_bytes, a.maxwin, a.wl_cap) <= kMax) {
                a.NA = NA;
                a.NSK = NSK;
                ok = true;
            }
    if (!ok) return cudaErrorNotSupported;
    if (getenv("ST_BF_NA")) a.NA = atoi(getenv("ST_BF_NA"));
    if (getenv("ST_BF_NSK")) a.NSK = atoi(getenv("ST_BF_NSK"));
    const size_t smem = bs_bytes<MODE, kDirect>(a.NA, a.NSK, a.row_bytes, a.maxwin, a.wl_cap);
    auto k = k_bsweep<MODE, kDirect, D>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<grid, 64 + 32 * kEW, smem, st>>>(a);
    ++g_bf_launches;
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
cudaError_t output_t(const BfGeo& g, const uint8_t* qp, const uint8_t* kp, const uint8_t* vp, const float* u,
                     const float* v, float* vec, float* O, cudaStream_t st) {
    const Vecs V = carve_vecs(g, vec);
    cudaError_t e;
    if ((e = prep(g, false, u, nullptr, nullptr, V.U2, nullptr, nullptr, nullptr, nullptr, st)) != cudaSuccess) return e;
    if ((e = prep(g, true, v, nullptr, nullptr, V.V2, nullptr, nullptr, nullptr, nullptr, st)) != cudaSuccess) return e;
    SweepArgs a = base_args(g, false);
    a.A1 = qp;
    a.B1 = kp;
    a.B2 = vp;
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
        a.A1 = p.kp; a.B1 = p.qp; a.B2 = p.gp;
        a.wv[0] = V.U2; a.ov[0] = V.V2;
        a.out_mat = p.dV;
        a.out1 = V.GV;
        a.dot_src = (const __nv_bfloat16*)p.V;
        BF((run_sweep<M_PV, false, D>(a, st)));
    }
    {   // R12: u2b_i = sum_j P22 (Z - g_v_j)
        SweepArgs a = base_args(g, false);
        a.A1 = p.qp; a.B1 = p.kp; a.A2 = p.gp; a.B2 = p.vp;
        a.wv[0] = V.V2; a.wv[1] = V.GV; a.ov[0] = V.U2;
        a.out1 = V.U2B;
        BF((run_sweep<M_R12, false, D>(a, st)));
    }
    {   // C3: v1b_j = -beta_j sum_i P22 u2b_i   (direct: -sum_i P21 u2b_i, P21 = ex2(s + u2_i + v1_j))
        SweepArgs a = base_args(g, true);
        a.A1 = p.kp; a.B1 = p.qp;
        a.wv[0] = V.U2; a.wv[1] = V.U2B; a.ov[0] = kDirect ? V.V1 : V.V2;
        a.fvec = kDirect ? nullptr : V.BETA;
        a.out1 = V.V1B;
        a.out2 = kDirect ? nullptr : V.BV1;
        BF((run_sweep<M_PX, false, D>(a, st)));
    }
    {   // R4: u1b_i = -alpha_i sum_j P22 beta_j v1b_j   (direct: -sum_j P11 v1b_j)
        SweepArgs a = base_args(g, false);
        a.A1 = p.qp; a.B1 = p.kp;
        a.wv[0] = kDirect ? V.V1 : V.V2; a.wv[1] = kDirect ? V.V1B : V.BV1; a.ov[0] = kDirect ? V.U1 : V.U2;
        a.fvec = kDirect ? nullptr : V.ALPHA;
        a.out1 = V.U1B;
        a.out2 = kDirect ? nullptr : V.AU1;
        BF((run_sweep<M_PX, false, D>(a, st)));
    }
    {   // R6: dQ_i = inv sum_j Sbar K_j, d_eps partials
        SweepArgs a = base_args(g, false);
        a.A1 = p.qp; a.B1 = p.kp; a.A2 = p.gp; a.B2 = p.vp;
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
        a.A1 = p.kp; a.B1 = p.qp; a.A2 = p.vp; a.B2 = p.gp;
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

cudaError_t launch_bfree_output(const BfGeo& g, const uint8_t* qp, const uint8_t* kp, const uint8_t* vp,
                                const float* u, const float* v, float* vec, float* O, cudaStream_t s) {
    if (g.d == 128) return output_t<128>(g, qp, kp, vp, u, v, vec, O, s);
    if (g.d == 64) return output_t<64>(g, qp, kp, vp, u, v, vec, O, s);
    return cudaErrorNotSupported;
}

cudaError_t launch_bfree_backward(const BfGeo& g, const BfBwd& p, bool direct, cudaStream_t s) {
    if (g.d == 128) return direct ? backward_t<true, 128>(g, p, s) : backward_t<false, 128>(g, p, s);
    if (g.d == 64) return direct ? backward_t<true, 64>(g, p, s) : backward_t<false, 64>(g, p, s);
    return cudaErrorNotSupported;
}

}  // namespace st
