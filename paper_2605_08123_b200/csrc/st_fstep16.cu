// st_fstep16.cu -- the tcgen05 FULL-STEP kernel of the bf16 Sinkhorn forward:
// one score evaluation per full step (row_half_step + col_half_step,
// sinkhorn.hpp:15-107, fused as in advance_full_step, sinkhorn.hpp:146-164).
//
// Per 128-row block I of one head (one TMEM lane per row), with the previous
// duals u^{t-1} (own rows) and v^{t-1} (window columns):
//   S  = Q_I K_win^T on tcgen05 (kind::f16, fp32 accumulation in TMEM); the
//        window is the block's <= 3 CR-column chunks, held in TMEM together
//   e_ij = ex2( s2_ij + v_j + o_i ),  o_i = u^{t-1}_i   (row pass; e written back
//        over S in TMEM: tcgen05.st)
//   r_i  = sum_j e_ij   ->   u^t_i = o_i - lg2 r_i    (one thread owns a row's sum
//        over its column part; the 4 parts combine in fixed order)
//   c_Ij = sum_{i in I} e_ij / r_i                    (column pass: e re-read from
//        TMEM, weighted, reduced over the warp's 32 lanes by a transpose
//        butterfly, then over the 4 lane quadrants in fixed order)
// The column partials c_Ij go to HBM ([BH][NB][maxwin], O(L * (1 + 2w/128)));
// k_vmerge then forms v^t_j = v^{t-1}_j - lg2 sum_I c_Ij over the <= 3 blocks
// whose rows meet column j, in ascending block order (deterministic).
// So a full step costs ONE S evaluation, ONE ex2 per cell and one read of the
// packed Q and K planes, against two of each for the row + column half-step pair
// (st_phase.cu).  The cold start (t = 1) takes an online row max per column part
// (the weights of part p then carry 2^(M_p - M)).
//
// Roles (persistent CTA, one per SM), as in k_phase:
//   warp 0   producer: 1-D bulk async copies of the packed Q block, the K window
//            chunks (shared chunks of consecutive blocks loaded once) and the
//            window / own duals from the -inf padded dual buffers
//   warp 1   MMA issuer: M=128, N=CR, K=16 per instruction into a ring of
//            512/CR TMEM slots; a block's chunks stay resident until its column
//            pass released them
//   warps 2..17  epilogue: 4 lane quadrants x 4 column parts (32 columns of every
//            chunk each)
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "st_common.cuh"
#include "st_phase.cuh"
#include "st_sm100.cuh"

namespace st {

using namespace sm100;

namespace {

constexpr int kNV = 3;     // dual-window ring slots
constexpr int kPH = 3;     // epilogue warps per 16-lane half of a TMEM lane quadrant
constexpr int kEW = 8 * kPH;  // epilogue warps
constexpr int kSlc = 4;    // 32-column slices per 128-column chunk

struct FSmem {
    uint8_t* A;       // [NA][128 * row_bytes]
    uint8_t* K;       // [NSK][CR * row_bytes]
    float* vwin;      // [kNV][maxwin + 128]
    float* rowp;      // [2][kPH][128]: row partial (sum, max) per sub-warp (one buffer: two barriers per block)
    float* colp;      // [8][maxwin]: column partials per 16-lane half quadrant
    uint64_t* v_full;
    uint64_t* v_empty;
    uint64_t* a_full;
    uint64_t* a_empty;
    uint64_t* k_full;
    uint64_t* k_empty;
    uint64_t* t_full;
    uint64_t* t_empty;
    uint32_t* tmem_base;
    int* wl;
};

__device__ __forceinline__ FSmem fcarve(uint8_t* base, const PhaseArgs& a, int nst) {
    FSmem s;
    const size_t blk = (size_t)128 * a.row_bytes, chk = (size_t)a.CR * a.row_bytes;
    s.A = base;
    s.K = s.A + (size_t)a.NA * blk;
    s.vwin = (float*)(s.K + (size_t)a.NSK * chk);
    s.rowp = s.vwin + kNV * (a.maxwin + 128);
    s.colp = s.rowp + 2 * kPH * 128;
    uint64_t* bars = (uint64_t*)(s.colp + 8 * a.maxwin);
    s.v_full = bars;
    s.v_empty = bars + kNV;
    bars += 2 * kNV;
    s.a_full = bars;
    s.a_empty = bars + a.NA;
    s.k_full = bars + 2 * a.NA;
    s.k_empty = s.k_full + a.NSK;
    s.t_full = s.k_empty + a.NSK;
    s.t_empty = s.t_full + nst;
    s.tmem_base = (uint32_t*)(s.t_empty + nst);
    s.wl = (int*)(s.tmem_base + 4);
    return s;
}

struct Blk {
    int bh, blk, i0, q0, q1;
};
__device__ __forceinline__ Blk fblock_of(const PhaseArgs& a, int g) {
    Blk b;
    b.bh = g / a.NB;
    b.blk = g % a.NB;
    b.i0 = b.blk * 128;
    const int nq = a.Lp_other / a.CR;
    b.q0 = max(0, (b.i0 - a.w + a.shift) / a.CR);
    b.q1 = min(nq - 1, (b.i0 + 128 + a.w + a.shift + a.CR - 1) / a.CR - 1);
    return b;
}

// Lane c of the warp returns sum over the 32 lanes of x[c] (x is destroyed):
// a transpose butterfly, 31 shuffles per 32 x 32 tile, fixed association order.
__device__ __forceinline__ float colsum32(float (&x)[32], int lane) {
#pragma unroll
    for (int h = 16; h >= 1; h >>= 1) {
        const bool up = (lane & h) != 0;
#pragma unroll
        for (int k = 0; k < h; ++k) {
            const float send = up ? x[k] : x[k + h];
            const float keep = up ? x[k + h] : x[k];
            x[k] = keep + __shfl_xor_sync(0xffffffffu, send, h);
        }
    }
    return x[0];
}

}  // namespace

template <bool kFirst, bool kRecompute>
__global__ void __launch_bounds__(64 + 32 * kEW, 1) k_fstep16(PhaseArgs a, float* __restrict__ part_out) {
    constexpr int NE = 32 * kEW;
    constexpr int kCR = 128;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    constexpr int NST = 512 / kCR;
    const FSmem s = fcarve(smem_raw, a, NST);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t blk_bytes = 128u * a.row_bytes, chk_bytes = (uint32_t)kCR * a.row_bytes;

    if (threadIdx.x == 0) {
        for (int k = 0; k < a.NA; ++k) {
            mbar_init(&s.a_full[k], 1);
            mbar_init(&s.a_empty[k], 1);
        }
        for (int k = 0; k < a.NSK; ++k) {
            mbar_init(&s.k_full[k], 1);
            mbar_init(&s.k_empty[k], 1);
        }
        for (int k = 0; k < NST; ++k) {
            mbar_init(&s.t_full[k], 1);
            mbar_init(&s.t_empty[k], kEW);
        }
        for (int k = 0; k < kNV; ++k) {
            mbar_init(&s.v_full[k], 1);
            mbar_init(&s.v_empty[k], kEW);
        }
        fence_mbar_init();
    }
    if (warp == 1) {
        tc_alloc(s.tmem_base, 512);
        tc_relinquish();
    }
    const int n = a.work ? *a.nwork : a.nwork_all;
    const int g_begin = (int)((long long)n * blockIdx.x / gridDim.x);
    const int g_end = min((int)((long long)n * (blockIdx.x + 1) / gridDim.x), g_begin + a.wl_cap);
    for (int k = threadIdx.x; k < g_end - g_begin; k += blockDim.x) s.wl[k] = a.work ? a.work[g_begin + k] : g_begin + k;
    if (threadIdx.x == 0 && (int)((long long)n * (blockIdx.x + 1) / gridDim.x) - g_begin > a.wl_cap)
        atomicOr(a.err, 16);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *s.tmem_base;

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        int last_bh = -1, last_q = -1;
        uint32_t kseq = 0;
        for (int gi = g_begin; gi < g_end; ++gi) {
            const Blk b = fblock_of(a, s.wl[gi - g_begin]);
            {
                const int vs = (gi - g_begin) % kNV;
                const uint32_t vn = (gi - g_begin) / kNV;
                mbar_wait(&s.v_empty[vs], (vn & 1) ^ 1);
                if (elect_one()) {
                    const int wbase = b.q0 * a.CR - a.shift, nwin = (b.q1 - b.q0 + 1) * a.CR;
                    float* dst = s.vwin + (size_t)vs * (a.maxwin + 128);
                    mbar_arrive_expect_tx(&s.v_full[vs], (uint32_t)(nwin + 128) * 4u);
                    bulk_g2s(dst, a.pad_other + (size_t)b.bh * a.pad_ld_other + a.pad_off + wbase, (uint32_t)nwin * 4u,
                             &s.v_full[vs]);
                    bulk_g2s(dst + a.maxwin, a.pad_own + (size_t)b.bh * a.pad_ld_own + a.pad_off + b.i0, 512u,
                             &s.v_full[vs]);
                }
                __syncwarp();
            }
            const int ab = (gi - g_begin) % a.NA;
            const uint32_t an = (gi - g_begin) / a.NA;
            mbar_wait(&s.a_empty[ab], (an & 1) ^ 1);
            if (elect_one()) {
                mbar_arrive_expect_tx(&s.a_full[ab], blk_bytes);
                bulk_g2s(s.A + (size_t)ab * blk_bytes, a.A_pack[0] + ((size_t)b.bh * a.Lp_own + b.i0 + a.shift) * a.row_bytes,
                         blk_bytes, &s.a_full[ab]);
            }
            __syncwarp();
            const int qstart = (b.bh == last_bh) ? max(b.q0, last_q + 1) : b.q0;
            for (int q = qstart; q <= b.q1; ++q) {
                const int sl = kseq % a.NSK;
                const uint32_t kn = kseq / a.NSK;
                mbar_wait(&s.k_empty[sl], (kn & 1) ^ 1);
                if (elect_one()) {
                    mbar_arrive_expect_tx(&s.k_full[sl], chk_bytes);
                    bulk_g2s(s.K + (size_t)sl * chk_bytes,
                             a.B_pack[0] + ((size_t)b.bh * a.Lp_other + (size_t)q * kCR) * a.row_bytes, chk_bytes,
                             &s.k_full[sl]);
                }
                __syncwarp();
                ++kseq;
            }
            if (b.bh != last_bh) last_q = -1;
            last_q = max(last_q, b.q1);
            last_bh = b.bh;
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        const uint32_t idesc = make_idesc(128, kCR, 1u);
        const uint32_t sbo = (uint32_t)(a.row_bytes / 16) * 128u;
        const int ksteps = a.row_bytes / 32;
        int last_bh = -1, last_q = -1;
        uint32_t last_seq = 0, rel_seq = 0, tseq = 0;
        bool have = false;
        for (int gi = g_begin; gi < g_end; ++gi) {
            const Blk b = fblock_of(a, s.wl[gi - g_begin]);
            const int ab = (gi - g_begin) % a.NA;
            const uint32_t an = (gi - g_begin) / a.NA;
            mbar_wait(&s.a_full[ab], an & 1);
            tc_fence_after();
            const uint64_t ad0 = make_desc(smem_u32(s.A + (size_t)ab * blk_bytes), 128, sbo);
            const bool same = have && b.bh == last_bh;
            const int new_start = same ? max(b.q0, last_q + 1) : b.q0;
            const uint32_t next_seq = have ? last_seq + 1 : 0;
            // chunks are issued as soon as their TMEM slot is free; a chunk whose successor's slot
            // (and K chunk) are ready too is paired with it (independent accumulators hide the
            // dependent-MMA latency of a lone chain)
            auto seq_of = [&](int q) {
                return (same && q <= last_q) ? last_seq - (uint32_t)(last_q - q) : next_seq + (uint32_t)(q - new_start);
            };
            for (int q = b.q0; q <= b.q1;) {
                const uint32_t sq0 = seq_of(q);
                mbar_wait(&s.k_full[sq0 % a.NSK], (sq0 / a.NSK) & 1);
                mbar_wait(&s.t_empty[tseq % NST], ((tseq / NST) & 1) ^ 1);
                int ng = 1;
                if (q + 1 <= b.q1) {
                    const uint32_t sq1 = seq_of(q + 1), t1 = tseq + 1;
                    bool ok = mbar_test(&s.k_full[sq1 % a.NSK], (sq1 / a.NSK) & 1) &&
                              mbar_test(&s.t_empty[t1 % NST], ((t1 / NST) & 1) ^ 1);
                    ok = __shfl_sync(0xffffffffu, ok ? 1 : 0, 0) != 0;
                    if (ok) ng = 2;
                }
                uint64_t bd[2];
                uint32_t dt[2];
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const uint32_t sq = seq_of(q + c);
                    bd[c] = make_desc(smem_u32(s.K + (size_t)(sq % a.NSK) * chk_bytes), 128, sbo);
                    dt[c] = tbase + (uint32_t)(((tseq + c) % NST) * kCR);
                }
                tc_fence_after();
                if (elect_one()) {
                    for (int kk = 0; kk < ksteps; ++kk) {
#pragma unroll
                        for (int c = 0; c < 2; ++c)
                            if (c < ng && (kk == 0 || !(a.dbg & 2)))
                                mma_bf16(dt[c], ad0 + (uint64_t)(kk * 16), bd[c] + (uint64_t)(kk * 16), idesc, kk > 0);
                    }
#pragma unroll
                    for (int c = 0; c < 2; ++c)
                        if (c < ng) tc_commit(&s.t_full[(tseq + c) % NST]);
                }
                __syncwarp();
                tseq += ng;
                q += ng;
            }
            if (elect_one()) tc_commit(&s.a_empty[ab]);
            __syncwarp();
            if (b.q1 >= new_start) last_seq = next_seq + (uint32_t)(b.q1 - new_start);
            if (!same) last_q = -1;
            last_q = max(last_q, b.q1);
            last_bh = b.bh;
            have = true;
            uint32_t keep_from = last_seq + 1;
            if (gi + 1 < g_end) {
                const Blk nb = fblock_of(a, s.wl[gi + 1 - g_begin]);
                if (nb.bh == last_bh && nb.q0 <= last_q) keep_from = last_seq - (uint32_t)(last_q - nb.q0);
            }
            if (elect_one()) {
                for (uint32_t r = rel_seq; r < keep_from; ++r) tc_commit(&s.k_empty[r % a.NSK]);
            }
            __syncwarp();
            rel_seq = max(rel_seq, keep_from);
        }
    } else {
        // ------------------------------------------------------------ epilogue
        // 24 warps: warp % 4 = TMEM lane quadrant; g = (warp - 2) / 4 in 0..5 picks the 16-lane half
        // (g & 1) of the quadrant and the sub-warp k = g >> 1 of that half.  A half's band union is
        // cut into 32-column slices; sub-warp k takes slices s_lo + k, s_lo + k + 3, ... (3 of the 9
        // slices of an interior config-4 block).  Tiles are read with tcgen05.ld.16x256b: thread
        // t holds rows t1 = t >> 2 and t1 + 8 and columns 8m + 2 t0 + {0, 1} (t0 = t & 3), so a
        // column sum is an in-thread sum over two rows plus a 3-stage butterfly over t1.
        const int qd = warp & 3;
        const int g6 = (warp - 2) >> 2;
        const int half = g6 & 1;
        const int sub = g6 >> 1;
        const int t0 = lane & 3, t1 = lane >> 2;
        const int rbase = qd * 32 + half * 16;
        const int ra = rbase + t1, rb = ra + 8;   // the thread's two rows (inside the block)
        const int et = threadIdx.x - 64;
        const float2 c2v = make_float2(a.c2, a.c2);
        uint32_t tseq = 0;
        for (int gi = g_begin; gi < g_end; ++gi) {
            const Blk b = fblock_of(a, s.wl[gi - g_begin]);
            const int vs = (gi - g_begin) % kNV;
            mbar_wait(&s.v_full[vs], ((gi - g_begin) / kNV) & 1);
            const float* vw = s.vwin + (size_t)vs * (a.maxwin + 128);
            const int wbase = b.q0 * kCR - a.shift;
            const int nch = b.q1 - b.q0 + 1;
            const int nsl = nch * kSlc;
            int ib[2];
            bool act[2];
            float ov[2];
            int lov[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int rr = h ? rb : ra;
                ib[h] = b.i0 + rr;
                const float so = vw[a.maxwin + rr];
                act[h] = ib[h] < a.L_own && so != -INFINITY;
                ov[h] = (!kFirst && act[h]) ? so : 0.f;
                lov[h] = ib[h] - a.w - wbase;               // band start of the row, window coordinates
            }
            const float2 o2a = make_float2(ov[0], ov[0]), o2b = make_float2(ov[1], ov[1]);
            const int wlo = b.i0 + rbase - a.w - wbase;     // union over the half's 16 rows
            const int whi = wlo + 15 + 2 * a.w;
            const int ilo = wlo + 15, ihi = wlo + 2 * a.w;  // intersection
            const int s_lo = wlo < 0 ? 0 : (wlo >> 5);
            const int s_hi = min(nsl - 1, whi >> 5);
            if (!kFirst && !kRecompute && a.w == 128 && nch == 3 && wbase == b.i0 - 128 && a.dbg == 0) {
                // ================= interior block, w = 128: 3 chunks, the half's band union is the 9
                // slices qd .. qd + 8 (window column of row r's band start = r); sub-warp k owns slices
                // qd + k + 3j (j < 3), of which qd and qd + 8 are the only partial (edge) ones.
                // Inactive rows carry o = -inf, so every exponential of theirs is 0 without a branch.
                const float oa = act[0] ? ov[0] : -INFINITY, ob = act[1] ? ov[1] : -INFINITY;
                const float2 oa2 = make_float2(oa, oa), ob2 = make_float2(ob, ob);
                const uint32_t tl = tbase + ((uint32_t)rbase << 16);
                float2 acc_a = make_float2(0.f, 0.f), acc_b = make_float2(0.f, 0.f);
                int waited = -1;
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    const int sl = qd + sub + 3 * j;
                    const int q = sl >> 2;
                    const int ts = (tseq + q) & (NST - 1);
                    if (q > waited) {
                        mbar_wait(&s.t_full[ts], ((tseq + q) / NST) & 1);
                        tc_fence_after();
                        waited = q;
                    }
                    const uint32_t taddr = tl + (uint32_t)(ts * kCR + (sl & 3) * 32);
                    float x[16];
                    tc_ld16x256(taddr, x);
                    const float* vp = vw + sl * 32 + 2 * t0;
                    float2 vv[4];
#pragma unroll
                    for (int mm = 0; mm < 4; ++mm) vv[mm] = *reinterpret_cast<const float2*>(vp + 8 * mm);
                    tc_wait_ld();
                    const bool edge = (j == 0 && sub == 0) || (j == 2 && sub == 2);
                    if (edge) {  // band check: window column - row in [0, 2w]
                        const int cb = sl * 32 + 2 * t0;
#pragma unroll
                        for (int mm = 0; mm < 4; ++mm) {
                            float2 za = __ffma2_rn(make_float2(x[4 * mm], x[4 * mm + 1]), c2v, __fadd2_rn(vv[mm], oa2));
                            float2 zb = __ffma2_rn(make_float2(x[4 * mm + 2], x[4 * mm + 3]), c2v, __fadd2_rn(vv[mm], ob2));
                            const int c = cb + 8 * mm;
                            za.x = (unsigned)(c - ra) <= 256u ? za.x : -INFINITY;
                            za.y = (unsigned)(c + 1 - ra) <= 256u ? za.y : -INFINITY;
                            zb.x = (unsigned)(c - rb) <= 256u ? zb.x : -INFINITY;
                            zb.y = (unsigned)(c + 1 - rb) <= 256u ? zb.y : -INFINITY;
                            x[4 * mm] = ex2(za.x);
                            x[4 * mm + 1] = ex2(za.y);
                            x[4 * mm + 2] = ex2(zb.x);
                            x[4 * mm + 3] = ex2(zb.y);
                            acc_a = __fadd2_rn(acc_a, make_float2(x[4 * mm], x[4 * mm + 1]));
                            acc_b = __fadd2_rn(acc_b, make_float2(x[4 * mm + 2], x[4 * mm + 3]));
                        }
                    } else {
#pragma unroll
                        for (int mm = 0; mm < 4; ++mm) {
                            const float2 za = __ffma2_rn(make_float2(x[4 * mm], x[4 * mm + 1]), c2v, __fadd2_rn(vv[mm], oa2));
                            const float2 zb = __ffma2_rn(make_float2(x[4 * mm + 2], x[4 * mm + 3]), c2v, __fadd2_rn(vv[mm], ob2));
                            x[4 * mm] = ex2(za.x);
                            x[4 * mm + 1] = ex2(za.y);
                            x[4 * mm + 2] = ex2(zb.x);
                            x[4 * mm + 3] = ex2(zb.y);
                            acc_a = __fadd2_rn(acc_a, make_float2(x[4 * mm], x[4 * mm + 1]));
                            acc_b = __fadd2_rn(acc_b, make_float2(x[4 * mm + 2], x[4 * mm + 3]));
                        }
                    }
                    tc_st16x256(taddr, x);
                }
                tc_wait_st();
                float sa = acc_a.x + acc_a.y, sb = acc_b.x + acc_b.y;
                sa += __shfl_xor_sync(0xffffffffu, sa, 1);
                sb += __shfl_xor_sync(0xffffffffu, sb, 1);
                sa += __shfl_xor_sync(0xffffffffu, sa, 2);
                sb += __shfl_xor_sync(0xffffffffu, sb, 2);
                if (t0 == 0) {
                    s.rowp[sub * 128 + ra] = sa;
                    s.rowp[sub * 128 + rb] = sb;
                }
                named_bar(2, NE);
                float ra_sum = 0.f, rb_sum = 0.f;
#pragma unroll
                for (int p = 0; p < kPH; ++p) {
                    ra_sum += s.rowp[p * 128 + ra];
                    rb_sum += s.rowp[p * 128 + rb];
                }
                float wa_ = 0.f, wb_ = 0.f;
                {
                    float ua = 0.f, ub = 0.f;
                    if (act[0]) {
                        ua = ov[0] - lg2(ra_sum);
                        if (!(ra_sum > 0.f) || !isfinite(ua)) { atomicOr(a.err, 4); ua = 0.f; } else wa_ = 1.f / ra_sum;
                    }
                    if (act[1]) {
                        ub = ov[1] - lg2(rb_sum);
                        if (!(rb_sum > 0.f) || !isfinite(ub)) { atomicOr(a.err, 4); ub = 0.f; } else wb_ = 1.f / rb_sum;
                    }
                    if (sub == 0 && t0 == 0) {
                        const size_t uo = (size_t)b.bh * a.Lr_own, po = (size_t)b.bh * a.pad_ld_own + a.pad_off;
                        if (ib[0] < a.L_own) {
                            a.out_own[uo + ib[0]] = ua;
                            a.pad_own[po + ib[0]] = act[0] ? ua : -INFINITY;
                        }
                        if (ib[1] < a.L_own) {
                            a.out_own[uo + ib[1]] = ub;
                            a.pad_own[po + ib[1]] = act[1] ? ub : -INFINITY;
                        }
                    }
                }
                const float2 wa2 = make_float2(wa_, wa_), wb2 = make_float2(wb_, wb_);
                float* cp = s.colp + (size_t)(qd * 2 + half) * a.maxwin;
                const int ccol = 16 * ((lane >> 4) & 1) + 8 * ((lane >> 3) & 1) + 2 * t0 + ((lane >> 2) & 1);
                const bool u4 = (lane & 16) != 0, u3 = (lane & 8) != 0, u2 = (lane & 4) != 0;
                // the half's 3 slices outside its union (0 .. qd-1, qd+9 .. 11): one per sub-warp
                cp[32 * (sub < qd ? sub : sub + 9) + ccol] = 0.f;
                int rel = 0;  // chunks released by this warp so far
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    const int sl = qd + sub + 3 * j;
                    const int q = sl >> 2;
                    for (; rel < q; ++rel) {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&s.t_empty[(tseq + rel) & (NST - 1)]);
                    }
                    const uint32_t taddr = tl + (uint32_t)(((tseq + q) & (NST - 1)) * kCR + (sl & 3) * 32);
                    tc_fence_after();
                    float x[16];
                    tc_ld16x256(taddr, x);
                    tc_wait_ld();
                    float y[8];
#pragma unroll
                    for (int mm = 0; mm < 4; ++mm) {
                        const float2 pr = __ffma2_rn(make_float2(x[4 * mm + 2], x[4 * mm + 3]), wb2,
                                                     __fmul2_rn(make_float2(x[4 * mm], x[4 * mm + 1]), wa2));
                        y[2 * mm] = pr.x;
                        y[2 * mm + 1] = pr.y;
                    }
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const float send = u4 ? y[k] : y[k + 4];
                        const float keep = u4 ? y[k + 4] : y[k];
                        y[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
                    }
#pragma unroll
                    for (int k = 0; k < 2; ++k) {
                        const float send = u3 ? y[k] : y[k + 2];
                        const float keep = u3 ? y[k + 2] : y[k];
                        y[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
                    }
                    const float send = u2 ? y[0] : y[1];
                    const float keep = u2 ? y[1] : y[0];
                    cp[sl * 32 + ccol] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
                }
                for (; rel < 3; ++rel) {
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&s.t_empty[(tseq + rel) & (NST - 1)]);
                }
                tseq += 3;
                __syncwarp();
                if (lane == 0) mbar_arrive(&s.v_empty[vs]);
                named_bar(2, NE);
                float* dst = part_out + ((size_t)b.bh * a.NB + b.blk) * a.maxwin;
                if (et < 3 * kCR) {
                    float sum = 0.f;
#pragma unroll
                    for (int k = 0; k < 8; ++k) sum += s.colp[(size_t)k * a.maxwin + et];
                    dst[et] = sum;
                }
                continue;
            }
            // ---- row pass: e = ex2(s2 + v + o), written back over S (later steps; kRec: not stored,
            // the column pass recomputes -- always so for the cold start, whose online max would
            // leave earlier slices relative to a stale max)
            constexpr bool kRec = kRecompute || kFirst;
            float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
            float Mx[2] = {-INFINITY, -INFINITY};
            int waited = -1;
            for (int sl = s_lo + sub; sl <= s_hi; sl += kPH) {
                const int q = sl >> 2;
                const int ts = (tseq + q) % NST;
                if (q > waited) {
                    mbar_wait(&s.t_full[ts], ((tseq + q) / NST) & 1);
                    tc_fence_after();
                    waited = q;
                }
                const int c0 = sl * 32;
                const bool inner = (c0 >= ilo) && (c0 + 31 <= ihi);
                const uint32_t taddr = tbase + ((uint32_t)rbase << 16) + (uint32_t)(ts * kCR + (sl & 3) * 32);
                float x[16];
                tc_ld16x256(taddr, x);
                tc_wait_ld();
                if (a.dbg & 1) {
                } else if (kFirst) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        float y[8];
                        float m = -INFINITY;
#pragma unroll
                        for (int mm = 0; mm < 4; ++mm)
#pragma unroll
                            for (int c = 0; c < 2; ++c) {
                                const int col = c0 + 8 * mm + 2 * t0 + c;
                                const float z = fmaf(x[4 * mm + 2 * h + c], a.c2, vw[col]);
                                y[2 * mm + c] = (act[h] && (unsigned)(col - lov[h]) <= (unsigned)(2 * a.w)) ? z : -INFINITY;
                                m = fmaxf(m, y[2 * mm + c]);
                            }
                        if (m > Mx[h]) {
                            const float sc = (Mx[h] == -INFINITY) ? 0.f : ex2(Mx[h] - m);
                            acc[h].x *= sc;
                            acc[h].y *= sc;
                            Mx[h] = m;
                        }
                        if (Mx[h] != -INFINITY) {
#pragma unroll
                            for (int k = 0; k < 8; k += 2) {
                                acc[h].x += ex2(y[k] - Mx[h]);
                                acc[h].y += ex2(y[k + 1] - Mx[h]);
                            }
                        }
                    }
                } else {
#pragma unroll
                    for (int mm = 0; mm < 4; ++mm) {
                        const float2 vv = *reinterpret_cast<const float2*>(vw + c0 + 8 * mm + 2 * t0);
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            float2 z = __ffma2_rn(make_float2(x[4 * mm + 2 * h], x[4 * mm + 2 * h + 1]), c2v,
                                                  __fadd2_rn(vv, h ? o2b : o2a));
                            if (!inner || !act[h]) {
                                const int col = c0 + 8 * mm + 2 * t0;
                                z.x = (act[h] && (unsigned)(col - lov[h]) <= (unsigned)(2 * a.w)) ? z.x : -INFINITY;
                                z.y = (act[h] && (unsigned)(col + 1 - lov[h]) <= (unsigned)(2 * a.w)) ? z.y : -INFINITY;
                            }
                            const float2 e = make_float2(ex2(z.x), ex2(z.y));
                            x[4 * mm + 2 * h] = e.x;
                            x[4 * mm + 2 * h + 1] = e.y;
                            acc[h] = __fadd2_rn(acc[h], e);
                        }
                    }
                }
                if (!kRec) tc_st16x256(taddr, x);
            }
            if (!kRec) tc_wait_st();
            // ---- row sums: over t0 (4 threads share a row), then over the 3 sub-warps in fixed order
            float rs[2], rm[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                float sm = acc[h].x + acc[h].y, M = Mx[h];
#pragma unroll
                for (int o = 1; o <= 2; o <<= 1) {
                    const float s2 = __shfl_xor_sync(0xffffffffu, sm, o);
                    if (kFirst) {
                        const float M2 = __shfl_xor_sync(0xffffffffu, M, o);
                        const float Mn = fmaxf(M, M2);
                        sm = (M == -INFINITY ? 0.f : sm * ex2(M - Mn)) + (M2 == -INFINITY ? 0.f : s2 * ex2(M2 - Mn));
                        M = Mn;
                    } else {
                        sm += s2;
                    }
                }
                rs[h] = sm;
                rm[h] = M;
            }
            if (t0 == 0) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int rr = h ? rb : ra;
                    s.rowp[sub * 128 + rr] = rs[h];
                    if (kFirst) s.rowp[(kPH + sub) * 128 + rr] = rm[h];
                }
            }
            named_bar(2, NE);
            float wgt[2], Mall[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int rr = h ? rb : ra;
                float rsum = 0.f, Ma = -INFINITY;
                if (kFirst) {
#pragma unroll
                    for (int p = 0; p < kPH; ++p) Ma = fmaxf(Ma, s.rowp[(kPH + p) * 128 + rr]);
#pragma unroll
                    for (int p = 0; p < kPH; ++p) {
                        const float Mp = s.rowp[(kPH + p) * 128 + rr];
                        rsum += (Mp == -INFINITY) ? 0.f : s.rowp[p * 128 + rr] * ex2(Mp - Ma);
                    }
                } else {
#pragma unroll
                    for (int p = 0; p < kPH; ++p) rsum += s.rowp[p * 128 + rr];
                }
                float u = 0.f;
                wgt[h] = 0.f;
                Mall[h] = Ma;
                if (act[h]) {
                    u = kFirst ? (-Ma - lg2(rsum)) : (ov[h] - lg2(rsum));
                    if (!(rsum > 0.f) || !isfinite(u)) {
                        atomicOr(a.err, 4);
                        u = 0.f;
                    } else {
                        wgt[h] = 1.f / rsum;
                    }
                }
                if (sub == 0 && t0 == 0 && ib[h] < a.L_own) {
                    a.out_own[(size_t)b.bh * a.Lr_own + ib[h]] = u;
                    a.pad_own[(size_t)b.bh * a.pad_ld_own + a.pad_off + ib[h]] = act[h] ? u : -INFINITY;
                }
            }
            // ---- column pass: c_Ij = sum_i e_ij / r_i over the half's 16 rows, per column.  Every
            // slice of the window is written by exactly one sub-warp of the half (zeros outside the
            // union); a chunk's TMEM slot is released by each warp once it is done with that chunk.
            const float2 wa = make_float2(wgt[0], wgt[0]), wb = make_float2(wgt[1], wgt[1]);
            float* cp = s.colp + (size_t)(qd * 2 + half) * a.maxwin;
            const int ph = (((s_lo + sub) % kPH) + kPH) % kPH;
            const int ccol = 16 * ((lane >> 4) & 1) + 8 * ((lane >> 3) & 1) + 2 * t0 + ((lane >> 2) & 1);
            for (int q = 0; q < nch; ++q) {
                const int ts = (tseq + q) % NST;
#pragma unroll
                for (int j = 0; j < kSlc; ++j) {
                    const int sl = q * kSlc + j;
                    if (sl % kPH != ph) continue;
                    const int c0 = sl * 32;
                    float val = 0.f;
                    if (sl >= s_lo && sl <= s_hi) {
                        tc_fence_after();
                        const uint32_t taddr = tbase + ((uint32_t)rbase << 16) + (uint32_t)(ts * kCR + j * 32);
                        float x[16];
                        tc_ld16x256(taddr, x);
                        tc_wait_ld();
                        if (kRec) {
#pragma unroll
                            for (int mm = 0; mm < 4; ++mm)
#pragma unroll
                                for (int h = 0; h < 2; ++h)
#pragma unroll
                                    for (int c = 0; c < 2; ++c) {
                                        const int col = c0 + 8 * mm + 2 * t0 + c;
                                        float z = fmaf(x[4 * mm + 2 * h + c], a.c2, vw[col]) + (kFirst ? -Mall[h] : ov[h]);
                                        z = (act[h] && (unsigned)(col - lov[h]) <= (unsigned)(2 * a.w)) ? z : -INFINITY;
                                        x[4 * mm + 2 * h + c] = ex2(z);
                                    }
                        }
                        float y[8];
#pragma unroll
                        for (int mm = 0; mm < 4; ++mm) {
                            const float2 p = __ffma2_rn(make_float2(x[4 * mm + 2], x[4 * mm + 3]), wb,
                                                        __fmul2_rn(make_float2(x[4 * mm], x[4 * mm + 1]), wa));
                            y[2 * mm] = p.x;
                            y[2 * mm + 1] = p.y;
                        }
                        if (a.dbg & 4) {
                            val = y[0];
                        } else {
                            const bool u4 = (lane & 16) != 0, u3 = (lane & 8) != 0, u2 = (lane & 4) != 0;
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                const float send = u4 ? y[k] : y[k + 4];
                                const float keep = u4 ? y[k + 4] : y[k];
                                y[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
                            }
#pragma unroll
                            for (int k = 0; k < 2; ++k) {
                                const float send = u3 ? y[k] : y[k + 2];
                                const float keep = u3 ? y[k + 2] : y[k];
                                y[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
                            }
                            const float send = u2 ? y[0] : y[1];
                            const float keep = u2 ? y[1] : y[0];
                            val = keep + __shfl_xor_sync(0xffffffffu, send, 4);
                        }
                    }
                    cp[c0 + ccol] = val;
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&s.t_empty[ts]);
            }
            tseq += nch;
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.v_empty[vs]);  // window duals no longer needed
            named_bar(2, NE);
            // ---- combine the 8 half-quadrant partials in fixed order; store the block's column partials
            float* dst = part_out + ((size_t)b.bh * a.NB + b.blk) * a.maxwin;
            for (int c = et; c < nch * kCR; c += NE) {
                float sum = 0.f;
#pragma unroll
                for (int k = 0; k < 8; ++k) sum += s.colp[(size_t)k * a.maxwin + c];
                dst[c] = sum;
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
// v^t_j = v^{t-1}_j - lg2( sum_{I : rows of I meet band(j)} c_Ij ), ascending I.
// pad_v in place (-inf stays on inactive / guard entries); v_out (standard layout).
// ---------------------------------------------------------------------------
__global__ void k_vmerge(const float* __restrict__ part, float* __restrict__ pad_v, float* __restrict__ v_out,
                         int BH, int H, int Lq, int Lk, int Lrk, int NB, int maxwin, int w, int CR, int shift,
                         int Lp_other, int pad_ld, int pad_off, const uint8_t* __restrict__ col_mask,
                         int* __restrict__ err) {
    const long n = (long)BH * Lk;
    for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (long)gridDim.x * blockDim.x) {
        const int bh = (int)(t / Lk), j = (int)(t % Lk);
        float* pv = pad_v + (size_t)bh * pad_ld + pad_off + j;
        const float vold = *pv;
        float v = 0.f;
        if (vold != -INFINITY) {  // active column (the padded buffer carries the mask)
            const int I0 = max(0, j - w) / 128, I1 = min(Lq - 1, j + w) / 128;
            const int nq = Lp_other / CR;
            float sum = 0.f;
            for (int I = I0; I <= I1; ++I) {
                const int q0 = max(0, (I * 128 - w + shift) / CR);
                (void)nq;
                const int wc = j - (q0 * CR - shift);
                sum += part[((size_t)bh * NB + I) * maxwin + wc];
            }
            v = vold - lg2(sum);
            if (!(sum > 0.f) || !isfinite(v)) {
                atomicOr(err, 8);
                v = 0.f;
            }
            *pv = v;
        }
        if (v_out) v_out[(size_t)bh * Lrk + j] = v;
    }
}

static thread_local long long g_fs_launches = 0;
long long fstep16_launch_count(bool reset) {
    const long long c = g_fs_launches;
    if (reset) g_fs_launches = 0;
    return c;
}

size_t fstep16_smem_bytes(const PhaseArgs& a) {
    const int nst = 512 / a.CR;
    return (size_t)a.NA * 128 * a.row_bytes + (size_t)a.NSK * a.CR * a.row_bytes +
           (size_t)(kNV * (a.maxwin + 128) + 2 * kPH * 128 + 8 * a.maxwin) * 4 +
           (size_t)(2 * kNV + 2 * a.NA + 2 * a.NSK + 2 * nst) * 8 + 16 + (size_t)a.wl_cap * 4;
}

template <bool kFirst, bool kRec>
static cudaError_t launch_fstep16_t(const PhaseArgs& a, float* part, int grid, cudaStream_t s) {
    const size_t smem = fstep16_smem_bytes(a);
    auto k = k_fstep16<kFirst, kRec>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<grid, 64 + 32 * kEW, smem, s>>>(a, part);
    ++g_fs_launches;
    return cudaGetLastError();
}

cudaError_t launch_fstep16(const PhaseArgs& a, float* part, bool first, int grid, cudaStream_t s) {
    static const bool rec = getenv("ST_FSTEP_RECOMPUTE") != nullptr;
    if (a.npl != 1 || a.CR != 128 || a.dustbin) return cudaErrorNotSupported;
    if (first) return rec ? launch_fstep16_t<true, true>(a, part, grid, s) : launch_fstep16_t<true, false>(a, part, grid, s);
    return rec ? launch_fstep16_t<false, true>(a, part, grid, s) : launch_fstep16_t<false, false>(a, part, grid, s);
}

cudaError_t launch_vmerge(const float* part, float* pad_v, float* v_out, int BH, int H, int Lq, int Lk, int Lrk, int NB,
                          int maxwin, int w, int CR, int shift, int Lp_other, int pad_ld, int pad_off,
                          const uint8_t* col_mask, int* err, cudaStream_t s) {
    const long n = (long)BH * Lk;
    const int nb = (int)std::min<long>((n + 255) / 256, 148L * 16);
    k_vmerge<<<nb, 256, 0, s>>>(part, pad_v, v_out, BH, H, Lq, Lk, Lrk, NB, maxwin, w, CR, shift, Lp_other, pad_ld,
                                pad_off, col_mask, err);
    ++g_fs_launches;
    return cudaGetLastError();
}

}  // namespace st
