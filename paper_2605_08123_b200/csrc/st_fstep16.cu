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
//   warps 2..9   epilogue: one warp per 16-lane half of a TMEM lane quadrant; it owns
//            whole rows (16 of them), so row sums need no cross-warp combine and the
//            column pass follows the row pass without a CTA barrier
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "st_common.cuh"
#include "st_phase.cuh"
#include "st_sm100.cuh"

namespace st {

using namespace sm100;

namespace {

constexpr int kNV = 3;     // dual-window ring slots
constexpr int kEW = 16;    // epilogue warps: two per 16-lane half of a TMEM lane quadrant
constexpr int kSlc = 4;    // 32-column slices per 128-column chunk
constexpr int kG = 3;      // tiles per epilogue round (shared TMEM-load wait, interleaved math)

struct FSmem {
    uint8_t* A;       // [NA][128 * row_bytes]
    uint8_t* K;       // [NSK][CR * row_bytes]
    float* vwin;      // [kNV][maxwin + 128]
    float* colp;      // [2][8][maxwin]: column partials per 16-lane half quadrant, by block parity
    float* rowx;      // [8][2][16]: row-sum exchange of the two warps of a half quadrant
    uint64_t* v_full;
    uint64_t* v_empty;
    uint64_t* a_full;
    uint64_t* a_empty;
    uint64_t* k_full;
    uint64_t* k_empty;
    uint64_t* t_full;
    uint64_t* t_empty;
    uint32_t* tmem_base;
    int4* bd;         // [wl_cap] block descriptors of this CTA's work-list slice: (bh, blk, q0, q1)
};

__device__ __forceinline__ FSmem fcarve(uint8_t* base, const PhaseArgs& a, int nst) {
    FSmem s;
    const size_t blk = (size_t)128 * a.row_bytes, chk = (size_t)a.CR * a.row_bytes;
    s.A = base;
    s.K = s.A + (size_t)a.NA * blk;
    s.vwin = (float*)(s.K + (size_t)a.NSK * chk);
    s.colp = s.vwin + kNV * (a.maxwin + 128);
    s.rowx = s.colp + 2 * 8 * a.maxwin;
    uint64_t* bars = (uint64_t*)(s.rowx + 8 * 2 * 16);
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
    s.bd = (int4*)(s.tmem_base + 4);
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

__device__ __forceinline__ Blk bdesc(int4 d) {
    Blk b;
    b.bh = d.x;
    b.blk = d.y;
    b.i0 = d.y * 128;
    b.q0 = d.z;
    b.q1 = d.w;
    return b;
}

__device__ __forceinline__ unsigned long long fgtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// development timeline (ST_TRACE_PHASE=<step>): trace[cta * 64 + slot] for CTAs 0..3
#ifdef ST_FSTEP_TRACE
#define FS_TRACE(slot) FS_TRACE_ON(slot)
#else
#define FS_TRACE(slot) \
    do {               \
    } while (0)
#endif
#define FS_TRACE_ON(slot)                                                                                 \
    do {                                                                                               \
        if (a.trace && blockIdx.x < 4 && (slot) < 64) a.trace[blockIdx.x * 64 + (slot)] = fgtimer(); \
    } while (0)

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

template <bool kFirst, bool kRecompute, bool kTma>
__global__ void __launch_bounds__(64 + 32 * kEW, 1) k_fstep16(const __grid_constant__ PhaseArgs a, float* __restrict__ part_out) {
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
    for (int k = threadIdx.x; k < g_end - g_begin; k += blockDim.x) {
        const int g = a.work ? a.work[g_begin + k] : g_begin + k;
        const Blk b = fblock_of(a, g);
        s.bd[k] = make_int4(b.bh, b.blk, b.q0, b.q1);
    }
    if (threadIdx.x == 0 && (int)((long long)n * (blockIdx.x + 1) / gridDim.x) - g_begin > a.wl_cap)
        atomicOr(a.err, 16);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *s.tmem_base;
    if (threadIdx.x == 0) FS_TRACE(57);

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        int last_bh = -1, last_q = -1;
        uint32_t kseq = 0;
        for (int gi = g_begin; gi < g_end; ++gi) {
            const Blk b = bdesc(s.bd[gi - g_begin]);
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
                if constexpr (kTma) {  // raw rows i0 .. i0 + 127 as [d half][128 rows][128 B] swizzled boxes
                    for (int kb = 0; kb < a.row_bytes / 128; ++kb)  // one 128-row box per d half
                        tma_load_3d(s.A + (size_t)ab * blk_bytes + kb * 16384, &a.tmA, kb * 64, b.i0, b.bh, &s.a_full[ab]);
                } else {
                    bulk_g2s(s.A + (size_t)ab * blk_bytes, a.A_pack[0] + ((size_t)b.bh * a.Lp_own + b.i0 + a.shift) * a.row_bytes,
                             blk_bytes, &s.a_full[ab]);
                }
            }
            __syncwarp();
            const int qstart = (b.bh == last_bh) ? max(b.q0, last_q + 1) : b.q0;
            for (int q = qstart; q <= b.q1; ++q) {
                const int sl = kseq % a.NSK;
                const uint32_t kn = kseq / a.NSK;
                mbar_wait(&s.k_empty[sl], (kn & 1) ^ 1);
                if (elect_one()) {
                    mbar_arrive_expect_tx(&s.k_full[sl], chk_bytes);
                    if constexpr (kTma) {  // chunk q = raw rows q * 128 - shift .. (out-of-range rows arrive as zeros)
                        for (int kb = 0; kb < a.row_bytes / 128; ++kb)
                            tma_load_3d(s.K + (size_t)sl * chk_bytes + kb * 16384, &a.tmB, kb * 64, q * kCR - a.shift, b.bh,
                                        &s.k_full[sl]);
                    } else {
                        bulk_g2s(s.K + (size_t)sl * chk_bytes,
                                 a.B_pack[0] + ((size_t)b.bh * a.Lp_other + (size_t)q * kCR) * a.row_bytes, chk_bytes,
                                 &s.k_full[sl]);
                    }
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
            const Blk b = bdesc(s.bd[gi - g_begin]);
            const int ab = (gi - g_begin) % a.NA;
            const uint32_t an = (gi - g_begin) / a.NA;
            mbar_wait(&s.a_full[ab], an & 1);
            tc_fence_after();
            const uint32_t as_ = smem_u32(s.A + (size_t)ab * blk_bytes);
            const uint64_t ad0 = make_desc(as_, 128, sbo);
            const uint64_t ad_sw = make_desc_sw128(as_, 16, 1024);
            const bool same = have && b.bh == last_bh;
            const int new_start = same ? max(b.q0, last_q + 1) : b.q0;
            const uint32_t next_seq = have ? last_seq + 1 : 0;
            // chunks are issued as soon as their TMEM slot is free; a chunk whose successor's slot
            // (and K chunk) are ready too is paired with it (independent accumulators hide the
            // dependent-MMA latency of a lone chain)
            auto seq_of = [&](int q) {
                return (same && q <= last_q) ? last_seq - (uint32_t)(last_q - q) : next_seq + (uint32_t)(q - new_start);
            };
            if (lane == 0 && gi - g_begin < 8) FS_TRACE(1 + (gi - g_begin));
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
                uint64_t bd[2], bd_sw[2];
                uint32_t dt[2], bs_[2];
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const uint32_t sq = seq_of(q + c);
                    bs_[c] = smem_u32(s.K + (size_t)(sq % a.NSK) * chk_bytes);
                    bd[c] = make_desc(bs_[c], 128, sbo);
                    bd_sw[c] = make_desc_sw128(bs_[c], 16, 1024);
                    dt[c] = tbase + (uint32_t)(((tseq + c) % NST) * kCR);
                }
                tc_fence_after();
                if (elect_one()) {
                    for (int kk = 0; kk < ksteps; ++kk) {
#pragma unroll
                        for (int c = 0; c < 2; ++c)
                            if (c < ng && (kk == 0 || !(a.dbg & 2))) {
                                if constexpr (kTma) {  // 128B-swizzled tiles: d half kk / 4, 32 bytes per K step inside the row
                                    const uint64_t ko = (uint64_t)((kk >> 2) * 1024 + (kk & 3) * 2);  // 16-byte units
                                    mma_bf16(dt[c], ad_sw + ko, bd_sw[c] + ko, idesc, kk > 0);
                                } else {
                                    mma_bf16(dt[c], ad0 + (uint64_t)(kk * 16), bd[c] + (uint64_t)(kk * 16), idesc, kk > 0);
                                }
                            }
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
            if (lane == 0 && gi - g_begin < 8) FS_TRACE(9 + (gi - g_begin));
            if (b.q1 >= new_start) last_seq = next_seq + (uint32_t)(b.q1 - new_start);
            if (!same) last_q = -1;
            last_q = max(last_q, b.q1);
            last_bh = b.bh;
            have = true;
            uint32_t keep_from = last_seq + 1;
            if (gi + 1 < g_end) {
                const Blk nb = bdesc(s.bd[gi + 1 - g_begin]);
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
        // warp w (2..17): lane quadrant qd = w % 4, g = (w - 2) / 4: half hf = g & 1 -> rows rbase ..
        // rbase + 15, part pt = g >> 1 (the two warps of a half split its slices).  Tiles of 16 rows x
        // 32 columns are read with tcgen05.ld.16x256b: thread t holds rows rA = rbase + t1 and
        // rB = rA + 8 and columns 8m + 2 t0 + {0, 1} (t0 = t & 3, t1 = t >> 2).
        const int qd = warp & 3, hf = ((warp - 2) >> 2) & 1, pt = (warp - 2) >> 3;
        const int hq = qd * 2 + hf;  // half-quadrant id (pair barrier 3 + hq)
        const int t0 = lane & 3, t1 = lane >> 2;
        const int rbase = qd * 32 + hf * 16;
        const int rA = rbase + t1, rB = rA + 8;
        const int et = threadIdx.x - 64;
        const uint32_t tl = tbase + ((uint32_t)rbase << 16);
        const int ccol = 16 * ((lane >> 4) & 1) + 8 * ((lane >> 3) & 1) + 2 * t0 + ((lane >> 2) & 1);
        const bool u4 = (lane & 16) != 0, u3 = (lane & 8) != 0, u2 = (lane & 4) != 0;
        const float2 c2v = make_float2(a.c2, a.c2);
        const int bandw = 2 * a.w;
        constexpr bool kRec = kRecompute || kFirst;  // cold start: e recomputed in the column pass
        uint32_t tseq = 0;
        for (int gi = g_begin; gi < g_end; ++gi) {
            const Blk b = bdesc(s.bd[gi - g_begin]);
            const int par = (gi - g_begin) & 1;
            const int vs = (gi - g_begin) % kNV;
            const int wbase = b.q0 * kCR - a.shift;
            const int nch = b.q1 - b.q0 + 1;
            const int nsl = nch * kSlc;
            const int iA = b.i0 + rA, iB = iA + 8;
            const int loA = iA - a.w - wbase, loB = loA + 8;  // band start of each row, window coordinates
            const int wlo = b.i0 + rbase - a.w - wbase;       // union over the warp's 16 rows
            const int s_lo = wlo < 0 ? 0 : (wlo >> 5);
            const int s_hi = min(nsl - 1, (wlo + 15 + bandw) >> 5);
            // tiles whose 32 columns lie in every row's band need no mask
            const int in_lo = (wlo + 15 + 31) >> 5, in_hi = (wlo + bandw - 31) >> 5;  // ceil / floor (arithmetic shifts)
            const bool trc = warp == 2 && lane == 0 && gi - g_begin < 8;
            if (trc) FS_TRACE(17 + (gi - g_begin));
            mbar_wait(&s.v_full[vs], ((gi - g_begin) / kNV) & 1);
            if (trc) FS_TRACE(25 + (gi - g_begin));
            const float* vw = s.vwin + (size_t)vs * (a.maxwin + 128);
            const float soA = vw[a.maxwin + rA], soB = vw[a.maxwin + rB];
            const bool actA = iA < a.L_own && soA != -INFINITY, actB = iB < a.L_own && soB != -INFINITY;
            // offsets; inactive rows get -inf so every exponential of theirs is 0 without a branch
            const float oA = actA ? (kFirst ? 0.f : soA) : -INFINITY, oB = actB ? (kFirst ? 0.f : soB) : -INFINITY;
            const float2 oA2 = make_float2(oA, oA), oB2 = make_float2(oB, oB);
            if (!kFirst && !kRecompute && a.w == 128 && nch == 3 && wbase == b.i0 - 128 && a.dbg == 0) {
                // ============ interior block, w = 128: the half's union is the 9 slices qd .. qd + 8 (row r's
                // band starts at window column r); part 0 owns slices qd .. qd + 3, part 1 qd + 4 .. qd + 8
                // (both warps of a half share one SMSP, so the 4 : 5 split costs no MUFU throughput); only
                // qd and qd + 8 are partial.  TMEM is read ONCE for 8 of the 9 tiles: their exponentials
                // stay in registers for the column pass, and chunk slots are released as soon as their
                // tiles are loaded.  Part 1's last tile goes back to TMEM (register budget of 18 warps).
                auto fast = [&](auto PTc) {
                constexpr int P = decltype(PTc)::value;
                constexpr int j0 = P ? 4 : 0;
                float e[4][16];
                float2 accA = make_float2(0.f, 0.f), accB = make_float2(0.f, 0.f);
                // part 0: rounds {0,1}, {2,3}; part 1: {4,5,8}, {6,7} -- part 1's last tile (slice qd + 8) is
                // exponentiated first and goes back to TMEM at once, so at most 4 tiles (64 registers) stay
                // live.  Round 1's TMEM loads are issued before round 0's exponentials (one wait::ld each).
                float x8[16];
                // tile k of the warp (j = j0 + k; k = 4 is part 1's TMEM-resident slice qd + 8)
                auto tile_addr = [&](int k) {
                    const int sl = qd + j0 + k;
                    return tl + (uint32_t)(((tseq + (sl >> 2)) & (NST - 1)) * kCR + (sl & 3) * 32);
                };
                auto exp_tile = [&](float (&ej)[16], int k) {
                    const int j = j0 + k;
                    const int cb = (qd + j) * 32 + 2 * t0;
                    const bool edge = (j == 0) || (j == 8);
#pragma unroll
                    for (int mm = 0; mm < 4; ++mm) {
                        const float2 vv = *reinterpret_cast<const float2*>(vw + cb + 8 * mm);
                        float2 za = __ffma2_rn(make_float2(ej[4 * mm], ej[4 * mm + 1]), c2v, __fadd2_rn(vv, oA2));
                        float2 zb = __ffma2_rn(make_float2(ej[4 * mm + 2], ej[4 * mm + 3]), c2v, __fadd2_rn(vv, oB2));
                        if (edge) {  // partial slices: band check window column - row in [0, 2w]
                            const int c = cb + 8 * mm;
                            za.x = (unsigned)(c - loA) <= 256u ? za.x : -INFINITY;
                            za.y = (unsigned)(c + 1 - loA) <= 256u ? za.y : -INFINITY;
                            zb.x = (unsigned)(c - loB) <= 256u ? zb.x : -INFINITY;
                            zb.y = (unsigned)(c + 1 - loB) <= 256u ? zb.y : -INFINITY;
                        }
                        const float2 ea = make_float2(ex2(za.x), ex2(za.y));
                        const float2 eb = make_float2(ex2(zb.x), ex2(zb.y));
                        ej[4 * mm] = ea.x;
                        ej[4 * mm + 1] = ea.y;
                        ej[4 * mm + 2] = eb.x;
                        ej[4 * mm + 3] = eb.y;
                        accA = __fadd2_rn(accA, ea);
                        accB = __fadd2_rn(accB, eb);
                    }
                };
                // part 1 first exponentiates its TMEM-resident tile 8 (slice qd + 8, chunk 2) and stores it
                // back before any register tile is loaded, so at most 4 tiles (64 registers) are ever live
                if (P) {
                    for (int q = 0; q <= 2; ++q) mbar_wait(&s.t_full[(tseq + q) & (NST - 1)], ((tseq + q) / NST) & 1);
                    tc_fence_after();
                    tc_ld16x256(tile_addr(4), x8);
                    tc_wait_ld();
                    exp_tile(x8, 4);
                    tc_st16x256(tile_addr(4), x8);
                    tc_wait_st();
                }
                const int qlast0 = (qd + j0 + 1) >> 2;  // last chunk of round 0 (tiles 0, 1)
                const int qlast1 = (qd + j0 + 3) >> 2;
                if (!P)
                    for (int q = 0; q <= qlast0; ++q) mbar_wait(&s.t_full[(tseq + q) & (NST - 1)], ((tseq + q) / NST) & 1);
                tc_fence_after();
                if (warp == 2 && lane == 0 && gi - g_begin == 4) FS_TRACE(58);
                tc_ld16x256(tile_addr(0), e[0]);
                tc_ld16x256(tile_addr(1), e[1]);
                tc_wait_ld();
                if (warp == 2 && lane == 0 && gi - g_begin == 4) FS_TRACE(59);
                if (!P)
                    for (int q = qlast0 + 1; q <= qlast1; ++q) mbar_wait(&s.t_full[(tseq + q) & (NST - 1)], ((tseq + q) / NST) & 1);
                tc_fence_after();
                tc_ld16x256(tile_addr(2), e[2]);
                tc_ld16x256(tile_addr(3), e[3]);
                exp_tile(e[0], 0);
                exp_tile(e[1], 1);
                tc_wait_ld();
                if (warp == 2 && lane == 0 && gi - g_begin == 4) FS_TRACE(60);
                // every tile loaded: release the chunks (part 1 keeps chunk 2 for its TMEM-resident tile)
                tc_fence_before();
                __syncwarp();
                if (lane == 0)
                    for (int q = 0; q < (P ? 2 : 3); ++q) mbar_arrive(&s.t_empty[(tseq + q) & (NST - 1)]);
                exp_tile(e[2], 2);
                exp_tile(e[3], 3);
                // ---- row sums: over t0, then the two parts of the half in fixed order (part 0 + part 1)
                float sA = accA.x + accA.y, sB = accB.x + accB.y;
                sA += __shfl_xor_sync(0xffffffffu, sA, 1);
                sB += __shfl_xor_sync(0xffffffffu, sB, 1);
                sA += __shfl_xor_sync(0xffffffffu, sA, 2);
                sB += __shfl_xor_sync(0xffffffffu, sB, 2);
                float* rx = s.rowx + hq * 32;
                if (t0 == 0) {
                    rx[P * 16 + t1] = sA;
                    rx[P * 16 + t1 + 8] = sB;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&s.v_empty[vs]);  // window duals no longer needed
                named_bar(3 + hq, 64);
                sA = rx[t1] + rx[16 + t1];
                sB = rx[t1 + 8] + rx[16 + t1 + 8];
                float wA = 0.f, wB = 0.f, uA = 0.f, uB = 0.f;
                if (actA) {
                    uA = oA - lg2(sA);
                    if (!(sA > 0.f) || !isfinite(uA)) { atomicOr(a.err, 4); uA = 0.f; } else wA = 1.f / sA;
                }
                if (actB) {
                    uB = oB - lg2(sB);
                    if (!(sB > 0.f) || !isfinite(uB)) { atomicOr(a.err, 4); uB = 0.f; } else wB = 1.f / sB;
                }
                if (P == 0 && t0 == 0) {
                    const size_t uo = (size_t)b.bh * a.Lr_own, po = (size_t)b.bh * a.pad_ld_own + a.pad_off;
                    if (iA < a.L_own) {
                        a.out_own[uo + iA] = uA;
                        a.pad_own[po + iA] = actA ? uA : -INFINITY;
                    }
                    if (iB < a.L_own) {
                        a.out_own[uo + iB] = uB;
                        a.pad_own[po + iB] = actB ? uB : -INFINITY;
                    }
                }
                if (trc) FS_TRACE(33 + (gi - g_begin));
                // ---- column pass from registers (part 1's slice qd + 8 re-read from TMEM last)
                const float2 wA2 = make_float2(wA, wA), wB2 = make_float2(wB, wB);
                float* cp = s.colp + ((size_t)par * 8 + (size_t)hq) * a.maxwin;
                if (P == 0) {
                    for (int sl = 0; sl < qd; ++sl) cp[sl * 32 + ccol] = 0.f;
                    for (int sl = qd + 9; sl < 12; ++sl) cp[sl * 32 + ccol] = 0.f;
                }
                auto col_tile = [&](const float (&ej)[16], int k) {
                    float y[8];
#pragma unroll
                    for (int mm = 0; mm < 4; ++mm) {
                        const float2 pr = __ffma2_rn(make_float2(ej[4 * mm + 2], ej[4 * mm + 3]), wB2,
                                                     __fmul2_rn(make_float2(ej[4 * mm], ej[4 * mm + 1]), wA2));
                        y[2 * mm] = pr.x;
                        y[2 * mm + 1] = pr.y;
                    }
#pragma unroll
                    for (int i2 = 0; i2 < 4; ++i2) {
                        const float send = u4 ? y[i2] : y[i2 + 4];
                        const float keep = u4 ? y[i2 + 4] : y[i2];
                        y[i2] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
                    }
#pragma unroll
                    for (int i2 = 0; i2 < 2; ++i2) {
                        const float send = u3 ? y[i2] : y[i2 + 2];
                        const float keep = u3 ? y[i2 + 2] : y[i2];
                        y[i2] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
                    }
                    const float send = u2 ? y[0] : y[1];
                    const float keep = u2 ? y[1] : y[0];
                    cp[(qd + j0 + k) * 32 + ccol] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
                };
                if (P) {  // start the TMEM re-read of slice qd + 8 first; it lands while tiles 0..3 reduce
                    tc_fence_after();
                    tc_ld16x256(tile_addr(4), x8);
                }
                col_tile(e[0], 0);
                col_tile(e[1], 1);
                col_tile(e[2], 2);
                col_tile(e[3], 3);
                if (P) {
                    tc_wait_ld();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&s.t_empty[(tseq + 2) & (NST - 1)]);
                    col_tile(x8, 4);
                }
                };
                if (pt) fast(std::integral_constant<int, 1>{});
                else fast(std::integral_constant<int, 0>{});
                tseq += 3;
                if (trc) FS_TRACE(41 + (gi - g_begin));
                named_bar(2, NE);
                if (trc) FS_TRACE(49 + (gi - g_begin));
                const float* cb8 = s.colp + (size_t)par * 8 * a.maxwin;
                float* dst = part_out + ((size_t)b.bh * a.NB + b.blk) * a.maxwin;
                if (et < 3 * kCR) {
                    float sum = 0.f;
#pragma unroll
                    for (int k = 0; k < 8; ++k) sum += cb8[(size_t)k * a.maxwin + et];
                    dst[et] = sum;
                }
                continue;
            }
            if (pt == 1) {
                // generic blocks run on the first warp of each pair; the second only keeps the barrier
                // and slot protocols (one arrival per chunk and per window) and joins the combine
                __syncwarp();
                if (lane == 0) {
                    for (int q = 0; q < nch; ++q) mbar_arrive(&s.t_empty[(tseq + q) & (NST - 1)]);
                    mbar_arrive(&s.v_empty[vs]);
                }
                tseq += nch;
                named_bar(2, NE);
                const float* cb8 = s.colp + (size_t)par * 8 * a.maxwin;
                float* dst = part_out + ((size_t)b.bh * a.NB + b.blk) * a.maxwin;
                for (int c = et; c < nch * kCR; c += NE) {
                    float sum = 0.f;
#pragma unroll
                    for (int k = 0; k < 8; ++k) sum += cb8[(size_t)k * a.maxwin + c];
                    dst[c] = sum;
                }
                continue;
            }
            // ---- row pass: e = ex2(s2 + v + o) over the warp's union slices, written back over S
            float2 accA = make_float2(0.f, 0.f), accB = make_float2(0.f, 0.f);
            float MA = -INFINITY, MB = -INFINITY;  // cold start: running row maxima
            int waited = -1;
            for (int g0 = s_lo; g0 <= s_hi; g0 += kG) {
                // kG tiles per round: their TMEM loads share one wait, their exponentials interleave
                const int gl = min(s_hi, g0 + kG - 1);
                const int qh = gl >> 2;
                if (qh > waited) {
                    for (int q = waited + 1; q <= qh; ++q) mbar_wait(&s.t_full[(tseq + q) & (NST - 1)], ((tseq + q) / NST) & 1);
                    tc_fence_after();
                    waited = qh;
                }
                float x[kG][16];
                float2 vv[kG][4];
#pragma unroll
                for (int k = 0; k < kG; ++k) {
                    const int sl = min(g0 + k, gl);
                    tc_ld16x256(tl + (uint32_t)(((tseq + (sl >> 2)) & (NST - 1)) * kCR + (sl & 3) * 32), x[k]);
#pragma unroll
                    for (int mm = 0; mm < 4; ++mm)
                        vv[k][mm] = *reinterpret_cast<const float2*>(vw + sl * 32 + 2 * t0 + 8 * mm);
                }
                tc_wait_ld();
#pragma unroll
                for (int k = 0; k < kG; ++k) {
                    const int sl = g0 + k;
                    if (sl > gl) break;
                    const int cb = sl * 32 + 2 * t0;
                    if (kFirst) {
                        float mA = -INFINITY, mB = -INFINITY;
#pragma unroll
                        for (int mm = 0; mm < 4; ++mm) {
                            const int c = cb + 8 * mm;
                            float2 za = __ffma2_rn(make_float2(x[k][4 * mm], x[k][4 * mm + 1]), c2v, vv[k][mm]);
                            float2 zb = __ffma2_rn(make_float2(x[k][4 * mm + 2], x[k][4 * mm + 3]), c2v, vv[k][mm]);
                            za.x = (actA && (unsigned)(c - loA) <= (unsigned)bandw) ? za.x : -INFINITY;
                            za.y = (actA && (unsigned)(c + 1 - loA) <= (unsigned)bandw) ? za.y : -INFINITY;
                            zb.x = (actB && (unsigned)(c - loB) <= (unsigned)bandw) ? zb.x : -INFINITY;
                            zb.y = (actB && (unsigned)(c + 1 - loB) <= (unsigned)bandw) ? zb.y : -INFINITY;
                            x[k][4 * mm] = za.x;
                            x[k][4 * mm + 1] = za.y;
                            x[k][4 * mm + 2] = zb.x;
                            x[k][4 * mm + 3] = zb.y;
                            mA = fmaxf(mA, fmaxf(za.x, za.y));
                            mB = fmaxf(mB, fmaxf(zb.x, zb.y));
                        }
                        if (mA > MA) {
                            const float sc = (MA == -INFINITY) ? 0.f : ex2(MA - mA);
                            accA.x *= sc;
                            accA.y *= sc;
                            MA = mA;
                        }
                        if (mB > MB) {
                            const float sc = (MB == -INFINITY) ? 0.f : ex2(MB - mB);
                            accB.x *= sc;
                            accB.y *= sc;
                            MB = mB;
                        }
#pragma unroll
                        for (int mm = 0; mm < 4; ++mm) {
                            if (MA != -INFINITY)
                                accA = __fadd2_rn(accA, make_float2(ex2(x[k][4 * mm] - MA), ex2(x[k][4 * mm + 1] - MA)));
                            if (MB != -INFINITY)
                                accB = __fadd2_rn(accB, make_float2(ex2(x[k][4 * mm + 2] - MB), ex2(x[k][4 * mm + 3] - MB)));
                        }
                    } else {
                        const bool inner = sl >= in_lo && sl <= in_hi;
#pragma unroll
                        for (int mm = 0; mm < 4; ++mm) {
                            float2 za = __ffma2_rn(make_float2(x[k][4 * mm], x[k][4 * mm + 1]), c2v, __fadd2_rn(vv[k][mm], oA2));
                            float2 zb = __ffma2_rn(make_float2(x[k][4 * mm + 2], x[k][4 * mm + 3]), c2v, __fadd2_rn(vv[k][mm], oB2));
                            if (!inner) {
                                const int c = cb + 8 * mm;
                                za.x = (unsigned)(c - loA) <= (unsigned)bandw ? za.x : -INFINITY;
                                za.y = (unsigned)(c + 1 - loA) <= (unsigned)bandw ? za.y : -INFINITY;
                                zb.x = (unsigned)(c - loB) <= (unsigned)bandw ? zb.x : -INFINITY;
                                zb.y = (unsigned)(c + 1 - loB) <= (unsigned)bandw ? zb.y : -INFINITY;
                            }
                            const float2 ea = make_float2(ex2(za.x), ex2(za.y));
                            const float2 eb = make_float2(ex2(zb.x), ex2(zb.y));
                            x[k][4 * mm] = ea.x;
                            x[k][4 * mm + 1] = ea.y;
                            x[k][4 * mm + 2] = eb.x;
                            x[k][4 * mm + 3] = eb.y;
                            accA = __fadd2_rn(accA, ea);
                            accB = __fadd2_rn(accB, eb);
                        }
                        tc_st16x256(tl + (uint32_t)(((tseq + (sl >> 2)) & (NST - 1)) * kCR + (sl & 3) * 32), x[k]);
                    }
                }
            }
            if (!kRec) tc_wait_st();
            if (trc) FS_TRACE(33 + (gi - g_begin));
            // ---- row sums over the 4 threads (t0) sharing a row: u and the column weights 1 / r
            float sA = accA.x + accA.y, sB = accB.x + accB.y;
#pragma unroll
            for (int o = 1; o <= 2; o <<= 1) {
                const float pA = __shfl_xor_sync(0xffffffffu, sA, o), pB = __shfl_xor_sync(0xffffffffu, sB, o);
                if (kFirst) {
                    const float qA = __shfl_xor_sync(0xffffffffu, MA, o), qB = __shfl_xor_sync(0xffffffffu, MB, o);
                    const float nA = fmaxf(MA, qA), nB = fmaxf(MB, qB);
                    sA = (MA == -INFINITY ? 0.f : sA * ex2(MA - nA)) + (qA == -INFINITY ? 0.f : pA * ex2(qA - nA));
                    sB = (MB == -INFINITY ? 0.f : sB * ex2(MB - nB)) + (qB == -INFINITY ? 0.f : pB * ex2(qB - nB));
                    MA = nA;
                    MB = nB;
                } else {
                    sA += pA;
                    sB += pB;
                }
            }
            float wA = 0.f, wB = 0.f, uA = 0.f, uB = 0.f;
            if (actA) {
                uA = kFirst ? (-MA - lg2(sA)) : (oA - lg2(sA));
                if (!(sA > 0.f) || !isfinite(uA)) { atomicOr(a.err, 4); uA = 0.f; } else wA = 1.f / sA;
            }
            if (actB) {
                uB = kFirst ? (-MB - lg2(sB)) : (oB - lg2(sB));
                if (!(sB > 0.f) || !isfinite(uB)) { atomicOr(a.err, 4); uB = 0.f; } else wB = 1.f / sB;
            }
            if (t0 == 0) {
                const size_t uo = (size_t)b.bh * a.Lr_own, po = (size_t)b.bh * a.pad_ld_own + a.pad_off;
                if (iA < a.L_own) {
                    a.out_own[uo + iA] = uA;
                    a.pad_own[po + iA] = actA ? uA : -INFINITY;
                }
                if (iB < a.L_own) {
                    a.out_own[uo + iB] = uB;
                    a.pad_own[po + iB] = actB ? uB : -INFINITY;
                }
            }
            // ---- column pass: c_Ij = sum_i e_ij / r_i over the warp's 16 rows, per column
            const float2 wA2 = make_float2(wA, wA), wB2 = make_float2(wB, wB);
            const float offA = kFirst ? -MA : oA, offB = kFirst ? -MB : oB;
            float* cp = s.colp + ((size_t)par * 8 + (size_t)(qd * 2 + hf)) * a.maxwin;
            for (int sl = 0; sl < s_lo; ++sl) cp[sl * 32 + ccol] = 0.f;
            for (int sl = s_hi + 1; sl < nsl; ++sl) cp[sl * 32 + ccol] = 0.f;
            int rel = 0;  // chunks this warp released
            for (int g0 = s_lo; g0 <= s_hi; g0 += kG) {
                const int gl = min(s_hi, g0 + kG - 1);
                for (; rel < (g0 >> 2); ++rel) {  // chunks wholly before this round: done
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&s.t_empty[(tseq + rel) & (NST - 1)]);
                }
                tc_fence_after();
                float x[kG][16];
#pragma unroll
                for (int k = 0; k < kG; ++k) {
                    const int sl = min(g0 + k, gl);
                    tc_ld16x256(tl + (uint32_t)(((tseq + (sl >> 2)) & (NST - 1)) * kCR + (sl & 3) * 32), x[k]);
                }
                tc_wait_ld();
                float y[kG][8];
#pragma unroll
                for (int k = 0; k < kG; ++k) {
                    const int sl = min(g0 + k, gl);
                    if (kRec) {
                        const int cb = sl * 32 + 2 * t0;
#pragma unroll
                        for (int mm = 0; mm < 4; ++mm)
#pragma unroll
                            for (int c = 0; c < 2; ++c) {
                                const int col = cb + 8 * mm + c;
                                float za = fmaf(x[k][4 * mm + c], a.c2, vw[col]) + offA;
                                float zb = fmaf(x[k][4 * mm + 2 + c], a.c2, vw[col]) + offB;
                                za = (actA && (unsigned)(col - loA) <= (unsigned)bandw) ? za : -INFINITY;
                                zb = (actB && (unsigned)(col - loB) <= (unsigned)bandw) ? zb : -INFINITY;
                                x[k][4 * mm + c] = ex2(za);
                                x[k][4 * mm + 2 + c] = ex2(zb);
                            }
                    }
#pragma unroll
                    for (int mm = 0; mm < 4; ++mm) {
                        const float2 pr = __ffma2_rn(make_float2(x[k][4 * mm + 2], x[k][4 * mm + 3]), wB2,
                                                     __fmul2_rn(make_float2(x[k][4 * mm], x[k][4 * mm + 1]), wA2));
                        y[k][2 * mm] = pr.x;
                        y[k][2 * mm + 1] = pr.y;
                    }
                }
                // reduce over t1 (lane bits 2..4): after the 3 stages lane holds column ccol
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                    for (int k = 0; k < kG; ++k) {
                        const float send = u4 ? y[k][j] : y[k][j + 4];
                        const float keep = u4 ? y[k][j + 4] : y[k][j];
                        y[k][j] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
                    }
#pragma unroll
                for (int j = 0; j < 2; ++j)
#pragma unroll
                    for (int k = 0; k < kG; ++k) {
                        const float send = u3 ? y[k][j] : y[k][j + 2];
                        const float keep = u3 ? y[k][j + 2] : y[k][j];
                        y[k][j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
                    }
#pragma unroll
                for (int k = 0; k < kG; ++k) {
                    const float send = u2 ? y[k][0] : y[k][1];
                    const float keep = u2 ? y[k][1] : y[k][0];
                    const float val = keep + __shfl_xor_sync(0xffffffffu, send, 4);
                    if (g0 + k <= gl) cp[(g0 + k) * 32 + ccol] = val;
                }
            }
            for (; rel < nch; ++rel) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&s.t_empty[(tseq + rel) & (NST - 1)]);
            }
            tseq += nch;
            if (trc) FS_TRACE(41 + (gi - g_begin));
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.v_empty[vs]);  // window duals no longer needed
            named_bar(2, NE);
            if (trc) FS_TRACE(49 + (gi - g_begin));
            // ---- combine the 8 half-quadrant partials in fixed order; store the block's column partials
            const float* cb8 = s.colp + (size_t)par * 8 * a.maxwin;
            float* dst = part_out + ((size_t)b.bh * a.NB + b.blk) * a.maxwin;
            for (int c = et; c < nch * kCR; c += NE) {
                float sum = 0.f;
#pragma unroll
                for (int k = 0; k < 8; ++k) sum += cb8[(size_t)k * a.maxwin + c];
                dst[c] = sum;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) FS_TRACE(0);
    if (warp == 1) {
        tc_fence_after();
        tc_dealloc(tbase, 512);
    }
}

// ---------------------------------------------------------------------------
// v^t_j = v^{t-1}_j - lg2( sum_{I : rows of I meet band(j)} c_Ij ), ascending I.
// pad_v in place (-inf stays on inactive / guard entries); v_out (standard layout).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_vmerge(const float* __restrict__ part, float* __restrict__ pad_v,
                                                float* __restrict__ v_out, int BH, int H, int Lq, int Lk, int Lrk,
                                                int NB, int maxwin, int w, int CR, int shift, int Lp_other, int pad_ld,
                                                int pad_off, const uint8_t* __restrict__ col_mask, int* __restrict__ err) {
    // grid (ceil(Lk / 256), BH): 32-bit indices, no divisions on the element path (CR is 64 or 128)
    const int bh = blockIdx.y;
    const int j = blockIdx.x * 256 + threadIdx.x;
    if (j >= Lk) return;
    const int lcr = CR == 128 ? 7 : 6;
    float* pv = pad_v + (size_t)bh * pad_ld + pad_off + j;
    // every load in flight together (the old dual and up to 3 partials; out-of-range slots re-read the last)
    const int I0 = max(0, j - w) >> 7, I1 = min(Lq - 1, j + w) >> 7;
    const float* pb = part + (size_t)bh * NB * maxwin;
    const float vold = *pv;
    float pr[3];
    const bool small = I1 - I0 < 3;
#pragma unroll
    for (int t = 0; t < 3; ++t) {
        const int I = min(I0 + t, I1);
        const int q0 = max(0, (I * 128 - w + shift) >> lcr);  // first window chunk of block I
        pr[t] = small ? pb[(size_t)I * maxwin + (j - ((q0 << lcr) - shift))] : 0.f;
    }
    float v = 0.f;
    if (vold != -INFINITY) {  // active column (the padded buffer carries the mask)
        float sum = 0.f;
        if (small) {
#pragma unroll
            for (int t = 0; t < 3; ++t)
                if (I0 + t <= I1) sum += pr[t];
        } else {  // bands wider than 128: more than 3 row blocks meet a column
            for (int I = I0; I <= I1; ++I) {
                const int q0 = max(0, (I * 128 - w + shift) >> lcr);
                sum += pb[(size_t)I * maxwin + (j - ((q0 << lcr) - shift))];
            }
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

static thread_local long long g_fs_launches = 0;
long long fstep16_launch_count(bool reset) {
    const long long c = g_fs_launches;
    if (reset) g_fs_launches = 0;
    return c;
}

size_t fstep16_smem_bytes(const PhaseArgs& a) {
    const int nst = 512 / a.CR;
    return (size_t)a.NA * 128 * a.row_bytes + (size_t)a.NSK * a.CR * a.row_bytes +
           (size_t)(kNV * (a.maxwin + 128) + 2 * 8 * a.maxwin + 8 * 2 * 16) * 4 +
           (size_t)(2 * kNV + 2 * a.NA + 2 * a.NSK + 2 * nst) * 8 + 16 + (size_t)a.wl_cap * 16;
}

template <bool kFirst, bool kRec, bool kTma>
static cudaError_t launch_fstep16_t(const PhaseArgs& a, float* part, int grid, cudaStream_t s) {
    const size_t smem = fstep16_smem_bytes(a);
    auto k = k_fstep16<kFirst, kRec, kTma>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<grid, 64 + 32 * kEW, smem, s>>>(a, part);
    ++g_fs_launches;
    return cudaGetLastError();
}

cudaError_t launch_fstep16(const PhaseArgs& a, float* part, bool first, int grid, cudaStream_t s) {
    static const bool rec = getenv("ST_FSTEP_RECOMPUTE") != nullptr;
    if (a.npl != 1 || a.CR != 128 || a.dustbin) return cudaErrorNotSupported;
    if (a.tma) {  // operand tiles through tensor maps (no packed planes)
        if (first) return rec ? launch_fstep16_t<true, true, true>(a, part, grid, s) : launch_fstep16_t<true, false, true>(a, part, grid, s);
        return rec ? launch_fstep16_t<false, true, true>(a, part, grid, s) : launch_fstep16_t<false, false, true>(a, part, grid, s);
    }
    if (first) return rec ? launch_fstep16_t<true, true, false>(a, part, grid, s) : launch_fstep16_t<true, false, false>(a, part, grid, s);
    return rec ? launch_fstep16_t<false, true, false>(a, part, grid, s) : launch_fstep16_t<false, false, false>(a, part, grid, s);
}

cudaError_t launch_vmerge(const float* part, float* pad_v, float* v_out, int BH, int H, int Lq, int Lk, int Lrk, int NB,
                          int maxwin, int w, int CR, int shift, int Lp_other, int pad_ld, int pad_off,
                          const uint8_t* col_mask, int* err, cudaStream_t s) {
    k_vmerge<<<dim3((Lk + 255) / 256, BH), 256, 0, s>>>(part, pad_v, v_out, BH, H, Lq, Lk, Lrk, NB, maxwin, w, CR,
                                                          shift, Lp_other, pad_ld, pad_off, col_mask, err);
    ++g_fs_launches;
    return cudaGetLastError();
}

}  // namespace st
