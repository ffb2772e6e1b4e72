// st_phase.cu -- the tcgen05 half-step ("phase") kernel of the Sinkhorn forward.
//
// One launch = one half-step for every head:
//   row phase:  u_i <- o_i - lg2 sum_{j in band(i)} 2^( s2_ij + v_j + o_i )      (row_half_step,  sinkhorn.hpp:15-61)
//   col phase:  v_j <- o_j - lg2 sum_{i in band(j)} 2^( s2_ij + u_i + o_j )      (col_half_step,  sinkhorn.hpp:64-107)
// with s2 = (q.k) * log2(e)/(sqrt(d) eps) RECOMPUTED on the tensor cores for
// every 128-row block and never stored (O(L) extra HBM).  The column phase is
// the row phase of the transposed problem (A = K block, B = Q window), so one
// kernel serves both and every log-sum-exp is an in-thread TMEM-lane reduction.
//
// Persistent CTA (one per SM), warp-specialised:
//   warp 0      producer: 1-D bulk async copies (TMA engine, UBLKCP) of the packed
//               A block and of the B window in CR-row chunks into an SMEM ring;
//               chunks shared by consecutive blocks of a head are loaded once
//   warp 1      MMA issuer: tcgen05.mma kind::f16 (BF16) M=128, N=CR, K=16, two
//               window chunks interleaved (independent accumulators hide the
//               ~80 ns dependent-MMA latency); fp32 inputs use a 3-plane bf16
//               split (hi, mid, lo) with the 6 products of order <= 2^-16,
//               i.e. fp32-accurate scores at bf16 tensor rate
//   warps 2..9  epilogue: two warps per TMEM lane quadrant (each owns half of
//               every chunk's columns): tcgen05.ld, FFMA scale + window dual,
//               MUFU.EX2, in-thread sums, lg2; window duals prefetched one
//               block ahead into a double-buffered SMEM slot
// Offsets: cold start uses an online running max; every later step uses the
// previous dual of the same row (terms <= 1, sums in [1/W, W]).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "st_common.cuh"
#include "st_phase.cuh"
#include "st_sm100.cuh"

namespace st {

using namespace sm100;

namespace {

constexpr int kNV = 3;  // dual-window ring slots

struct Smem {
    uint8_t* A;       // [NA][npl][128 * row_bytes]
    uint8_t* K;       // [NSK][npl][CR * row_bytes]
    float* vwin;      // [kNV][maxwin + 128]: the block's window duals, then its 128 own previous duals
    float* part;      // [2][3][256] partial (sum, max) of the column parts 1..3, by block parity
    uint64_t* v_full;
    uint64_t* v_empty;
    uint64_t* a_full;
    uint64_t* a_empty;
    uint64_t* k_full;
    uint64_t* k_empty;
    uint64_t* t_full;
    uint64_t* t_empty;
    uint32_t* tmem_base;
    int* wl;          // [wl_cap] this CTA's slice of the work list (no global loads on the block path)
    float* stage;     // band write passes: [kEW][32][33] per-warp transpose tiles
};

__device__ __forceinline__ Smem carve(uint8_t* base, const PhaseArgs& a, int nst) {
    Smem s;
    const size_t blk = (size_t)128 * a.row_bytes, chk = (size_t)a.CR * a.row_bytes;
    s.A = base;
    s.K = s.A + (size_t)a.NA * a.npl * blk;
    s.vwin = (float*)(s.K + (size_t)a.NSK * a.npl * chk);
    s.part = s.vwin + kNV * (a.maxwin + 128);
    uint64_t* bars = (uint64_t*)(s.part + 1536);
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
    s.stage = (float*)(((uintptr_t)(s.wl + a.wl_cap) + 15) & ~(uintptr_t)15);
    return s;
}

// A 128-row block of the own side and its window chunks [q0, q1] of the other side.
// Chunk q = packed rows [q*CR, (q+1)*CR) = original rows [q*CR - shift, ...).
struct Blk {
    int bh, i0, q0, q1;
};
__device__ __forceinline__ Blk block_of(const PhaseArgs& a, int g) {
    Blk b;
    b.bh = g / a.NB;
    b.i0 = (g % a.NB) * 128;
    const int nq = a.Lp_other / a.CR;
    b.q0 = max(0, (b.i0 - a.w + a.shift) / a.CR);  // exact: shift = w mod CR, CR | 128
    b.q1 = min(nq - 1, (b.i0 + 128 + a.w + a.shift + a.CR - 1) / a.CR - 1);
    return b;
}

__device__ __forceinline__ bool on_mask(const uint8_t* m, int H, int L, int bh, int i) {
    return m == nullptr || m[(size_t)(bh / H) * L + i] != 0;
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// debug timeline: trace[cta][slot] for the first 16 CTAs (ST_TRACE_PHASE, st_api.cu)
#define ST_TRACE(slot)                                                                                \
    do {                                                                                              \
        if (a.trace && blockIdx.x < 16 && (slot) < 64) a.trace[blockIdx.x * 64 + (slot)] = gtimer(); \
    } while (0)


}  // namespace

// kWrite = 0: the half-step.  kWrite = 1 / 2: the same tiles written out as the stored score band
// (s2 = q.k c2, -inf off the support) / cotangent band (dO.v, 0 off the support) of the own side,
// [BH][band_ld][Wf] (the transposed band from the column geometry); activity from the padded duals.
// kTma: the operand tiles come from the raw tensors through tensor maps (128B-swizzled boxes) instead of
// the packed planes (bf16, one plane).
template <int kNPL, int kCR, bool kFirst, int kEW, int kWrite = 0, bool kTma = false>
__global__ void __launch_bounds__(64 + 32 * kEW, 1) k_phase(const __grid_constant__ PhaseArgs a) {
    constexpr int kParts = kEW / 4;         // epilogue warps per TMEM lane quadrant (column parts)
    constexpr int NE = 32 * kEW;            // epilogue threads
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    constexpr int NST = 512 / kCR;  // TMEM accumulator slots
    const Smem s = carve(smem_raw, a, NST);
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
        atomicOr(a.err, 16);  // cannot happen: wl_cap = ceil(max work / grid)
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *s.tmem_base;
    if (threadIdx.x == 0) ST_TRACE(0);

    if (warp == 0) {
        // ------------------------------------------------------------ producer (warp-uniform loop)
        int last_bh = -1, last_q = -1;
        uint32_t kseq = 0;
        for (int gi = g_begin; gi < g_end; ++gi) {
            const Blk b = block_of(a, s.wl[gi - g_begin]);
            {   // masked window duals of the other side + previous own duals (padded buffers, -inf guards)
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
                ST_TRACE(1 + min(gi - g_begin, 7));
                mbar_arrive_expect_tx(&s.a_full[ab], blk_bytes * kNPL);
                if constexpr (kTma) {  // raw rows i0 .. i0 + 127: one 128-row swizzled box per d half
                    for (int kb = 0; kb < a.row_bytes / 128; ++kb)
                        tma_load_3d(s.A + (size_t)ab * blk_bytes + kb * 16384, &a.tmA, kb * 64, b.i0, b.bh, &s.a_full[ab]);
                } else {
#pragma unroll
                    for (int p = 0; p < kNPL; ++p)
                        bulk_g2s(s.A + ((size_t)ab * kNPL + p) * blk_bytes,
                                 a.A_pack[p] + ((size_t)b.bh * a.Lp_own + b.i0 + a.shift) * a.row_bytes, blk_bytes,
                                 &s.a_full[ab]);
                }
            }
            __syncwarp();
            const int qstart = (b.bh == last_bh) ? max(b.q0, last_q + 1) : b.q0;
            for (int q = qstart; q <= b.q1; ++q) {
                const int sl = kseq % a.NSK;
                const uint32_t kn = kseq / a.NSK;
                mbar_wait(&s.k_empty[sl], (kn & 1) ^ 1);
                if (elect_one()) {
                    mbar_arrive_expect_tx(&s.k_full[sl], chk_bytes * kNPL);
                    if constexpr (kTma) {  // chunk q = raw rows q * kCR - shift .. (zeros outside the tensor)
                        for (int kb = 0; kb < a.row_bytes / 128; ++kb)
                            tma_load_3d(s.K + (size_t)sl * chk_bytes + kb * (kCR * 128), &a.tmB, kb * 64, q * kCR - a.shift, b.bh,
                                        &s.k_full[sl]);
                    } else {
#pragma unroll
                        for (int p = 0; p < kNPL; ++p)
                            bulk_g2s(s.K + ((size_t)sl * kNPL + p) * chk_bytes,
                                     a.B_pack[p] + ((size_t)b.bh * a.Lp_other + (size_t)q * kCR) * a.row_bytes, chk_bytes,
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
        // ------------------------------------------------------------ MMA issuer (warp-uniform loop)
        const uint32_t idesc = make_idesc(128, kCR, 1u);            // BF16 x BF16 -> F32
        const uint32_t sbo = (uint32_t)(a.row_bytes / 16) * 128u;   // bytes between 8-row groups
        const int ksteps = a.row_bytes / 32;                         // MMA-K slices of 32 bytes (16 bf16)
        const uint64_t a_plane = (uint64_t)(blk_bytes >> 4), b_plane = (uint64_t)(chk_bytes >> 4);
        // products (plane of A, plane of B): exact for bf16 inputs; fp32 = hi+mid+lo with the
        // 6 products hh, hm, mh, hl, mm, lh (omitted terms are below 2^-24 relative)
        constexpr int kNP = (kNPL == 1) ? 1 : 6;
        constexpr int pa_[6] = {0, 0, 1, 0, 1, 2};
        constexpr int pb_[6] = {0, 1, 0, 2, 1, 0};
        int last_bh = -1, last_q = -1;
        uint32_t last_seq = 0, rel_seq = 0, tseq = 0;
        bool have = false;
        for (int gi = g_begin; gi < g_end; ++gi) {
            const Blk b = block_of(a, s.wl[gi - g_begin]);
            const int ab = (gi - g_begin) % a.NA;
            const uint32_t an = (gi - g_begin) / a.NA;
            mbar_wait(&s.a_full[ab], an & 1);
            if (lane == 0) ST_TRACE(9 + min(gi - g_begin, 7));
            tc_fence_after();
            const uint32_t as_ = smem_u32(s.A + (size_t)ab * kNPL * blk_bytes);
            const uint64_t ad0 = make_desc(as_, 128, sbo);
            const uint64_t ad_sw = make_desc_sw128(as_, 16, 1024);
            const bool same = have && b.bh == last_bh;
            const int new_start = same ? max(b.q0, last_q + 1) : b.q0;
            const uint32_t next_seq = have ? last_seq + 1 : 0;
            constexpr int kG = 2;  // chunks per MMA group (independent accumulators)
            for (int q0 = b.q0; q0 <= b.q1; q0 += kG) {
                const int ng = min(kG, b.q1 - q0 + 1);
                uint64_t bd[kG], bd_sw[kG];
                uint32_t dt[kG], bs_[kG];
#pragma unroll
                for (int c = 0; c < kG; ++c) {
                    if (c < ng) {
                        const int q = q0 + c;
                        const uint32_t seq = (same && q <= last_q) ? last_seq - (uint32_t)(last_q - q)
                                                                   : next_seq + (uint32_t)(q - new_start);
                        const int sl = seq % a.NSK;
                        mbar_wait(&s.k_full[sl], (seq / a.NSK) & 1);
                        const uint32_t tq = tseq + c;
                        mbar_wait(&s.t_empty[tq % NST], ((tq / NST) & 1) ^ 1);
                        bs_[c] = smem_u32(s.K + (size_t)sl * kNPL * chk_bytes);
                        bd[c] = make_desc(bs_[c], 128, sbo);
                        bd_sw[c] = make_desc_sw128(bs_[c], 16, 1024);
                        dt[c] = tbase + (uint32_t)((tq % NST) * kCR);
                    }
                }
                tc_fence_after();
                if (elect_one()) {
#pragma unroll
                    for (int pr = 0; pr < kNP; ++pr)
                        for (int kk = 0; kk < ((a.dbg & 2) ? 1 : ksteps); ++kk) {
                            const uint64_t adk = ad0 + (uint64_t)pa_[pr] * a_plane + (uint64_t)(kk * 16);
#pragma unroll
                            for (int c = 0; c < kG; ++c)
                                if (c < ng) {
                                    if constexpr (kTma)  // swizzled tiles: d half kk / 4, 32 bytes per K step inside the row
                                        mma_bf16(dt[c], ad_sw + (uint64_t)((kk >> 2) * 1024 + (kk & 3) * 2),
                                                 bd_sw[c] + (uint64_t)((kk >> 2) * (kCR * 8) + (kk & 3) * 2), idesc, kk > 0);
                                    else
                                        mma_bf16(dt[c], adk, bd[c] + (uint64_t)pb_[pr] * b_plane + (uint64_t)(kk * 16),
                                                 idesc, (pr | kk) > 0);
                                }
                        }
#pragma unroll
                    for (int c = 0; c < kG; ++c)
                        if (c < ng) tc_commit(&s.t_full[(tseq + c) % NST]);
                }
                __syncwarp();
                tseq += ng;
            }
            if (elect_one()) tc_commit(&s.a_empty[ab]);  // A is free once this block's MMAs completed
            __syncwarp();
            if (lane == 0) ST_TRACE(17 + min(gi - g_begin, 7));
            // chunk bookkeeping (mirrors the producer)
            if (b.q1 >= new_start) last_seq = next_seq + (uint32_t)(b.q1 - new_start);
            if (!same) last_q = -1;
            last_q = max(last_q, b.q1);
            last_bh = b.bh;
            have = true;
            // release ring slots the next block of this CTA does not need
            uint32_t keep_from = last_seq + 1;
            if (gi + 1 < g_end) {
                const Blk nb = block_of(a, s.wl[gi + 1 - g_begin]);
                if (nb.bh == last_bh && nb.q0 <= last_q) keep_from = last_seq - (uint32_t)(last_q - nb.q0);
            }
            if (elect_one()) {
                for (uint32_t r = rel_seq; r < keep_from; ++r) tc_commit(&s.k_empty[r % a.NSK]);
            }
            __syncwarp();
            rel_seq = max(rel_seq, keep_from);
        }
    } else if constexpr (kWrite != 0) {
        // ------------------------------------------------------------ band write epilogue
        // A warp owns 32 rows x HC columns of each chunk; it stages them through a padded SMEM tile so
        // that, row by row, the 32 lanes store 32 consecutive band cells (coalesced), instead of 32 rows
        // per store instruction.  Cells outside the window (j before / after it) get the fill value.
        constexpr int HC = kCR / kParts;
        const int ew = warp - 2, qd = warp & 3, half = ew >> 2;
        float* stg = s.stage + (size_t)ew * 32 * 33;
        const float fill = kWrite == 1 ? -INFINITY : 0.f;
        uint32_t tseq = 0;
        for (int gi = g_begin; gi < g_end; ++gi) {
            const Blk b = block_of(a, s.wl[gi - g_begin]);
            const int vs = (gi - g_begin) % kNV;
            mbar_wait(&s.v_full[vs], ((gi - g_begin) / kNV) & 1);
            const float* vw = s.vwin + (size_t)vs * (a.maxwin + 128);
            const int wbase = b.q0 * kCR - a.shift;
            const int nwin = (b.q1 - b.q0 + 1) * kCR;
            const int wlo = b.i0 + qd * 32 - a.w - wbase;  // window column of band cell k = 0, row 32 qd
            const int i = b.i0 + qd * 32 + lane;
            const bool act = i < a.L_own && vw[a.maxwin + qd * 32 + lane] != -INFINITY;
            const unsigned actm = __ballot_sync(0xffffffffu, act);
            float* obase = a.band_out + ((size_t)b.bh * a.band_ld + b.i0 + qd * 32) * a.Wf;
            for (int q = b.q0; q <= b.q1; ++q) {
                const int ts = tseq % NST;
                mbar_wait(&s.t_full[ts], (tseq / NST) & 1);
                tc_fence_after();
                const int c0 = (q - b.q0) * kCR + half * HC;
                const bool any = !(wlo + 31 + 2 * a.w < c0 || wlo > c0 + HC - 1);
                float v[HC];
                if (any) {
                    const uint32_t taddr = tbase + ((uint32_t)(qd * 32) << 16) + (uint32_t)(ts * kCR + half * HC);
#pragma unroll
                    for (int h = 0; h < HC / 32; ++h) tc_ld32(taddr + 32 * h, *reinterpret_cast<float(*)[32]>(v + 32 * h));
                    tc_wait_ld();
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&s.t_empty[ts]);
                ++tseq;
                if (!any) continue;
#pragma unroll
                for (int h = 0; h < HC / 32; ++h) {
#pragma unroll
                    for (int cc = 0; cc < 32; ++cc) stg[lane * 33 + cc] = v[32 * h + cc];
                    __syncwarp();
                    const int c = c0 + 32 * h + lane;  // this lane's window column
                    const bool con = vw[c] != -INFINITY;
                    for (int rr = 0; rr < 32; ++rr) {
                        const int k = c - (wlo + rr);
                        if ((unsigned)k <= (unsigned)(2 * a.w)) {
                            const float x = stg[rr * 33 + lane];
                            const bool on = ((actm >> rr) & 1u) && con;
                            obase[(size_t)rr * a.Wf + k] = on ? (kWrite == 1 ? x * a.c2 : x) : fill;
                        }
                    }
                    __syncwarp();
                }
            }
            if (half == 0) {  // band cells whose column lies outside the block's window
                for (int rr = 0; rr < 32; ++rr) {
                    const int lo = wlo + rr;
                    for (int k = lane; k < min(-lo, 2 * a.w + 1); k += 32) obase[(size_t)rr * a.Wf + k] = fill;
                    for (int k = max(0, nwin - lo) + lane; k <= 2 * a.w; k += 32) obase[(size_t)rr * a.Wf + k] = fill;
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.v_empty[vs]);
        }
    } else {
        // ------------------------------------------------------------ epilogue (warps 2 .. 2 + kEW)
        constexpr int HC = kCR / kParts;          // columns per warp per chunk
        static_assert(HC % 32 == 0, "32-column TMEM loads");
        const int ew = warp - 2;                  // 0 .. kEW-1
        const int qd = warp & 3;                  // TMEM lane quadrant (warp_id % 4)
        const int half = ew >> 2;                 // column part 0 .. kParts-1
        const int r = qd * 32 + lane;             // row inside the 128-row block
        const int et = threadIdx.x - 64;          // 0 .. NE-1
        uint32_t tseq = 0;
        for (int gi = g_begin; gi < g_end; ++gi) {
            const Blk b = block_of(a, s.wl[gi - g_begin]);
            const int vs = (gi - g_begin) % kNV;
            mbar_wait(&s.v_full[vs], ((gi - g_begin) / kNV) & 1);
            const float* vw = s.vwin + (size_t)vs * (a.maxwin + 128);
            const int wbase = b.q0 * kCR - a.shift;   // original column of window column 0
            if (et == 0) ST_TRACE(25 + min(gi - g_begin, 7));
            const int i = b.i0 + r;
            const float so = vw[a.maxwin + r];        // previous own dual; -inf marks an inactive row
            const bool active = i < a.L_own && so != -INFINITY;
            float o = 0.f, acc0 = 0.f, acc1 = 0.f, M = -INFINITY;
            if (!kFirst && active) o = so;
            const int lo = i - a.w - wbase;               // band of this lane, window coordinates
            const int wlo = b.i0 + qd * 32 - a.w - wbase; // union over the warp
            const int whi = wlo + 31 + 2 * a.w;
            const int ilo = wlo + 31, ihi = wlo + 2 * a.w; // intersection over the warp
            for (int q = b.q0; q <= b.q1; ++q) {
                const int ts = tseq % NST;
                mbar_wait(&s.t_full[ts], (tseq / NST) & 1);
                tc_fence_after();
                const int c0 = (q - b.q0) * kCR + half * HC;
                const bool any = !(whi < c0 || wlo > c0 + HC - 1);
                const bool inner = (c0 >= ilo) && (c0 + HC - 1 <= ihi);
                float v[HC];
                if (any) {
                    const uint32_t taddr = tbase + ((uint32_t)(qd * 32) << 16) + (uint32_t)(ts * kCR + half * HC);
#pragma unroll
                    for (int h = 0; h < HC / 32; ++h) tc_ld32(taddr + 32 * h, *reinterpret_cast<float(*)[32]>(v + 32 * h));
                    tc_wait_ld();
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&s.t_empty[ts]);
                ++tseq;
                if (!any || !active || (a.dbg & 1)) continue;
                if (kFirst) {
                    float m = -INFINITY;
#pragma unroll
                    for (int cc = 0; cc < HC; ++cc) {
                        const int c = c0 + cc;
                        const float x = fmaf(v[cc], a.c2, vw[c]);
                        v[cc] = ((unsigned)(c - lo) <= (unsigned)(2 * a.w)) ? x : -INFINITY;
                        m = fmaxf(m, v[cc]);
                    }
                    if (m > M) {
                        acc0 = (M == -INFINITY) ? 0.f : acc0 * ex2(M - m);
                        M = m;
                    }
                    if (M != -INFINITY) {
#pragma unroll
                        for (int cc = 0; cc < HC; ++cc) acc0 += ex2(v[cc] - M);
                    }
                } else if (inner) {
#pragma unroll
                    for (int cc = 0; cc < HC; cc += 4) {
                        const float4 w4 = *reinterpret_cast<const float4*>(vw + c0 + cc);
                        acc0 += ex2(fmaf(v[cc + 0], a.c2, w4.x) + o);
                        acc1 += ex2(fmaf(v[cc + 1], a.c2, w4.y) + o);
                        acc0 += ex2(fmaf(v[cc + 2], a.c2, w4.z) + o);
                        acc1 += ex2(fmaf(v[cc + 3], a.c2, w4.w) + o);
                    }
                } else {
#pragma unroll
                    for (int cc = 0; cc < HC; ++cc) {
                        const int c = c0 + cc;
                        float x = fmaf(v[cc], a.c2, vw[c]) + o;
                        x = ((unsigned)(c - lo) <= (unsigned)(2 * a.w)) ? x : -INFINITY;
                        if (cc & 1) acc1 += ex2(x);
                        else acc0 += ex2(x);
                    }
                }
            }
            float acc_s = acc0 + acc1;
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.v_empty[vs]);  // window slot free for the producer
            if (et == 0) ST_TRACE(33 + min(gi - g_begin, 7));
            // combine the column parts of every row (fixed order 0, 1, .., kParts-1); the partials
            // are double-buffered by block parity, so one barrier per block suffices
            float* part = s.part + ((gi - g_begin) & 1) * 768;
            if (half > 0) {
                part[(half - 1) * 256 + r] = acc_s;
                part[(half - 1) * 256 + 128 + r] = M;
            }
            named_bar(2, NE);
            if (half == 0 && i < a.L_own) {
                float u = 0.f;
#pragma unroll
                for (int pp = 1; pp < kParts; ++pp) {
                    const float s1 = part[(pp - 1) * 256 + r];
                    if (kFirst) {
                        const float M1 = part[(pp - 1) * 256 + 128 + r];
                        const float Mx = fmaxf(M, M1);
                        acc_s = (M == -INFINITY ? 0.f : acc_s * ex2(M - Mx)) +
                                (M1 == -INFINITY ? 0.f : s1 * ex2(M1 - Mx));
                        M = Mx;
                    } else {
                        acc_s += s1;
                    }
                }
                if (active) {
                    if (a.dustbin) {  // the spoke cell (i, dustbin) with constant score sd2
                        const float x = a.sd2 + a.dual_other[(size_t)b.bh * a.Lr_other + a.L_other];
                        if (kFirst) {
                            if (x > M) {
                                acc_s = (M == -INFINITY) ? 0.f : acc_s * ex2(M - x);
                                M = x;
                            }
                            acc_s += ex2(x - M);
                        } else {
                            acc_s += ex2(x + o);
                        }
                    }
                    u = kFirst ? (-M - lg2(acc_s)) : (o - lg2(acc_s));
                    if (!(acc_s > 0.f) || !isfinite(u)) {
                        atomicOr(a.err, 4);
                        u = 0.f;
                    }
                }
                a.out_own[(size_t)b.bh * a.Lr_own + i] = u;
                a.pad_own[(size_t)b.bh * a.pad_ld_own + a.pad_off + i] = active ? u : -INFINITY;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) {
        ST_TRACE(41);
        if (a.trace && blockIdx.x < 16) a.trace[blockIdx.x * 64 + 42] = (unsigned long long)(g_end - g_begin);
    }
    if (warp == 1) {
        tc_fence_after();
        tc_dealloc(tbase, 512);
    }
}

// ---------------------------------------------------------------------------
// Dustbin row/column (spoke support): u_L <- o - lg2( sum_{j active} 2^(sd2 + v_j + o) + 2^(sd2 + v_L + o) )
// one CTA per head, fixed-order block reduction.
// ---------------------------------------------------------------------------
template <bool kFirst>
__global__ void __launch_bounds__(256) k_dustbin(DustArgs a) {
    const int bh = blockIdx.x;
    const float* dual = a.dual_other + (size_t)bh * a.Lr_other;
    const int n = a.L_other + 1;
    __shared__ float red[256];
    float off;
    if (kFirst) {
        float m = -INFINITY;
        for (int j = threadIdx.x; j < n; j += 256)
            if (j == a.L_other || on_mask(a.mask_other, a.H, a.L_other, bh, j)) m = fmaxf(m, a.sd2 + dual[j]);
        red[threadIdx.x] = m;
        __syncthreads();
        for (int o = 128; o > 0; o >>= 1) {
            if (threadIdx.x < o) red[threadIdx.x] = fmaxf(red[threadIdx.x], red[threadIdx.x + o]);
            __syncthreads();
        }
        off = -red[0];
        __syncthreads();
    } else {
        off = a.off_own[(size_t)bh * a.Lr_own + a.L_own];
    }
    float sum = 0.f;
    for (int j = threadIdx.x; j < n; j += 256)
        if (j == a.L_other || on_mask(a.mask_other, a.H, a.L_other, bh, j)) sum += ex2(a.sd2 + dual[j] + off);
    red[threadIdx.x] = sum;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        float u = off - lg2(red[0]);
        if (!(red[0] > 0.f) || !isfinite(u)) {
            atomicOr(a.err, 8);
            u = 0.f;
        }
        a.out_own[(size_t)bh * a.Lr_own + a.L_own] = u;
    }
}

// ---------------------------------------------------------------------------
// Packing: one thread per (head, packed row, 16-byte K chunk of 8 elements).
// bf16 input -> 1 plane (verbatim); fp32 input -> 3 bf16 planes
//   hi = bf16(x), mid = bf16(x - hi), lo = bf16(x - hi - mid)   (x - hi and x - hi - mid are exact in fp32)
// Packed row p holds original row p - shift (zero outside [0, L)).
// ---------------------------------------------------------------------------
template <class TIn>
__global__ void k_pack(const TIn* __restrict__ X, int BH, int L, int Lr, int Lp, int d, int shift,
                       uint8_t* __restrict__ p0, uint8_t* __restrict__ p1, uint8_t* __restrict__ p2) {
    const int kc_n = d / 8;
    const long total = (long)BH * Lp * kc_n;
    const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= total) return;
    const int kc = (int)(t % kc_n);
    const long rowg = t / kc_n;
    const int p = (int)(rowg % Lp);
    const int bh = (int)(rowg / Lp);
    const int r = p - shift;
    const size_t row_bytes = (size_t)d * 2;
    const size_t off = ((size_t)bh * Lp + (p & ~7)) * row_bytes + (size_t)kc * 128 + (p & 7) * 16;
    if (sizeof(TIn) == 2) {
        uint4 v = make_uint4(0, 0, 0, 0);
        if (r >= 0 && r < L) v = *reinterpret_cast<const uint4*>(X + ((size_t)bh * Lr + r) * d + kc * 8);
        *reinterpret_cast<uint4*>(p0 + off) = v;
    } else {
        float x[8];
        if (r >= 0 && r < L) {
            const float4* src = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(X) +
                                                                ((size_t)bh * Lr + r) * d + kc * 8);
            const float4 a = src[0], b = src[1];
            x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w; x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) x[k] = 0.f;
        }
        __align__(16) __nv_bfloat16 h[8], m[8], l[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            h[k] = __float2bfloat16_rn(x[k]);
            const float r1 = x[k] - __bfloat162float(h[k]);
            m[k] = __float2bfloat16_rn(r1);
            l[k] = __float2bfloat16_rn(r1 - __bfloat162float(m[k]));
        }
        *reinterpret_cast<uint4*>(p0 + off) = *reinterpret_cast<const uint4*>(h);
        *reinterpret_cast<uint4*>(p1 + off) = *reinterpret_cast<const uint4*>(m);
        *reinterpret_cast<uint4*>(p2 + off) = *reinterpret_cast<const uint4*>(l);
    }
}

// ---------------------------------------------------------------------------
// Padded masked dual buffers [BH][pad_ld]: entry pad_off + j holds the dual of column j when it is
// active, -inf otherwise (also on the guards j < 0, j >= L), so the producer can bulk-copy any
// window.  init: 0 on active entries (the cold start); refresh: copy from a standard [BH][Lr] vector.
// ---------------------------------------------------------------------------
__global__ void k_pad_fill(float* __restrict__ pad, const float* __restrict__ src, int BH, int H, int L, int Lr,
                           int pad_ld, int pad_off, const uint8_t* __restrict__ mask) {
    const long n = (long)BH * pad_ld;
    for (long t = (long)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (long)gridDim.x * blockDim.x) {
        const int bh = (int)(t / pad_ld), j = (int)(t % pad_ld) - pad_off;
        float x = -INFINITY;
        if (j >= 0 && j < L && on_mask(mask, H, L, bh, j)) x = src ? src[(size_t)bh * Lr + j] : 0.f;
        pad[t] = x;
    }
}

// ---------------------------------------------------------------------------
// Work lists: active 128-row blocks (any active row) in (head, block) order.
// ---------------------------------------------------------------------------
__global__ void k_block_flags(const uint8_t* __restrict__ mask, int H, int BH, int L, int NB, int* __restrict__ flags) {
    const int g = blockIdx.x;
    if (g >= BH * NB) return;
    const int bh = g / NB, b = g % NB;
    int any = 0;
    for (int r = threadIdx.x; r < 128; r += blockDim.x) {
        const int i = b * 128 + r;
        if (i < L && on_mask(mask, H, L, bh, i)) any = 1;
    }
    any = __syncthreads_or(any);
    if (threadIdx.x == 0) flags[g] = any;
}

__global__ void __launch_bounds__(1024) k_compact(const int* __restrict__ flags, int n, int* __restrict__ work,
                                                  int* __restrict__ count) {
    __shared__ int base;
    __shared__ int warp_tot[32];
    if (threadIdx.x == 0) base = 0;
    __syncthreads();
    for (int c0 = 0; c0 < n; c0 += 1024) {
        const int g = c0 + threadIdx.x;
        const int f = (g < n) ? flags[g] : 0;
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        const int pre = __popc(bal & ((1u << lane) - 1));
        if (lane == 0) warp_tot[wid] = __popc(bal);
        __syncthreads();
        int woff = 0;
        for (int k = 0; k < wid; ++k) woff += warp_tot[k];
        if (f) work[base + woff + pre] = g;
        __syncthreads();
        if (threadIdx.x == 0) {
            int tot = 0;
            for (int k = 0; k < 32; ++k) tot += warp_tot[k];
            base += tot;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *count = base;
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
static thread_local long long g_phase_launches = 0;
long long phase_launch_count(bool reset) {
    const long long c = g_phase_launches;
    if (reset) g_phase_launches = 0;
    return c;
}

size_t phase_smem_bytes(const PhaseArgs& a) {
    const int nst = 512 / a.CR;
    return (size_t)a.NA * a.npl * 128 * a.row_bytes + (size_t)a.NSK * a.npl * a.CR * a.row_bytes +
           (size_t)(kNV * (a.maxwin + 128) + 1536) * 4 + (size_t)(2 * kNV + 2 * a.NA + 2 * a.NSK + 2 * nst) * 8 + 16 + (size_t)a.wl_cap * 4 +
           (a.band_out ? (size_t)a.ew_write * 32 * 33 * 4 + 16 : 0);
}

template <int kNPL, int kCR, int kEW>
static cudaError_t launch_phase_t(const PhaseArgs& a, bool first, int grid, cudaStream_t s) {
    const size_t smem = phase_smem_bytes(a);
    auto k = first ? k_phase<kNPL, kCR, true, kEW> : k_phase<kNPL, kCR, false, kEW>;
    if (kNPL == 1 && a.tma) k = first ? k_phase<kNPL, kCR, true, kEW, 0, kNPL == 1> : k_phase<kNPL, kCR, false, kEW, 0, kNPL == 1>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<grid, 64 + 32 * kEW, smem, s>>>(a);
    ++g_phase_launches;
    return cudaGetLastError();
}

cudaError_t launch_phase(const PhaseArgs& a, bool first, int grid, cudaStream_t s) {
    // 128-column chunks: 16 epilogue warps (4 per TMEM lane quadrant, 32 columns each) hide the
    // tcgen05.ld -> MUFU latency; 64-column chunks keep 8 (2 per quadrant)
    static const int ew = getenv("ST_PHASE_EW") ? atoi(getenv("ST_PHASE_EW")) : 16;
    if (a.npl == 1) {
        if (a.CR == 128) return ew == 8 ? launch_phase_t<1, 128, 8>(a, first, grid, s) : launch_phase_t<1, 128, 16>(a, first, grid, s);
        return launch_phase_t<1, 64, 8>(a, first, grid, s);
    }
    if (a.CR == 128) return ew == 8 ? launch_phase_t<3, 128, 8>(a, first, grid, s) : launch_phase_t<3, 128, 16>(a, first, grid, s);
    return launch_phase_t<3, 64, 8>(a, first, grid, s);
}

template <int kCR, int kEW, int kW>
static cudaError_t launch_band_t(const PhaseArgs& a, int grid, cudaStream_t s) {
    const size_t smem = phase_smem_bytes(a);
    auto k = k_phase<1, kCR, false, kEW, kW>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k<<<grid, 64 + 32 * kEW, smem, s>>>(a);
    ++g_phase_launches;
    return cudaGetLastError();
}

cudaError_t launch_phase_band(const PhaseArgs& a, bool cotangent, int grid, cudaStream_t s) {
    if (a.npl != 1 || a.band_out == nullptr) return cudaErrorNotSupported;  // bf16 operand planes only
    if (a.CR == 128)
        return a.ew_write == 8 ? (cotangent ? launch_band_t<128, 8, 2>(a, grid, s) : launch_band_t<128, 8, 1>(a, grid, s))
                               : (cotangent ? launch_band_t<128, 16, 2>(a, grid, s) : launch_band_t<128, 16, 1>(a, grid, s));
    return cotangent ? launch_band_t<64, 8, 2>(a, grid, s) : launch_band_t<64, 8, 1>(a, grid, s);
}

cudaError_t launch_dustbin(const DustArgs& a, bool first, int BH, cudaStream_t s) {
    if (first) k_dustbin<true><<<BH, 256, 0, s>>>(a);
    else k_dustbin<false><<<BH, 256, 0, s>>>(a);
    ++g_phase_launches;
    return cudaGetLastError();
}

cudaError_t launch_pack(int dtype, const void* X, int BH, int L, int Lr, int Lp, int d, int shift, uint8_t* p0,
                        uint8_t* p1, uint8_t* p2, cudaStream_t s) {
    const long total = (long)BH * Lp * (d / 8);
    const unsigned nb = (unsigned)((total + 255) / 256);
    if (dtype == 0) k_pack<float><<<nb, 256, 0, s>>>((const float*)X, BH, L, Lr, Lp, d, shift, p0, p1, p2);
    else k_pack<__nv_bfloat16><<<nb, 256, 0, s>>>((const __nv_bfloat16*)X, BH, L, Lr, Lp, d, shift, p0, p1, p2);
    ++g_phase_launches;
    return cudaGetLastError();
}

cudaError_t launch_pad_fill(float* pad, const float* src, int BH, int H, int L, int Lr, int pad_ld, int pad_off,
                            const uint8_t* mask, cudaStream_t s) {
    const long n = (long)BH * pad_ld;
    const int nb = (int)std::min<long>((n + 255) / 256, 148L * 8);
    k_pad_fill<<<nb, 256, 0, s>>>(pad, src, BH, H, L, Lr, pad_ld, pad_off, mask);
    ++g_phase_launches;
    return cudaGetLastError();
}

cudaError_t launch_compact(const int* flags, int n, int* work, int* count, cudaStream_t s) {
    k_compact<<<1, 1024, 0, s>>>(flags, n, work, count);
    return cudaGetLastError();
}

cudaError_t launch_worklist(const uint8_t* mask, int H, int BH, int L, int NB, int* flags, int* work, int* count,
                            cudaStream_t s) {
    k_block_flags<<<BH * NB, 128, 0, s>>>(mask, H, BH, L, NB, flags);
    k_compact<<<1, 1024, 0, s>>>(flags, BH * NB, work, count);
    g_phase_launches += 2;
    return cudaGetLastError();
}

}  // namespace st
