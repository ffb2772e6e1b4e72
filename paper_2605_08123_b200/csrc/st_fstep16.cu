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
constexpr int kEW = 16;    // epilogue warps
constexpr int kParts = 4;  // column parts per lane quadrant

struct FSmem {
    uint8_t* A;       // [NA][128 * row_bytes]
    uint8_t* K;       // [NSK][CR * row_bytes]
    float* vwin;      // [kNV][maxwin + 128]
    float* rowp;      // [2][2][kParts][128]: row partial (sum, max) per part, by block parity
    float* colp;      // [2][4][maxwin]: column partials per lane quadrant, by block parity
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
    s.colp = s.rowp + 2 * 2 * kParts * 128;
    uint64_t* bars = (uint64_t*)(s.colp + 2 * 4 * a.maxwin);
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
    constexpr int HC = kCR / kParts;  // 32 columns per warp per chunk
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
            constexpr int kG = 2;
            for (int q0 = b.q0; q0 <= b.q1; q0 += kG) {
                const int ng = min(kG, b.q1 - q0 + 1);
                uint64_t bd[kG];
                uint32_t dt[kG];
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
                        bd[c] = make_desc(smem_u32(s.K + (size_t)sl * chk_bytes), 128, sbo);
                        dt[c] = tbase + (uint32_t)((tq % NST) * kCR);
                    }
                }
                tc_fence_after();
                if (elect_one()) {
                    for (int kk = 0; kk < ksteps; ++kk) {
#pragma unroll
                        for (int c = 0; c < kG; ++c)
                            if (c < ng && (kk == 0 || !(a.dbg & 2)))
                                mma_bf16(dt[c], ad0 + (uint64_t)(kk * 16), bd[c] + (uint64_t)(kk * 16), idesc, kk > 0);
                    }
#pragma unroll
                    for (int c = 0; c < kG; ++c)
                        if (c < ng) tc_commit(&s.t_full[(tseq + c) % NST]);
                }
                __syncwarp();
                tseq += ng;
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
        const int ew = warp - 2;
        const int qd = warp & 3;       // TMEM lane quadrant (warp_id % 4)
        const int part = ew >> 2;      // column part 0..3
        const int r = qd * 32 + lane;  // row inside the block
        const int et = threadIdx.x - 64;
        uint32_t tseq = 0;
        for (int gi = g_begin; gi < g_end; ++gi) {
            const Blk b = fblock_of(a, s.wl[gi - g_begin]);
            const int par = (gi - g_begin) & 1;
            const int vs = (gi - g_begin) % kNV;
            mbar_wait(&s.v_full[vs], ((gi - g_begin) / kNV) & 1);
            const float* vw = s.vwin + (size_t)vs * (a.maxwin + 128);
            const int wbase = b.q0 * kCR - a.shift;
            const int nch = b.q1 - b.q0 + 1;
            const int i = b.i0 + r;
            const float so = vw[a.maxwin + r];
            const bool active = i < a.L_own && so != -INFINITY;
            const float o = (!kFirst && active) ? so : 0.f;
            const int lo = i - a.w - wbase;                // band of this lane, window coordinates
            const int wlo = b.i0 + qd * 32 - a.w - wbase;  // union over the warp
            const int whi = wlo + 31 + 2 * a.w;
            const int ilo = wlo + 31, ihi = wlo + 2 * a.w;  // intersection over the warp
            // ---- row pass: e = ex2(s2 + v + o), written back over S (later steps)
            // kRec: the column pass recomputes e instead (the cold start always does: its online
            // per-part max would leave earlier slices relative to a stale max)
            constexpr bool kRec = kRecompute || kFirst;
            float acc0 = 0.f, acc1 = 0.f, M = -INFINITY;
            for (int q = 0; q < nch; ++q) {
                const int ts = (tseq + q) % NST;
                mbar_wait(&s.t_full[ts], ((tseq + q) / NST) & 1);
                tc_fence_after();
                const int c0 = q * kCR + part * HC;
                const bool any = !(whi < c0 || wlo > c0 + HC - 1);
                if (!any) continue;
                const bool inner = (c0 >= ilo) && (c0 + HC - 1 <= ihi);
                const uint32_t taddr = tbase + ((uint32_t)(qd * 32) << 16) + (uint32_t)(ts * kCR + part * HC);
                float v[32];
                tc_ld32(taddr, v);
                tc_wait_ld();
                if (a.dbg & 1) {  // ablation: no row math
                } else if (!active) {  // no early exit: tcgen05.st below is warp-collective
#pragma unroll
                    for (int cc = 0; cc < HC; ++cc) v[cc] = 0.f;
                } else if (kFirst) {
                    float m = -INFINITY;
#pragma unroll
                    for (int cc = 0; cc < HC; ++cc) {
                        const int c = c0 + cc;
                        const float x = fmaf(v[cc], a.c2, vw[c]);
                        v[cc] = ((unsigned)(c - lo) <= (unsigned)(2 * a.w)) ? x : -INFINITY;
                        m = fmaxf(m, v[cc]);
                    }
                    if (m > M) {
                        const float sc = (M == -INFINITY) ? 0.f : ex2(M - m);
                        acc0 *= sc;
                        acc1 *= sc;
                        M = m;
                    }
                    if (M != -INFINITY) {
#pragma unroll
                        for (int cc = 0; cc < HC; cc += 2) {
                            acc0 += ex2(v[cc] - M);
                            acc1 += ex2(v[cc + 1] - M);
                        }
                    }
                } else if (inner) {
#pragma unroll
                    for (int cc = 0; cc < HC; cc += 4) {
                        const float4 w4 = *reinterpret_cast<const float4*>(vw + c0 + cc);
                        v[cc + 0] = ex2(fmaf(v[cc + 0], a.c2, w4.x) + o);
                        v[cc + 1] = ex2(fmaf(v[cc + 1], a.c2, w4.y) + o);
                        v[cc + 2] = ex2(fmaf(v[cc + 2], a.c2, w4.z) + o);
                        v[cc + 3] = ex2(fmaf(v[cc + 3], a.c2, w4.w) + o);
                        acc0 += v[cc + 0] + v[cc + 2];
                        acc1 += v[cc + 1] + v[cc + 3];
                    }
                } else {
#pragma unroll
                    for (int cc = 0; cc < HC; ++cc) {
                        const int c = c0 + cc;
                        float x = fmaf(v[cc], a.c2, vw[c]) + o;
                        x = ((unsigned)(c - lo) <= (unsigned)(2 * a.w)) ? x : -INFINITY;
                        v[cc] = ex2(x);
                        if (cc & 1) acc1 += v[cc];
                        else acc0 += v[cc];
                    }
                }
                if (!kRec) tc_st32(taddr, v);
            }
            if (!kRec) tc_wait_st();
            // ---- row sums: combine the 4 column parts in fixed order
            float* rp = s.rowp + (size_t)par * 2 * kParts * 128;
            rp[part * 128 + r] = acc0 + acc1;
            if (kFirst) rp[(kParts + part) * 128 + r] = M;
            named_bar(2, NE);
            float rsum = 0.f, Mall = -INFINITY;
            if (kFirst) {
#pragma unroll
                for (int p = 0; p < kParts; ++p) Mall = fmaxf(Mall, rp[(kParts + p) * 128 + r]);
#pragma unroll
                for (int p = 0; p < kParts; ++p) {
                    const float Mp = rp[(kParts + p) * 128 + r];
                    rsum += (Mp == -INFINITY) ? 0.f : rp[p * 128 + r] * ex2(Mp - Mall);
                }
            } else {
#pragma unroll
                for (int p = 0; p < kParts; ++p) rsum += rp[p * 128 + r];
            }
            float u = 0.f, wgt = 0.f;
            if (active) {
                u = kFirst ? (-Mall - lg2(rsum)) : (o - lg2(rsum));
                if (!(rsum > 0.f) || !isfinite(u)) {
                    atomicOr(a.err, 4);
                    u = 0.f;
                } else {
                    wgt = 1.f / rsum;
                }
            }
            if (part == 0 && i < a.L_own) {
                a.out_own[(size_t)b.bh * a.Lr_own + i] = u;
                a.pad_own[(size_t)b.bh * a.pad_ld_own + a.pad_off + i] = active ? u : -INFINITY;
            }
            // ---- column pass: c_Ij = sum_i e_ij / r_i over the warp's 32 rows, per column
            const float off = kFirst ? -Mall : o;
            float* cp = s.colp + (size_t)par * 4 * a.maxwin + (size_t)qd * a.maxwin;
            for (int q = 0; q < nch; ++q) {
                const int ts = (tseq + q) % NST;
                const int c0 = q * kCR + part * HC;
                const bool any = !(whi < c0 || wlo > c0 + HC - 1);
                float val = 0.f;
                if (any) {
                    tc_fence_after();
                    const uint32_t taddr = tbase + ((uint32_t)(qd * 32) << 16) + (uint32_t)(ts * kCR + part * HC);
                    float v[32];
                    tc_ld32(taddr, v);
                    tc_wait_ld();
                    if (kRec) {
#pragma unroll
                        for (int cc = 0; cc < HC; ++cc) {
                            const int c = c0 + cc;
                            float x = fmaf(v[cc], a.c2, vw[c]) + off;
                            x = ((unsigned)(c - lo) <= (unsigned)(2 * a.w) && active) ? x : -INFINITY;
                            v[cc] = ex2(x) * wgt;
                        }
                    } else {
#pragma unroll
                        for (int cc = 0; cc < HC; ++cc) v[cc] *= wgt;
                    }
                    val = (a.dbg & 4) ? v[0] : colsum32(v, lane);
                }
                cp[c0 + lane] = val;
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&s.t_empty[ts]);
            }
            tseq += nch;
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.v_empty[vs]);  // window duals no longer needed
            named_bar(2, NE);
            // ---- combine the 4 lane quadrants in fixed order; store the block's column partials
            const float* cb = s.colp + (size_t)par * 4 * a.maxwin;
            float* dst = part_out + ((size_t)b.bh * a.NB + b.blk) * a.maxwin;
            for (int c = et; c < nch * kCR; c += NE)
                dst[c] = ((cb[c] + cb[a.maxwin + c]) + cb[2 * a.maxwin + c]) + cb[3 * a.maxwin + c];
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
           (size_t)(kNV * (a.maxwin + 128) + 2 * 2 * kParts * 128 + 2 * 4 * a.maxwin) * 4 +
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
