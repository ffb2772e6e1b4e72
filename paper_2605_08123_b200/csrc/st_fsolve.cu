// st_fsolve.cu -- persistent, band-resident fused Sinkhorn solve (fp32 path).
//
// The whole stopped base solve + tail (stopped_base_solve / tail_refine,
// inc/sinkhorn.hpp:171-221) in ONE cooperative launch:
//   * each CTA owns one active 128-row block and keeps its score-band tile
//     (128 x Wf fp32) resident in SMEM for all T+R steps when the compacted
//     active-block list fits the co-resident grid (config 2: ~390 blocks x
//     66 KB <= 148 SMs x 3 CTAs); otherwise the same kernel re-streams each
//     tile every step (bulk copy), several tiles per CTA;
//   * per step: combine the column partials of the previous step (fixed block
//     order) into v_{t-1} on the block window, row pass u_t (one exp per
//     cell), column pass partials sum_i 2^(s2 + u_t + v_{t-1}) (a second exp
//     per cell -- the tile stays intact), then one grid barrier;
//   * u_t is kept by the row's thread (ubuf), v_t by the owner block (vbuf),
//     written every step so the non-resident mode and the saved slots share
//     one code path.
// Results are identical to the per-step k_fstep launches up to fp32 rounding
// of e/r vs 2^(s2+u+v).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "st_common.cuh"
#include "st_kernels.cuh"
#include "st_phase.cuh"
#include "st_sm100.cuh"

namespace st {

namespace {

constexpr int kThreads = 256;

using u64 = unsigned long long;

struct FSolve {
    const float* S2;
    float* ubuf;             // [BH][Lrq] raw base-2 u (final step; every step when non-resident)
    float* vbuf;             // [BH][Lrk] v_{T+R} (owners)
    float* u_slot[9];        // saved u at tail steps T .. T+8 (or null)
    float* v_slot[9];
    u64* part[2];            // [BH][NB][Nw] tagged column partials {sum, step}, by step parity
    u64* partm;              // [BH][NB][Nw] tagged cold-start maxima {max, 1}
    float* vpriv;            // [n][Nw] window duals of each work item (non-resident mode only)
    const int* flags;        // [BH][NB] 1 = block is in the work list
    const int* work;         // compacted active blocks, bh * NB + b
    const int* nwork;
    int NB, Nw, T, R;
    int nst;                 // epsilon stages (run-length over the base steps): step t <= st_end[q] -> st_scale[q]
    int st_end[8];
    float st_scale[8];
    int* err;
};

__device__ __forceinline__ void st_tagged(u64* p, float v, unsigned tag) {
    const u64 x = ((u64)tag << 32) | (u64)__float_as_uint(v);
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(x) : "memory");
}
__device__ __forceinline__ u64 ld_tagged(const u64* p) {
    u64 x;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(x) : "l"(p) : "memory");
    return x;
}
__device__ __forceinline__ float tag_value(u64 x) { return __uint_as_float((unsigned)x); }

// The tagged partials of window column c of block b from the (active) blocks
// b-2 .. b+2 for step `want`, spinning only on entries not yet published.
__device__ __forceinline__ void gather5(const FSolve& f, const u64* buf, int bh, int b, int c, unsigned want,
                                       float out[5]) {
    const u64* p[5];
    bool ok[5];
    u64 x[5];
#pragma unroll
    for (int d = 0; d < 5; ++d) {
        const int bb = b - 2 + d;
        const int cc = c + 128 * (2 - d);
        ok[d] = bb >= 0 && bb < f.NB && cc >= 0 && cc < f.Nw && f.flags[bh * f.NB + bb] != 0;
        p[d] = buf + ((size_t)bh * f.NB + (ok[d] ? bb : 0)) * f.Nw + (ok[d] ? cc : 0);
        x[d] = ok[d] ? ld_tagged(p[d]) : ((u64)want << 32);
    }
#pragma unroll
    for (int d = 0; d < 5; ++d) {
        while ((unsigned)(x[d] >> 32) != want) x[d] = ld_tagged(p[d]);
        out[d] = ok[d] ? tag_value(x[d]) : 0.f;
    }
}

// v_{t-1} of window column c (cold-start pairs at t = 2)
__device__ __forceinline__ float combine(const FSolve& f, int bh, int b, int c, int t, float prev) {
    float pv[5];
    gather5(f, f.part[(t - 1) & 1], bh, b, c, (unsigned)(t - 1), pv);
    if (t == 2) {
        float pm[5];
        gather5(f, f.partm, bh, b, c, 1u, pm);
        float M = -INFINITY;
#pragma unroll
        for (int d = 0; d < 5; ++d)
            if (pv[d] > 0.f) M = fmaxf(M, pm[d]);
        float sum = 0.f;
#pragma unroll
        for (int d = 0; d < 5; ++d)
            if (pv[d] > 0.f) sum += pv[d] * ex2(pm[d] - M);
        return -(M + lg2(sum));
    }
    float sum = 0.f;
#pragma unroll
    for (int d = 0; d < 5; ++d) sum += pv[d];
    return prev - lg2(sum);
}

__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {  // FADD2 (packed fp32, sm_100)
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
__device__ __forceinline__ float2 ex2x2(float2 x) { return make_float2(ex2(x.x), ex2(x.y)); }

// score scale of full step t: the band is stored at the final temperature; base step t of an
// EpsSchedule stage runs at that stage's (scale_to_temperature, sinkhorn.hpp:186-195); tail: 1
template <class F>
__device__ __forceinline__ float stage_scale(const F& f, int t) {
    if (t > f.T) return 1.f;
    float lam = 1.f;
    for (int q = f.nst - 1; q >= 0; --q)
        if (t <= f.st_end[q]) lam = f.st_scale[q];
    return lam;
}
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {  // FFMA2 (packed fp32, sm_100)
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "mov.b64 rc, {%6, %7};\n\tfma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}

// SMEM geometry: tile [128][P] (P = Wf + 1, even: 8-byte aligned rows, half-warp
// LDS.64 conflict free), the window duals twice (shift 0 / 1, so every row reads
// aligned pairs), column-pass halves.
struct FsGeo {
    int P, P2;
    __host__ __device__ FsGeo(int Wf, int Nw) : P(Wf + 1), P2(((Nw + 2 + 31) / 32) * 32 + 16) {}
    __host__ __device__ size_t floats(int Nw) const { return (size_t)128 * P + 2 * (size_t)P2 + 4 * (size_t)Nw; }
};

__global__ void __launch_bounds__(kThreads) k_fsolve(Geo g, FSolve f) {
    extern __shared__ __align__(16) float smf[];
    __shared__ __align__(8) float unew[128];
    const int Wf = g.Wf, Nw = f.Nw, tid = threadIdx.x;
    const FsGeo sg(Wf, Nw);
    const int P = sg.P;
    const int lane = tid & 31, h = lane >> 4, r = (tid >> 5) * 16 + (lane & 15);
    const unsigned pmask = (1u << (lane & 15)) | (1u << ((lane & 15) + 16));
    float* tile = smf;                    // [128][P] s2 (never overwritten), pad column = -inf
    float* vw0 = smf + 128 * P;           // [P2] v_{t-1}(c)
    float* vw1 = vw0 + sg.P2;             // [P2] v_{t-1}(c + 1)
    float* csum = vw1 + sg.P2;            // [2][Nw]
    float* cmax = csum + 2 * Nw;          // [2][Nw]
    const int n = *f.nwork;
    const int G = gridDim.x;
    const bool resident = n <= G;
    const int TR = f.T + f.R;
    for (int x = tid; x < sg.P2; x += kThreads) {
        if (x >= Nw) vw0[x] = -INFINITY;
        if (x >= Nw - 1) vw1[x] = -INFINITY;
    }
    // step-invariant per-thread state (resident mode keeps it across steps)
    bool con[2] = {false, false}, act = false;
    float ureg = 0.f;
    for (int t = 1; t <= TR + 1; ++t) {
        const bool fin = t == TR + 1;  // final combine only (v_{T+R})
        for (int k = blockIdx.x; k < n; k += G) {
            const int blk = f.work[k];
            const int bh = blk / f.NB, b = blk % f.NB, i0 = b * 128;
            const bool need_load = !fin && (!resident || t == 1);
            if (need_load) {  // re-pitch the band tile Wf -> P (once when resident)
                const float* src = f.S2 + ((size_t)bh * g.Lqp + i0) * Wf;
                for (int e = tid; e < 128 * Wf; e += kThreads) {
                    const int rr = e / Wf;
                    tile[rr * P + (e - rr * Wf)] = (i0 + rr < g.Lq) ? __ldcs(src + e) : -INFINITY;  // pad rows unwritten
                }
                for (int rr = tid; rr < 128; rr += kThreads) tile[rr * P + Wf] = -INFINITY;
            }
            const int i = i0 + r;
            if (!resident || t == 1) {
                const uint8_t* rmask = g.row_mask ? g.row_mask + (size_t)(bh / g.H) * g.Lq : nullptr;
                const uint8_t* cmask = g.col_mask ? g.col_mask + (size_t)(bh / g.H) * g.Lk : nullptr;
                act = i < g.Lq && (rmask == nullptr || rmask[i] != 0);
#pragma unroll
                for (int a = 0; a < 2; ++a) {
                    const int j = i0 - g.w + tid + kThreads * a;
                    con[a] = tid + kThreads * a < Nw && j >= 0 && j < g.Lk && (cmask == nullptr || cmask[j] != 0);
                }
                if (!resident && t >= 2 && act) ureg = f.ubuf[(size_t)bh * g.Lrq + i];
            }
            // ---- combine: v_{t-1} on the window; owners publish their 128 columns
#pragma unroll
            for (int a = 0; a < 2; ++a) {
                const int c = tid + kThreads * a;
                if (c >= Nw) break;
                const int j = i0 - g.w + c;
                const bool owner = c >= g.w && c < g.w + 128 && j < g.Lk;
                if (fin && !owner) continue;
                float v = -INFINITY;
                if (t == 1) {
                    if (con[a]) v = 0.f;
                } else if (con[a]) {
                    const float prev = (t < 3) ? 0.f : resident ? vw0[c] : f.vpriv[(size_t)k * Nw + c];
                    v = combine(f, bh, b, c, t, prev);
                    if (!isfinite(v)) {
                        atomicOr(f.err, 32);
                        v = 0.f;
                    }
                }
                if (!fin) {
                    vw0[c] = v;
                    if (c >= 1) vw1[c - 1] = v;
                }
                if (!resident) f.vpriv[(size_t)k * Nw + c] = v;
                if (t >= 2 && owner) {
                    const float vo = (v == -INFINITY) ? 0.f : v;
                    const int rv = t - 1 - f.T;
                    if (rv >= 0 && rv <= 8 && f.v_slot[rv]) f.v_slot[rv][(size_t)bh * g.Lrk + j] = vo;
                    if (fin) f.vbuf[(size_t)bh * g.Lrk + j] = vo;
                }
            }
            if (fin) continue;
            __syncthreads();
            const float lam = stage_scale(f, t);
            const float2 ll = make_float2(lam, lam);
            // ---- row pass: threads (r, h) share row i; h takes the 16-cell groups h, h+2, ...
            const float* trow = tile + r * P;
            const float* vrow = ((r & 1) ? vw1 : vw0) + (r & ~1);  // vrow[k] = v(r + k), k even aligned
            if (act) {
                float o;
                if (t == 1) {
                    float m = -INFINITY;
                    for (int k0 = 16 * h; k0 < P; k0 += 32)
#pragma unroll
                        for (int kk = 0; kk < 16; ++kk)
                            if (k0 + kk < P) m = fmaxf(m, fmaf(trow[k0 + kk], lam, vrow[k0 + kk]));
                    m = fmaxf(m, __shfl_xor_sync(pmask, m, 16));
                    o = -m;
                } else {
                    o = ureg;
                }
                const float2 oo = make_float2(o, o);
                float2 a0 = make_float2(0.f, 0.f), a1 = a0;
                for (int k0 = 16 * h; k0 < P; k0 += 32) {
                    if (k0 + 16 <= P) {
#pragma unroll
                        for (int kk = 0; kk < 16; kk += 4) {
                            const float2 sa = *reinterpret_cast<const float2*>(trow + k0 + kk);
                            const float2 sb = *reinterpret_cast<const float2*>(trow + k0 + kk + 2);
                            const float2 va = *reinterpret_cast<const float2*>(vrow + k0 + kk);
                            const float2 vb = *reinterpret_cast<const float2*>(vrow + k0 + kk + 2);
                            a0 = fadd2(a0, ex2x2(fadd2(ffma2(sa, ll, va), oo)));
                            a1 = fadd2(a1, ex2x2(fadd2(ffma2(sb, ll, vb), oo)));
                        }
                    } else {
                        for (int kx = k0; kx < P; kx += 2) {
                            const float2 sa = *reinterpret_cast<const float2*>(trow + kx);
                            const float2 va = *reinterpret_cast<const float2*>(vrow + kx);
                            a0 = fadd2(a0, ex2x2(fadd2(ffma2(sa, ll, va), oo)));
                        }
                    }
                }
                float rs = (a0.x + a0.y) + (a1.x + a1.y);
                rs += __shfl_xor_sync(pmask, rs, 16);
                float u = o - lg2(rs);
                if (!(rs > 0.f) || !isfinite(u)) {
                    if (h == 0) atomicOr(f.err, 64);
                    u = 0.f;
                }
                ureg = u;
                if (h == 0) {
                    unew[r] = u;
                    if (!resident || t == TR) f.ubuf[(size_t)bh * g.Lrq + i] = u;
                    const int ru = t - f.T;
                    if (ru >= 0 && ru <= 8 && f.u_slot[ru]) f.u_slot[ru][(size_t)bh * g.Lrq + i] = u;
                }
            } else if (h == 0) {
                unew[r] = -INFINITY;  // no contribution to any column
            }
            __syncthreads();
            // ---- column pass.  Thread t7 = tid & 127 owns the window columns {t7 + 128 m}:
            // exactly Wf cells for every t7 (balanced lanes); the thread pair hh = tid >> 7
            // splits that concatenated cell list at Wf/2 and the halves are combined in
            // a fixed order through SMEM.  Cell (ii, c) sits at ii * (P - 1) + c.
            {
                const int t7 = tid & 127, hh = tid >> 7;
                const int half = (Wf + 1) >> 1;
                const int beg = hh ? half : 0, end = hh ? Wf : half;
                const int step = P - 1;
                int off = 0;
                for (int c = t7; c < Nw; c += 128) {
                    const int lo = max(0, c - 2 * g.w), hi = min(127, c);
                    const int n_c = hi - lo + 1;
                    const int a0 = max(beg, off), a1 = min(end, off + n_c);  // my slice of this column
                    const int ilo = lo + (a0 - off), ihi = lo + (a1 - off) - 1;
                    off += n_c;
                    const float vc = vw0[c];
                    float ps = 0.f, pm = -INFINITY;
                    if (ilo <= ihi) {
                        const float* tp = tile + ilo * step + c;
                        if (t == 1) {
                            for (int ii = ilo; ii <= ihi; ++ii) pm = fmaxf(pm, fmaf(tp[(ii - ilo) * step], lam, unew[ii]));
                            if (pm != -INFINITY)
                                for (int ii = ilo; ii <= ihi; ++ii) ps += ex2(fmaf(tp[(ii - ilo) * step], lam, unew[ii]) - pm);
                        } else if (vc != -INFINITY) {
                            const float2 vv = make_float2(vc, vc);
                            float2 q0 = make_float2(0.f, 0.f), q1 = q0;
                            int ii = ilo;
                            if (ii & 1) {  // align the unew pairs
                                q0.x += ex2(fmaf(tp[0], lam, unew[ii]) + vc);
                                ++ii;
                                tp += step;
                            }
                            for (; ii + 3 <= ihi; ii += 4, tp += 4 * step) {
                                const float2 ua = *reinterpret_cast<const float2*>(unew + ii);
                                const float2 ub = *reinterpret_cast<const float2*>(unew + ii + 2);
                                q0 = fadd2(q0, ex2x2(ffma2(make_float2(tp[0], tp[step]), ll, fadd2(ua, vv))));
                                q1 = fadd2(q1, ex2x2(ffma2(make_float2(tp[2 * step], tp[3 * step]), ll, fadd2(ub, vv))));
                            }
                            for (; ii <= ihi; ++ii, tp += step) q1.x += ex2(fmaf(tp[0], lam, unew[ii]) + vc);
                            ps = (q0.x + q0.y) + (q1.x + q1.y);
                        }
                    }
                    csum[hh * Nw + c] = ps;
                    if (t == 1) cmax[hh * Nw + c] = pm;
                }
            }
            __syncthreads();
            {
                u64* pout = f.part[t & 1] + ((size_t)bh * f.NB + b) * Nw;
                for (int c = tid; c < Nw; c += kThreads) {
                    const float s0 = csum[c], s1 = csum[Nw + c];
                    if (t == 1) {
                        const float m0 = cmax[c], m1 = cmax[Nw + c];
                        const float M = fmaxf(m0, m1);
                        float sum = 0.f;
                        if (M != -INFINITY) {
                            if (m0 != -INFINITY) sum += s0 * ex2(m0 - M);
                            if (m1 != -INFINITY) sum += s1 * ex2(m1 - M);
                        }
                        st_tagged(f.partm + ((size_t)bh * f.NB + b) * Nw + c, M, 1u);
                        st_tagged(pout + c, sum, 1u);
                    } else {
                        st_tagged(pout + c, s0 + s1, (unsigned)t);
                    }
                }
            }
            __syncthreads();  // tile / unew / vw reuse by the next tile of this CTA
        }
    }
}

// ---------------------------------------------------------------------------
// TMEM-resident variant (bands up to Wf = 129): the score cells k < 128 of the
// 128-row tile live in Tensor Memory (128 columns per CTA, row = TMEM lane,
// three CTAs per SM use 384 of the 512 columns; the cell k = 128 of a w = 64
// band stays in SMEM), so SMEM is free to hold the row-pass exponentials and
// the column pass reuses them: ONE exp per cell per full step
// (sum_i e_ij / r_i = sum_i 2^(s2 + u_t,i + v_{t-1},j)).
// Warp w reads its TMEM lane quarter: row r = 32 (w & 3) + lane, and warps w,
// w + 4 split the row's columns [0, 64) / [64, 128) (+ the SMEM cell).
// ---------------------------------------------------------------------------
constexpr int kTmCols = 128;
constexpr int kTmGroups = 3;  // tiles (warp groups) per CTA: 3 x 128 TMEM columns

struct TmGeo {
    int P, P2;
    // pitch 130 for every Wf <= 129: the row pass writes all 128 TMEM cells (+1), 8-byte aligned rows.
    // The row pass reads the window duals of all 128 TMEM cells of its row (vw[r + k], k < 128) even
    // when the band is narrower, so the -inf-filled window vectors span at least 2 * 128 entries.
    __host__ __device__ TmGeo(int Wf, int Nw)
        : P(kTmCols + 2), P2(max(((Nw + 2 + 31) / 32) * 32, 2 * kTmCols + 2) + 16) { (void)Wf; }
    // e tile [128][P] | extra cells [128] | vw0 [P2] | vw1 [P2] | csum [2][Nw] | cmax [2][Nw]
    __host__ __device__ size_t floats(int Nw) const { return (size_t)128 * P + 128 + 2 * (size_t)P2 + 4 * (size_t)Nw; }
};

__global__ void __launch_bounds__(kTmGroups * kThreads, 1) k_fsolve_tm(Geo g, FSolve f) {
    extern __shared__ __align__(16) float smf[];
    __shared__ __align__(8) float inv_r_all[kTmGroups][128];  // 1 / r_i (t >= 2) or lg2 r_i (cold start)
    __shared__ float rpart_all[kTmGroups][2][128];            // per-half row sums / maxima
    __shared__ uint32_t tmem_base;
    // one CTA per SM, kTmGroups independent warp groups of 256 threads, one band tile each
    const int grp = threadIdx.x / kThreads, tid = threadIdx.x % kThreads;
    float* inv_r = inv_r_all[grp];
    float(*rpart)[128] = rpart_all[grp];
    auto gsync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(kThreads) : "memory"); };
    const int Wf = g.Wf, Nw = f.Nw;
    const TmGeo sg(Wf, Nw);
    const int P = sg.P;
    const int wq = (tid >> 5) & 3, hh = tid >> 7, lane = tid & 31;
    const int r = 32 * wq + lane;
    float* et = smf + (size_t)grp * sg.floats(Nw);  // [128][P]: s2 staging, then e (or x at the cold start)
    float* extra = et + 128 * P;           // [128] cell k = 128 (Wf = 129)
    float* vw0 = extra + 128;              // [P2] v_{t-1}(c)
    float* vw1 = vw0 + sg.P2;              // [P2] v_{t-1}(c + 1)
    float* csum = vw1 + sg.P2;             // [2][Nw]
    float* cmax = csum + 2 * Nw;           // [2][Nw]
    const int n = *f.nwork;
    const int G = gridDim.x * kTmGroups;  // tile slots
    const int slot = blockIdx.x * kTmGroups + grp;
    const bool resident = n <= G;
    const int TR = f.T + f.R;
    const int kt = Wf < kTmCols ? Wf : kTmCols;  // cells held in TMEM
    if (threadIdx.x < 32) {
        sm100::tc_alloc(&tmem_base, 512);
        sm100::tc_relinquish();
    }
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
    const uint32_t trow = tmem_base + ((uint32_t)(32 * wq) << 16) + (uint32_t)(kTmCols * grp);  // lane quarter
    for (int x = tid; x < sg.P2; x += kThreads) {
        if (x >= Nw) vw0[x] = -INFINITY;
        if (x >= Nw - 1) vw1[x] = -INFINITY;
    }
    bool con[2] = {false, false}, act = false;
    float ureg = 0.f;
    for (int t = 1; t <= TR + 1; ++t) {
        const bool fin = t == TR + 1;
        for (int k = slot; k < n; k += G) {
            const int blk = f.work[k];
            const int bh = blk / f.NB, b = blk % f.NB, i0 = b * 128;
            const bool need_load = !fin && (!resident || t == 1);
            if (need_load) {  // stage the band tile in SMEM, then move cells k < 128 into TMEM
                const float* src = f.S2 + ((size_t)bh * g.Lqp + i0) * Wf;
                for (int e = tid; e < 128 * Wf; e += kThreads) {
                    const int rr = e / Wf;
                    et[rr * P + (e - rr * Wf)] = (i0 + rr < g.Lq) ? __ldcs(src + e) : -INFINITY;  // pad rows unwritten
                }
                gsync();
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const int c0 = 64 * hh + 32 * q;
                    float vv[32];
#pragma unroll
                    for (int x = 0; x < 32; ++x) vv[x] = (c0 + x < kt) ? et[r * P + c0 + x] : -INFINITY;
                    sm100::tc_st32(trow + (uint32_t)c0, vv);
                }
                if (hh == 0) extra[r] = (Wf > kTmCols) ? et[r * P + kTmCols] : -INFINITY;
                sm100::tc_wait_st();
            }
            const int i = i0 + r;
            if (!resident || t == 1) {
                const uint8_t* rmask = g.row_mask ? g.row_mask + (size_t)(bh / g.H) * g.Lq : nullptr;
                const uint8_t* cmask = g.col_mask ? g.col_mask + (size_t)(bh / g.H) * g.Lk : nullptr;
                act = i < g.Lq && (rmask == nullptr || rmask[i] != 0);
#pragma unroll
                for (int a = 0; a < 2; ++a) {
                    const int j = i0 - g.w + tid + kThreads * a;
                    con[a] = tid + kThreads * a < Nw && j >= 0 && j < g.Lk && (cmask == nullptr || cmask[j] != 0);
                }
                if (!resident && t >= 2 && act) ureg = f.ubuf[(size_t)bh * g.Lrq + i];
            }
            // ---- combine: v_{t-1} on the window; owners publish their 128 columns
#pragma unroll
            for (int a = 0; a < 2; ++a) {
                const int c = tid + kThreads * a;
                if (c >= Nw) break;
                const int j = i0 - g.w + c;
                const bool owner = c >= g.w && c < g.w + 128 && j < g.Lk;
                if (fin && !owner) continue;
                float v = -INFINITY;
                if (t == 1) {
                    if (con[a]) v = 0.f;
                } else if (con[a]) {
                    const float prev = (t < 3) ? 0.f : resident ? vw0[c] : f.vpriv[(size_t)k * Nw + c];
                    v = combine(f, bh, b, c, t, prev);
                    if (!isfinite(v)) {
                        atomicOr(f.err, 32);
                        v = 0.f;
                    }
                }
                if (!fin) {
                    vw0[c] = v;
                    if (c >= 1) vw1[c - 1] = v;
                }
                if (!resident) f.vpriv[(size_t)k * Nw + c] = v;
                if (t >= 2 && owner) {
                    const float vo = (v == -INFINITY) ? 0.f : v;
                    const int rv = t - 1 - f.T;
                    if (rv >= 0 && rv <= 8 && f.v_slot[rv]) f.v_slot[rv][(size_t)bh * g.Lrk + j] = vo;
                    if (fin) f.vbuf[(size_t)bh * g.Lrk + j] = vo;
                }
            }
            if (fin) continue;
            gsync();
            // ---- row pass: half hh of row r -- TMEM cells [64 hh, 64 hh + 64) (+ the SMEM cell for hh = 1)
            const float* vrow = ((r & 1) ? vw1 : vw0) + (r & ~1);  // vrow[k] = v(r + k), k even aligned
            float* erow = et + r * P;
            float o = 0.f;
            const float lam = stage_scale(f, t);
            const float2 ll = make_float2(lam, lam);
            // tcgen05.ld is warp-collective (.sync.aligned): every lane loads (one 32-column chunk
            // at a time), inactive rows only mask the math
            if (t == 1) {  // cold start: row max of s2 + v over both halves
                float m = -INFINITY;
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    float sv[32];
                    sm100::tc_ld32(trow + (uint32_t)(64 * hh + 32 * q), sv);
                    sm100::tc_wait_ld();
                    if (act) {
#pragma unroll
                        for (int x = 0; x < 32; ++x) m = fmaxf(m, fmaf(sv[x], lam, vrow[64 * hh + 32 * q + x]));
                    }
                }
                if (act && hh == 1) m = fmaxf(m, fmaf(extra[r], lam, vrow[kTmCols]));
                rpart[hh][r] = m;
                gsync();
                o = -fmaxf(rpart[0][r], rpart[1][r]);
                gsync();
            } else {
                o = ureg;
            }
            float2 a0 = make_float2(0.f, 0.f), a1 = a0;
            const float2 oo = make_float2(o, o);
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int c0 = 64 * hh + 32 * q;
                float sv[32];
                sm100::tc_ld32(trow + (uint32_t)c0, sv);
                sm100::tc_wait_ld();
                if (act) {
#pragma unroll
                    for (int x = 0; x < 32; x += 4) {
                        const float2 va = *reinterpret_cast<const float2*>(vrow + c0 + x);
                        const float2 vb = *reinterpret_cast<const float2*>(vrow + c0 + x + 2);
                        const float2 xa = fadd2(ffma2(make_float2(sv[x], sv[x + 1]), ll, va), oo);
                        const float2 xb = fadd2(ffma2(make_float2(sv[x + 2], sv[x + 3]), ll, vb), oo);
                        const float2 ea = ex2x2(xa), eb = ex2x2(xb);
                        a0 = fadd2(a0, ea);
                        a1 = fadd2(a1, eb);
                        *reinterpret_cast<float2*>(erow + c0 + x) = (t == 1) ? xa : ea;
                        *reinterpret_cast<float2*>(erow + c0 + x + 2) = (t == 1) ? xb : eb;
                    }
                } else {  // inactive row: contributes nothing to any column
                    const float z = (t == 1) ? -INFINITY : 0.f;
#pragma unroll
                    for (int x = 0; x < 32; ++x) erow[c0 + x] = z;
                }
            }
            if (hh == 1) {
                if (act && Wf > kTmCols) {
                    const float x = fmaf(extra[r], lam, vrow[kTmCols]) + o;
                    const float e = ex2(x);
                    a0.x += e;
                    erow[kTmCols] = (t == 1) ? x : e;
                } else if (!act) {
                    erow[kTmCols] = (t == 1) ? -INFINITY : 0.f;
                }
            }
            rpart[hh][r] = (a0.x + a0.y) + (a1.x + a1.y);
            gsync();
            if (hh == 0) {
                if (act) {
                    const float rs = rpart[0][r] + rpart[1][r];
                    const float lr = lg2(rs);
                    float u = o - lr;
                    if (!(rs > 0.f) || !isfinite(u)) {
                        atomicOr(f.err, 64);
                        u = 0.f;
                    }
                    inv_r[r] = (t == 1) ? lr : 1.f / rs;
                    if (!resident || t == TR) f.ubuf[(size_t)bh * g.Lrq + i] = u;
                    const int ru = t - f.T;
                    if (ru >= 0 && ru <= 8 && f.u_slot[ru]) f.u_slot[ru][(size_t)bh * g.Lrq + i] = u;
                    rpart[0][r] = u;  // hand the new dual to the other half
                } else {
                    inv_r[r] = (t == 1) ? INFINITY : 0.f;
                }
            }
            gsync();
            if (act) ureg = rpart[0][r];
            // ---- column pass over the stored exponentials.  Thread t7 = tid & 127 owns the
            // window columns {t7 + 128 m} (Wf cells for every t7); the thread pair hh splits
            // that list at Wf/2, halves combined in a fixed order.  Cell (ii, c) at ii (P-1) + c.
            {
                const int t7 = tid & 127;
                const int half = (Wf + 1) >> 1;
                const int beg = hh ? half : 0, end = hh ? Wf : half;
                const int step = P - 1;
                int off = 0;
                for (int c = t7; c < Nw; c += 128) {
                    const int lo = max(0, c - 2 * g.w), hi = min(127, c);
                    const int n_c = hi - lo + 1;
                    const int x0 = max(beg, off), x1 = min(end, off + n_c);
                    const int ilo = lo + (x0 - off), ihi = lo + (x1 - off) - 1;
                    off += n_c;
                    float ps = 0.f, pm = -INFINITY;
                    if (ilo <= ihi) {
                        const float* tp = et + ilo * step + c;
                        if (t == 1) {
                            for (int ii = ilo; ii <= ihi; ++ii) pm = fmaxf(pm, tp[(ii - ilo) * step] - inv_r[ii]);
                            if (pm != -INFINITY)
                                for (int ii = ilo; ii <= ihi; ++ii) ps += ex2(tp[(ii - ilo) * step] - inv_r[ii] - pm);
                        } else {  // row pairs: FFMA2 with an aligned LDS.64 of inv_r
                            float2 q0 = make_float2(0.f, 0.f), q1 = q0;
                            int ii = ilo;
                            if (ii & 1) {
                                q0.x = fmaf(tp[0], inv_r[ii], q0.x);
                                ++ii;
                                tp += step;
                            }
                            for (; ii + 3 <= ihi; ii += 4, tp += 4 * step) {
                                const float2 ia = *reinterpret_cast<const float2*>(inv_r + ii);
                                const float2 ib = *reinterpret_cast<const float2*>(inv_r + ii + 2);
                                q0 = ffma2(make_float2(tp[0], tp[step]), ia, q0);
                                q1 = ffma2(make_float2(tp[2 * step], tp[3 * step]), ib, q1);
                            }
                            for (; ii <= ihi; ++ii, tp += step) q1.x = fmaf(tp[0], inv_r[ii], q1.x);
                            ps = (q0.x + q0.y) + (q1.x + q1.y);
                        }
                    }
                    csum[hh * Nw + c] = ps;
                    if (t == 1) cmax[hh * Nw + c] = pm;
                }
            }
            gsync();
            {
                u64* pout = f.part[t & 1] + ((size_t)bh * f.NB + b) * Nw;
                for (int c = tid; c < Nw; c += kThreads) {
                    const float s0 = csum[c], s1 = csum[Nw + c];
                    if (t == 1) {
                        const float m0 = cmax[c], m1 = cmax[Nw + c];
                        const float M = fmaxf(m0, m1);
                        float sum = 0.f;
                        if (M != -INFINITY) {
                            if (m0 != -INFINITY) sum += s0 * ex2(m0 - M);
                            if (m1 != -INFINITY) sum += s1 * ex2(m1 - M);
                        }
                        st_tagged(f.partm + ((size_t)bh * f.NB + b) * Nw + c, M, 1u);
                        st_tagged(pout + c, sum, 1u);
                    } else {
                        st_tagged(pout + c, s0 + s1, (unsigned)t);
                    }
                }
            }
            if (!resident) gsync();  // the next tile of this group restages the SMEM tile
        }
    }
    sm100::tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) sm100::tc_dealloc(tmem_base, 512);
}

// blocks with any active row or any active column (their owner duties)
__global__ void k_fs_flags(Geo g, int NB, int* __restrict__ flags) {
    const int bh = blockIdx.y, b = blockIdx.x;
    const int x = b * 128 + threadIdx.x;
    int any = 0;
    if (x < g.Lq && row_on(g, bh, x)) any = 1;
    if (x < g.Lk && col_on(g, bh, x)) any = 1;
    any = __syncthreads_or(any);
    if (threadIdx.x == 0) flags[bh * NB + b] = any;
}

}  // namespace

static bool use_tmem(const Geo& g) {
    const int Nw = 128 + 2 * g.w;
    return g.Wf <= kTmCols + 1 && kTmGroups * TmGeo(g.Wf, Nw).floats(Nw) * 4 <= 220 * 1024 && !getenv("ST_NO_TMEM");
}

size_t fsolve_smem_bytes(const Geo& g) {
    const int Nw = 128 + 2 * g.w;
    return FsGeo(g.Wf, Nw).floats(Nw) * 4;  // the SMEM-only variant (eligibility check)
}

bool fsolve_supported(const Geo& g) {
    return !g.dustbin && g.Lq == g.Lk && g.w <= 128 && fsolve_smem_bytes(g) <= 227 * 1024;
}

cudaError_t launch_fsolve(const Geo& g, int T, int R, const FSolvePtrs& p, cudaStream_t s) {
    const int NB = (g.Lq + 127) / 128, Nw = 128 + 2 * g.w;
    const bool tm = use_tmem(g);
    const size_t smem = tm ? kTmGroups * TmGeo(g.Wf, Nw).floats(Nw) * 4 : fsolve_smem_bytes(g);
    auto kern = tm ? k_fsolve_tm : k_fsolve;
    const int threads = tm ? kTmGroups * kThreads : kThreads;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0, dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const int G = tm ? std::min(per_sm * nsm, (g.BH * NB + kTmGroups - 1) / kTmGroups)
                     : std::min(per_sm * nsm, g.BH * NB);
    // work list: active blocks in (head, block) order
    k_fs_flags<<<dim3(NB, g.BH), 128, 0, s>>>(g, NB, p.flags);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if ((e = launch_compact(p.flags, g.BH * NB, p.work, p.count, s)) != cudaSuccess) return e;
    const size_t nq = sizeof(float) * (size_t)g.BH * g.Lrq, nk = sizeof(float) * (size_t)g.BH * g.Lrk;
    const size_t np = sizeof(u64) * (size_t)g.BH * NB * Nw;
    // tags must not survive from a previous call: step tags start at 1
    cudaMemsetAsync(p.part[0], 0, np, s);
    cudaMemsetAsync(p.part[1], 0, np, s);
    cudaMemsetAsync(p.partm, 0, np, s);
    cudaMemsetAsync(p.ubuf, 0, nq, s);
    cudaMemsetAsync(p.vbuf, 0, nk, s);
    for (int q = 0; q < 9; ++q) {
        if (p.u_slot[q]) cudaMemsetAsync(p.u_slot[q], 0, nq, s);
        if (p.v_slot[q]) cudaMemsetAsync(p.v_slot[q], 0, nk, s);
    }
    FSolve f;
    f.S2 = p.S2;
    f.ubuf = p.ubuf;
    f.vbuf = p.vbuf;
    for (int q = 0; q < 9; ++q) {
        f.u_slot[q] = p.u_slot[q];
        f.v_slot[q] = p.v_slot[q];
    }
    f.part[0] = (u64*)p.part[0];
    f.part[1] = (u64*)p.part[1];
    f.partm = (u64*)p.partm;
    f.vpriv = p.vpriv;
    f.flags = p.flags;
    f.work = p.work;
    f.nwork = p.count;
    f.NB = NB;
    f.Nw = Nw;
    f.T = T;
    f.R = R;
    f.err = p.err;
    f.nst = p.nst;
    for (int q = 0; q < 8; ++q) {
        f.st_end[q] = p.st_end[q];
        f.st_scale[q] = p.st_scale[q];
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;  // co-residency: CTAs wait on their neighbours' tags
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, g, f);
    if (tm && e != cudaSuccess) {  // co-residency refused: the SMEM-only variant
        cudaGetLastError();
        const size_t smem2 = FsGeo(g.Wf, Nw).floats(Nw) * 4;
        if ((e = cudaFuncSetAttribute(k_fsolve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2)) != cudaSuccess)
            return e;
        int ps2 = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps2, k_fsolve, kThreads, smem2);
        cfg.gridDim = dim3(std::min(std::max(ps2, 1) * nsm, g.BH * NB));
        cfg.dynamicSmemBytes = smem2;
        e = cudaLaunchKernelEx(&cfg, k_fsolve, g, f);
    }
    add_launches(3);
    return e;
}

}  // namespace st
