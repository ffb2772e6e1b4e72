// oracle_capi.cpp -- batched C entry points over the CPU restatement.
//
// TEST INFRASTRUCTURE ONLY (see sinktail_oracle.hpp header).  Loaded with
// ctypes by tests/ (as the parity checker) and by bench.py (cpu_baseline and
// --impl reference legs, as the timed reference CPU path).  The product never
// loads this library.
//
// One call runs, for every (b, h) head in [head_begin, head_end), exactly the
// reference's validation pipeline for this path
//   run_surrogate(...)  then  r2_backward(..., mode)
// (inc/validation.hpp:102-114), in f32 or f64, sharded over host threads like
// the reference CLI's parallel_for (proj/tools/sinktail_main.cpp:138-154).
#include <atomic>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "sinktail_oracle.hpp"

namespace {

thread_local std::string g_err;

enum : int {
    STOC_OK = 0,
    STOC_INVALID_ARGUMENT = 1,
    STOC_INFEASIBLE_SUPPORT = 2,
    STOC_INVALID_TEMPERATURE = 3,
    STOC_UNSUPPORTED_DEPTH = 4,
    STOC_SIZE_CAP_EXCEEDED = 6,
    STOC_INTERNAL = 99,
};

struct BatchArgs {
    std::int64_t B, H, L, d, half_band, T, R;
    double eps;
    int dustbin;
    double dustbin_cost;
    const double *Q, *K, *V, *G;
    const std::uint8_t *row_mask, *col_mask;
    int precision, mode, tile_block, centered;
    double *O, *dQ, *dK, *dV, *d_eps, *eta_v, *duals, *gauges;
    // EpsSchedule stages (trace.hpp:12-50); n_stages == 0 -> one stage at eps
    int n_stages = 0;
    const double* stage_eps = nullptr;
    const std::int64_t* stage_iters = nullptr;
    std::int64_t Lk = -1;  // key count (rectangular problems, no dustbin); -1: Lk = L
    double* eta_u = nullptr;              // base cotangent u part (u-bar^(0))
    double *cQ = nullptr, *cK = nullptr;  // base_solve_vjp of the adjoint's base cotangent (certificates)
};

template <class T>
void run_head(const BatchArgs& a, std::int64_t bh) {
    using namespace stoc;
    const std::int64_t b = bh / a.H;
    const std::int64_t L = a.L, Lr = a.L + (a.dustbin ? 1 : 0), d = a.d;
    const std::int64_t Lk = a.Lk < 0 ? L : a.Lk, Lrk = Lk + (a.dustbin ? 1 : 0);
    const size_t off = static_cast<size_t>(bh * Lr * d), offk = static_cast<size_t>(bh * Lrk * d);
    auto load = [&](const double* src, std::int64_t rows, size_t o) {
        Mat<T> m(rows, d);
        for (size_t k = 0; k < m.a.size(); ++k) m.a[k] = static_cast<T>(src[o + k]);
        return m;
    };
    Mat<T> Q = load(a.Q, Lr, off), K = load(a.K, Lrk, offk), V = load(a.V, Lrk, offk), G = load(a.G, Lr, off);
    std::vector<bool> rm, cm;
    if (a.row_mask) {
        rm.resize(static_cast<size_t>(L));
        for (std::int64_t i = 0; i < L; ++i) rm[static_cast<size_t>(i)] = a.row_mask[b * L + i] != 0;
    }
    if (a.col_mask) {
        cm.resize(static_cast<size_t>(Lk));
        for (std::int64_t j = 0; j < Lk; ++j) cm[static_cast<size_t>(j)] = a.col_mask[b * Lk + j] != 0;
    }
    SupportMask sup = a.dustbin ? spoke_dustbin_support(L, a.half_band, rm, cm)
                                : build_band_support(L, Lk, a.half_band, rm, cm);
    // linear loss: G zeroed on inactive rows (inc/loss.hpp:78-82)
    for (std::int64_t i = 0; i < Lr; ++i)
        if (!sup.row_active(i)) for (std::int64_t x = 0; x < d; ++x) G(i, x) = T(0);
    ConstantEdges<T> cst;
    const ConstantEdges<T>* pc = nullptr;
    if (a.dustbin) {
        cst.row = L;
        cst.col = L;
        cst.value = static_cast<T>(-a.dustbin_cost);
        pc = &cst;
    }
    auto sched = TileSchedule::build(sup, a.tile_block);
    EpsSchedule<T> es = EpsSchedule<T>::single(static_cast<T>(a.eps), a.T);
    if (a.n_stages > 0) {
        es.stages.clear();
        for (int q = 0; q < a.n_stages; ++q) es.stages.push_back({static_cast<T>(a.stage_eps[q]), a.stage_iters[q]});
        es.validate(a.T);
    }
    SurrogateRun<T> run = run_surrogate<T>(Q, K, V, sched, a.T, a.R, es, a.centered != 0, pc);
    for (size_t k = 0; k < run.output.a.size(); ++k) a.O[off + k] = static_cast<double>(run.output.a[k]);
    if (a.duals && Lk == L) {
        double* dp = a.duals + static_cast<size_t>(bh) * 6 * Lr;
        for (std::int64_t r = 0; r <= 2 && r <= a.R; ++r) {
            const auto& u = run.trace.tail_u(r);
            const auto& v = run.trace.tail_v(r);
            for (std::int64_t i = 0; i < Lr; ++i) dp[r * Lr + i] = static_cast<double>(u[static_cast<size_t>(i)]);
            for (std::int64_t j = 0; j < Lr; ++j) dp[(3 + r) * Lr + j] = static_cast<double>(v[static_cast<size_t>(j)]);
            if (a.gauges) a.gauges[bh * 3 + r] = static_cast<double>(run.trace.gauge(run.trace.tail_step(r)));
        }
    }
    if (a.dQ == nullptr) return;  // forward only
    // mode 0 / 1: r2_backward (OneReference / DirectFourPlan); mode 2: tail_adjoint_generic (any R)
    CotangentSet<T> c = (a.mode == 2)
                            ? tail_adjoint_generic<T>(run.scaled, run.trace, G, Q, K, V, pc)
                            : r2_backward<T>(run.scaled, run.trace, G, Q, K, V,
                                             a.mode == 1 ? BackwardMode::DirectFourPlan : BackwardMode::OneReference,
                                             pc);
    for (size_t k = 0; k < c.grad_q.a.size(); ++k) a.dQ[off + k] = static_cast<double>(c.grad_q.a[k]);
    for (size_t k = 0; k < c.grad_k.a.size(); ++k) {
        a.dK[offk + k] = static_cast<double>(c.grad_k.a[k]);
        a.dV[offk + k] = static_cast<double>(c.grad_v.a[k]);
    }
    if (a.d_eps) a.d_eps[bh] = static_cast<double>(c.d_eps);
    if (a.eta_v)
        for (std::int64_t j = 0; j < Lrk; ++j)
            a.eta_v[bh * Lrk + j] = static_cast<double>(c.base_v[static_cast<size_t>(j)]);
    if (a.eta_u)
        for (std::int64_t i = 0; i < Lr; ++i) a.eta_u[bh * Lr + i] = static_cast<double>(c.base_u[static_cast<size_t>(i)]);
    if (a.cQ) {  // certificates.hpp:112-118: c_R = base_solve_vjp(raw, trace, base_cotangent)
        BaseVjpResult<T> bv = base_solve_vjp<T>(run.raw, run.trace, c.base_u, c.base_v, Q, K);
        for (size_t k = 0; k < bv.grad_q.a.size(); ++k) a.cQ[off + k] = static_cast<double>(bv.grad_q.a[k]);
        for (size_t k = 0; k < bv.grad_k.a.size(); ++k) a.cK[offk + k] = static_cast<double>(bv.grad_k.a[k]);
    }
}

int classify(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const stoc::InfeasibleSupport*>(&e)) return STOC_INFEASIBLE_SUPPORT;
    if (dynamic_cast<const stoc::InvalidTemperature*>(&e)) return STOC_INVALID_TEMPERATURE;
    if (dynamic_cast<const stoc::UnsupportedDepth*>(&e)) return STOC_UNSUPPORTED_DEPTH;
    if (dynamic_cast<const stoc::SizeCapExceeded*>(&e)) return STOC_SIZE_CAP_EXCEEDED;
    if (dynamic_cast<const std::invalid_argument*>(&e)) return STOC_INVALID_ARGUMENT;
    return STOC_INTERNAL;
}

}  // namespace

extern "C" {

const char* stoc_last_error() { return g_err.c_str(); }

// Fill out[k] = scale * counter_normal(seed, tag, start + k), k < n (inc/rng.hpp:38-56).
void stoc_normal_fill(std::uint64_t seed, const char* tag, std::uint64_t start, std::int64_t n, double scale,
                      double* out) {
    const std::uint64_t base = stoc::fold_tag(seed, tag);
    for (std::int64_t k = 0; k < n; ++k)
        out[k] = scale * stoc::counter_normal_base(base, start + static_cast<std::uint64_t>(k));
}

// Fill out[k] = counter_uniform(fold_tag(seed, tag) + start + k), k < n (inc/rng.hpp:21-35).
void stoc_uniform_fill(std::uint64_t seed, const char* tag, std::uint64_t start, std::int64_t n, double* out) {
    const std::uint64_t base = stoc::fold_tag(seed, tag);
    for (std::int64_t k = 0; k < n; ++k) out[k] = stoc::counter_uniform(base + start + static_cast<std::uint64_t>(k));
}

std::int64_t stoc_banded_entry_count(std::int64_t L, std::int64_t w) { return stoc::banded_entry_count(L, w); }

// Batched reference path.  Tensors are [B, H, Lr, d] doubles (Lr = L + dustbin),
// masks [B, L] uint8 or NULL.  dQ == NULL runs the forward only.
int stoc_run_batch_sched(std::int64_t B, std::int64_t H, std::int64_t L, std::int64_t d, std::int64_t half_band,
                         std::int64_t T, std::int64_t R, double eps, int dustbin, double dustbin_cost,
                         const double* Q, const double* K, const double* V, const double* G,
                         const std::uint8_t* row_mask, const std::uint8_t* col_mask, int precision, int mode,
                         int tile_block, int centered, int nthreads, std::int64_t head_begin, std::int64_t head_end,
                         double* O, double* dQ, double* dK, double* dV, double* d_eps, double* eta_v, double* duals,
                         double* gauges, int n_stages, const double* stage_eps, const std::int64_t* stage_iters) {
    BatchArgs a{B,      H,        L,    d,       half_band, T,          R,        eps,  dustbin, dustbin_cost,
                Q,      K,        V,    G,       row_mask,  col_mask,   precision, mode, tile_block, centered,
                O,      dQ,       dK,   dV,      d_eps,     eta_v,      duals,    gauges};
    a.n_stages = n_stages;
    a.stage_eps = stage_eps;
    a.stage_iters = stage_iters;
    if (head_end < 0 || head_end > B * H) head_end = B * H;
    if (head_begin < 0) head_begin = 0;
    if (nthreads < 1) nthreads = 1;
    std::atomic<std::int64_t> next{head_begin};
    std::atomic<int> status{STOC_OK};
    std::string first_err;
    std::atomic<bool> err_taken{false};
    auto worker = [&]() {
        for (;;) {
            const std::int64_t bh = next.fetch_add(1);
            if (bh >= head_end || status.load() != STOC_OK) return;
            try {
                if (precision == 32) run_head<float>(a, bh);
                else run_head<double>(a, bh);
            } catch (const std::exception& e) {
                int code = classify(e);
                bool expected = false;
                if (err_taken.compare_exchange_strong(expected, true)) {
                    first_err = e.what();
                    status.store(code);
                }
                return;
            }
        }
    };
    std::vector<std::thread> pool;
    const int n = static_cast<int>(std::min<std::int64_t>(nthreads, head_end - head_begin));
    for (int t = 1; t < n; ++t) pool.emplace_back(worker);
    worker();
    for (auto& th : pool) th.join();
    if (status.load() != STOC_OK) g_err = first_err;
    return status.load();
}

// rectangular problems (L_q != L_k, no dustbin): Q, G [B*H][Lq][d]; K, V, dK, dV [B*H][Lk][d]
int stoc_run_batch_rect(std::int64_t B, std::int64_t H, std::int64_t Lq, std::int64_t Lk, std::int64_t d,
                        std::int64_t half_band, std::int64_t T, std::int64_t R, double eps, const double* Q,
                        const double* K, const double* V, const double* G, const std::uint8_t* row_mask,
                        const std::uint8_t* col_mask, int precision, int mode, int nthreads, double* O, double* dQ,
                        double* dK, double* dV, double* d_eps, double* eta_v) {
    BatchArgs a{B,    H,  Lq, d,  half_band, T,        R,        eps,  0,   0.0,     Q,       K,      V,      G,
                row_mask, col_mask, precision, mode, 128, 1, O, dQ, dK, dV, d_eps, eta_v, nullptr, nullptr};
    a.Lk = Lk;
    if (nthreads < 1) nthreads = 1;
    std::atomic<std::int64_t> next{0};
    std::atomic<int> status{STOC_OK};
    auto worker = [&]() {
        for (;;) {
            const std::int64_t bh = next.fetch_add(1);
            if (bh >= B * H || status.load() != STOC_OK) return;
            try {
                if (precision == 32) run_head<float>(a, bh);
                else run_head<double>(a, bh);
            } catch (const std::exception& e) {
                status.store(classify(e));
                return;
            }
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < std::min<std::int64_t>(nthreads, B * H); ++t) pool.emplace_back(worker);
    worker();
    for (auto& th : pool) th.join();
    return status.load();
}

// generic tail adjoint + base-solve VJP per head (the bias certificate's c_R, certificates.hpp:112-118)
int stoc_run_batch_cert(std::int64_t B, std::int64_t H, std::int64_t L, std::int64_t d, std::int64_t half_band,
                        std::int64_t T, std::int64_t R, double eps, const double* Q, const double* K,
                        const double* V, const double* G, const std::uint8_t* row_mask, const std::uint8_t* col_mask,
                        int precision, int nthreads, int n_stages, const double* stage_eps,
                        const std::int64_t* stage_iters, double* O, double* dQ, double* dK, double* dV,
                        double* d_eps, double* eta_u, double* eta_v, double* cQ, double* cK) {
    BatchArgs a{B,    H,  L, d,  half_band, T,        R,        eps,  0,   0.0,     Q,       K,      V,      G,
                row_mask, col_mask, precision, 2, 128, 1, O, dQ, dK, dV, d_eps, eta_v, nullptr, nullptr};
    a.n_stages = n_stages;
    a.stage_eps = stage_eps;
    a.stage_iters = stage_iters;
    a.cQ = cQ;
    a.cK = cK;
    a.eta_u = eta_u;
    if (nthreads < 1) nthreads = 1;
    std::atomic<std::int64_t> next{0};
    std::atomic<int> status{STOC_OK};
    auto worker = [&]() {
        for (;;) {
            const std::int64_t bh = next.fetch_add(1);
            if (bh >= B * H || status.load() != STOC_OK) return;
            try {
                if (precision == 32) run_head<float>(a, bh);
                else run_head<double>(a, bh);
            } catch (const std::exception& e) {
                status.store(classify(e));
                return;
            }
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < std::min<std::int64_t>(nthreads, B * H); ++t) pool.emplace_back(worker);
    worker();
    for (auto& th : pool) th.join();
    return status.load();
}

int stoc_run_batch(std::int64_t B, std::int64_t H, std::int64_t L, std::int64_t d, std::int64_t half_band,
                   std::int64_t T, std::int64_t R, double eps, int dustbin, double dustbin_cost, const double* Q,
                   const double* K, const double* V, const double* G, const std::uint8_t* row_mask,
                   const std::uint8_t* col_mask, int precision, int mode, int tile_block, int centered,
                   int nthreads, std::int64_t head_begin, std::int64_t head_end, double* O, double* dQ, double* dK,
                   double* dV, double* d_eps, double* eta_v, double* duals, double* gauges) {
    return stoc_run_batch_sched(B, H, L, d, half_band, T, R, eps, dustbin, dustbin_cost, Q, K, V, G, row_mask,
                                col_mask, precision, mode, tile_block, centered, nthreads, head_begin, head_end, O, dQ,
                                dK, dV, d_eps, eta_v, duals, gauges, 0, nullptr, nullptr);
}

}  // extern "C"
