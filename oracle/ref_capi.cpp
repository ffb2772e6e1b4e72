// oracle/ref_capi.cpp -- C entry point around the REFERENCE ITSELF (oracle/_ref).
//
// TEST INFRASTRUCTURE: compiled by oracle/Makefile (target `ref`) from the
// unmodified reference sources where they lie (/root/reference/proj/include,
// /root/reference/proj/src/support.cpp) against oracle/ref_shim/Eigen/Core (a
// minimal Eigen-API stand-in; Eigen3 is absent from this image) and the image's
// nlohmann json.hpp.  Output: oracle/_ref/libref.so (git-ignored).  No reference
// source is copied into this repository.
//
// Per head: build_band_support (src/support.cpp:111-117) -> TileSchedule::build
// (src/support.cpp:150) -> run_surrogate (inc/sinkhorn.hpp:288-302) ->
// r2_backward(run.scaled, run.trace, G, Q, K, V, mode) (inc/adjoint.hpp:232-373),
// the call sequence of validation::run_kernel_backward (inc/validation.hpp:102-114).
//
// The constant-cost spoke dustbin (config 3) has no reference hook (scores always
// come from QK^T, inc/score.hpp:57-59); it is expressed in reference semantics with
// SupportMask::explicit_edges plus two extra feature dims:
//   s = ((d+2)/d)^(1/4), q~_i = [s q_i, c, 0], k~_j = [s k_j, 0, 1],
//   q~_dust = [0, 0, -c sqrt(d+2)], k~_dust = [0, -sqrt(d+2), 1]
// so every base edge scores q.k/sqrt(d) and every dustbin edge -c; dQ_i = s dQ~_i[0:d].
#include <cmath>
#include <cstdint>
#include <exception>
#include <string>
#include <thread>
#include <atomic>
#include <vector>

#include "sinktail/adjoint.hpp"
#include "sinktail/sinkhorn.hpp"
#include "sinktail/support.hpp"

namespace {

thread_local std::string g_err;

struct Args {
    std::int64_t Lq, Lk, d, w, T, R;
    double eps;
    int dustbin;
    double dustbin_cost;
    const double *Q, *K, *V, *G;
    const std::uint8_t *row_mask, *col_mask;
    int mode, tile_block, centered;
    int n_stages;
    const double* stage_eps;
    const std::int64_t* stage_iters;
    double *O, *dQ, *dK, *dV, *eta_v, *duals, *gauges;
};

template <class T>
void run_head(const Args& a, std::int64_t h) {
    using namespace sinktail;
    const std::int64_t L = a.Lq, Lk = a.Lk, d = a.d;
    const std::int64_t Lr = L + a.dustbin, Lrk = Lk + a.dustbin;
    const std::int64_t dd = a.dustbin ? d + 2 : d;
    const double s = a.dustbin ? std::pow(double(d + 2) / double(d), 0.25) : 1.0;
    const double c = a.dustbin_cost, rt = std::sqrt(double(d + 2));
    const double* Qh = a.Q + h * Lr * d;
    const double* Kh = a.K + h * Lrk * d;
    const double* Vh = a.V + h * Lrk * d;
    const double* Gh = a.G + h * Lr * d;
    Matrix<T> Q = Matrix<T>::Zero(Lr, dd), K = Matrix<T>::Zero(Lrk, dd), V(Lrk, d), G(Lr, d);
    for (std::int64_t i = 0; i < Lr; ++i)
        for (std::int64_t x = 0; x < d; ++x) {
            if (i < L) Q(i, x) = static_cast<T>(s * Qh[i * d + x]);
            G(i, x) = static_cast<T>(Gh[i * d + x]);
        }
    for (std::int64_t j = 0; j < Lrk; ++j)
        for (std::int64_t x = 0; x < d; ++x) {
            if (j < Lk) K(j, x) = static_cast<T>(s * Kh[j * d + x]);
            V(j, x) = static_cast<T>(Vh[j * d + x]);
        }
    std::vector<bool> rm(static_cast<size_t>(Lr), true), cm(static_cast<size_t>(Lrk), true);
    if (a.row_mask)
        for (std::int64_t i = 0; i < L; ++i) rm[size_t(i)] = a.row_mask[h * L + i] != 0;
    if (a.col_mask)
        for (std::int64_t j = 0; j < Lk; ++j) cm[size_t(j)] = a.col_mask[h * Lk + j] != 0;
    SupportMask sup;
    if (a.dustbin) {
        for (std::int64_t i = 0; i < L; ++i) {
            Q(i, d) = static_cast<T>(c);
            K(i, d + 1) = T(1);
        }
        Q(L, d + 1) = static_cast<T>(-c * rt);
        K(L, d) = static_cast<T>(-rt);
        K(L, d + 1) = T(1);
        std::vector<std::pair<Index, Index>> edges;
        for (std::int64_t i = 0; i < L; ++i) {
            for (std::int64_t j = std::max<std::int64_t>(0, i - a.w); j <= std::min<std::int64_t>(L - 1, i + a.w); ++j)
                edges.emplace_back(i, j);
            edges.emplace_back(i, L);
        }
        for (std::int64_t j = 0; j <= L; ++j) edges.emplace_back(L, j);
        sup = SupportMask::explicit_edges(Lr, Lrk, std::move(edges), rm, cm);
        sup.validate();
    } else {
        sup = build_band_support(L, Lk, a.w, rm, cm);
    }
    // linear loss: G on valid rows only (inc/loss.hpp:74-98)
    for (std::int64_t i = 0; i < Lr; ++i)
        if (!sup.row_active(i))
            for (std::int64_t x = 0; x < d; ++x) G(i, x) = T(0);
    auto sched = TileSchedule::build(sup, a.tile_block);
    EpsSchedule<T> es = EpsSchedule<T>::single(static_cast<T>(a.eps), a.T);
    if (a.n_stages > 0) {
        es.stages.clear();
        for (int q = 0; q < a.n_stages; ++q) es.stages.push_back({static_cast<T>(a.stage_eps[q]), a.stage_iters[q]});
    }
    SurrogateRun<T> run = run_surrogate<T>(Q, K, V, sched, a.T, a.R, es, a.centered != 0);
    for (std::int64_t k = 0; k < Lr * d; ++k) a.O[h * Lr * d + k] = static_cast<double>(run.output.data()[k]);
    if (a.duals && Lk == L) {
        double* dp = a.duals + h * 6 * Lr;
        for (std::int64_t r = 0; r <= 2 && r <= a.R; ++r) {
            for (std::int64_t i = 0; i < Lr; ++i) dp[r * Lr + i] = static_cast<double>(run.trace.tail_u(r)[i]);
            for (std::int64_t j = 0; j < Lr; ++j) dp[(3 + r) * Lr + j] = static_cast<double>(run.trace.tail_v(r)[j]);
            if (a.gauges) a.gauges[h * 3 + r] = static_cast<double>(run.trace.gauge(run.trace.tail_step(r)));
        }
    }
    if (!a.dQ) return;
    CotangentSet<T> cs = r2_backward<T>(run.scaled, run.trace, G, Q, K, V,
                                        a.mode == 1 ? BackwardMode::DirectFourPlan : BackwardMode::OneReference);
    for (std::int64_t i = 0; i < Lr; ++i)
        for (std::int64_t x = 0; x < d; ++x)
            a.dQ[(h * Lr + i) * d + x] = i < L ? s * static_cast<double>(cs.grad_q(i, x)) : 0.0;
    for (std::int64_t j = 0; j < Lrk; ++j)
        for (std::int64_t x = 0; x < d; ++x) {
            a.dK[(h * Lrk + j) * d + x] = j < Lk ? s * static_cast<double>(cs.grad_k(j, x)) : 0.0;
            a.dV[(h * Lrk + j) * d + x] = static_cast<double>(cs.grad_v(j, x));
        }
    if (a.eta_v)
        for (std::int64_t j = 0; j < Lrk; ++j) a.eta_v[h * Lrk + j] = static_cast<double>(cs.base_cotangent.v[j]);
}

}  // namespace

extern "C" {

const char* refc_last_error() { return g_err.c_str(); }

// nh independent heads; tensors [nh][L'][d] doubles (values already rounded to the
// input dtype), masks [nh][L] uint8 or NULL.  precision 32 / 64 = the reference's
// float / double template instantiation.  dQ == NULL: forward only.  Returns 0 or 1.
int refc_run(std::int64_t nh, std::int64_t Lq, std::int64_t Lk, std::int64_t d, std::int64_t w, std::int64_t T,
             std::int64_t R, double eps, int dustbin, double dustbin_cost, const double* Q, const double* K,
             const double* V, const double* G, const std::uint8_t* row_mask, const std::uint8_t* col_mask,
             int precision, int mode, int tile_block, int centered, int nthreads, int n_stages,
             const double* stage_eps, const std::int64_t* stage_iters, double* O, double* dQ, double* dK, double* dV,
             double* eta_v, double* duals, double* gauges) {
    Args a{Lq, Lk, d, w, T, R, eps, dustbin, dustbin_cost, Q, K, V, G, row_mask, col_mask, mode, tile_block, centered,
           n_stages, stage_eps, stage_iters, O, dQ, dK, dV, eta_v, duals, gauges};
    std::atomic<std::int64_t> next{0};
    std::atomic<int> status{0};
    std::string first;
    std::atomic<bool> taken{false};
    auto worker = [&]() {
        for (;;) {
            const std::int64_t h = next.fetch_add(1);
            if (h >= nh || status.load() != 0) return;
            try {
                if (precision == 32) run_head<float>(a, h);
                else run_head<double>(a, h);
            } catch (const std::exception& e) {
                bool exp = false;
                if (taken.compare_exchange_strong(exp, true)) first = e.what();
                status.store(1);
                return;
            }
        }
    };
    std::vector<std::thread> pool;
    const int n = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>(nthreads, nh)));
    for (int t = 1; t < n; ++t) pool.emplace_back(worker);
    worker();
    for (auto& th : pool) th.join();
    if (status.load() != 0) g_err = first;
    return status.load();
}

}  // extern "C"
