// kat_tests.cpp -- the reference's own known-answer and cross-path tests for
// this path, ported one-for-one onto the CPU restatement (TEST INFRASTRUCTURE).
// Each TEST cites the reference test it ports.  Run by tests/test_oracle_kat.py.
// Usage: kat_tests [filter-substring]
#include <cstdio>
#include <functional>
#include <set>
#include <string>
#include <vector>

#include "sinktail_oracle.hpp"

using namespace stoc;
using dense::DenseProblem;

namespace {

struct TestCase {
    const char* name;
    std::function<void()> fn;
};
std::vector<TestCase>& registry() {
    static std::vector<TestCase> r;
    return r;
}
struct Registrar {
    Registrar(const char* n, std::function<void()> f) { registry().push_back({n, std::move(f)}); }
};
int g_checks = 0, g_fail = 0;
const char* g_current = "";

#define KAT_CAT2(a, b) a##b
#define KAT_CAT(a, b) KAT_CAT2(a, b)
#define TEST(name)                                                        \
    static void KAT_CAT(kat_fn_, __LINE__)();                             \
    static Registrar KAT_CAT(kat_reg_, __LINE__)(name, KAT_CAT(kat_fn_, __LINE__)); \
    static void KAT_CAT(kat_fn_, __LINE__)()
#define CHECK(cond)                                                                         \
    do {                                                                                    \
        ++g_checks;                                                                         \
        if (!(cond)) {                                                                      \
            ++g_fail;                                                                       \
            std::printf("  FAIL [%s] %s:%d: %s\n", g_current, __FILE__, __LINE__, #cond);   \
        }                                                                                   \
    } while (0)
#define CHECK_THROWS_AS(expr, Exc)                  \
    do {                                            \
        bool thrown = false;                        \
        try { (void)(expr); } catch (const Exc&) { thrown = true; } catch (...) {} \
        CHECK(thrown && #Exc);                      \
    } while (0)

bool approx(double a, double b, double rel = 1e-12) {
    return std::abs(a - b) <= rel * std::max(1.0, std::max(std::abs(a), std::abs(b)));
}

std::shared_ptr<const TileSchedule> full_sched(Index n, Index block = 64) {
    return TileSchedule::build(build_band_support(n, n, n), block);
}
Mat<double> dense_plan_of(const ScoreField<double>& S, const DualTrace<double>& tr, Index hu, Index hv) {
    return densify(staircase_plan(S, tr, hu, hv));
}
Mat<double> zeros(Index r, Index c) { return Mat<double>(r, c); }
Mat<double> identity(Index n) {
    Mat<double> m(n, n);
    for (Index i = 0; i < n; ++i) m(i, i) = 1;
    return m;
}
std::int64_t brute_band_count(Index Lq, Index Lk, Index W) {
    std::int64_t n = 0;
    for (Index i = 0; i < Lq; ++i)
        for (Index j = 0; j < Lk; ++j)
            if (std::abs(i - j) <= W) ++n;
    return n;
}

struct Ran {
    Instance<double> inst;
    SurrogateRun<double> run;
    Mat<double> G;
    LossSpec<double> loss;
};
Ran run_linear(InstanceSpec spec, double loss_scale = 1.0) {
    Ran r{make_instance<double>(spec), {}, {}, {}};
    r.run = run_surrogate(r.inst.Q, r.inst.K, r.inst.V, r.inst.schedule, spec.base_depth, spec.tail_depth, r.inst.eps);
    r.loss = random_linear_loss(r.inst, loss_scale);
    r.G = r.loss.output_cotangent(r.run.output, r.inst.V, r.inst.schedule->support().row_mask());
    return r;
}

// ======================= test_support.cpp =======================
TEST("support: zero band is the diagonal (test_support.cpp:25-33)") {
    SupportMask m = build_band_support(3, 3, 0);
    std::set<std::pair<Index, Index>> e;
    for (Index i = 0; i < 3; ++i) m.for_each_in_row(i, [&](Index j) { e.insert({i, j}); });
    CHECK((e == std::set<std::pair<Index, Index>>{{0, 0}, {1, 1}, {2, 2}}));
}
TEST("support: banded counts match brute force (test_support.cpp:35-45)") {
    for (Index L : {1, 2, 3, 5, 8, 13, 33, 64})
        for (Index W : {0, 1, 2, 3, 5, 8}) {
            SupportMask m = build_band_support(L, L, W);
            CHECK(m.active_edge_count() == brute_band_count(L, L, W));
            CHECK(banded_entry_count(L, W) == brute_band_count(L, L, W));
        }
    CHECK(build_band_support(4, 4, 1).active_edge_count() == 10);
}
TEST("support: rectangular bands (test_support.cpp:47-54)") {
    SupportMask m = build_band_support(4, 7, 3);
    CHECK(m.active_edge_count() == brute_band_count(4, 7, 3));
    CHECK(m.contains(0, 3));
    CHECK(!m.contains(0, 4));
    CHECK_THROWS_AS(build_band_support(4, 7, 2), InfeasibleSupport);
}
TEST("support: long-context band count 32,521,216 (test_support.cpp:56-60)") {
    CHECK(banded_entry_count(16384, 1024) == 32521216);
    CHECK(build_band_support(16384, 16384, 1024).active_edge_count() == 32521216);
}
TEST("support: masked rows and columns (test_support.cpp:62-70)") {
    SupportMask m = build_band_support(4, 4, 1, {true, false, true, true}, {true, true, false, true});
    CHECK(!m.contains(1, 1));
    CHECK(!m.contains(2, 2));
    CHECK(m.contains(2, 1));
    CHECK(m.contains(3, 3));
}
TEST("support: infeasible supports rejected (test_support.cpp:72-79)") {
    CHECK_THROWS_AS(build_band_support(3, 3, 0, {}, {false, true, true}), InfeasibleSupport);
    CHECK_THROWS_AS(build_band_support(3, 3, 0, {true, true, false}, {}), InfeasibleSupport);
}
TEST("support: explicit sorted edges (test_support.cpp:81-90)") {
    SupportMask m = SupportMask::explicit_edges(3, 3, {{2, 1}, {0, 0}, {1, 2}, {0, 2}, {2, 1}});
    std::vector<std::pair<Index, Index>> seen;
    for (Index i = 0; i < 3; ++i) m.for_each_in_row(i, [&](Index j) { seen.push_back({i, j}); });
    CHECK((seen == std::vector<std::pair<Index, Index>>{{0, 0}, {0, 2}, {1, 2}, {2, 1}}));
    CHECK(m.contains(0, 2));
    CHECK(!m.contains(2, 2));
}
TEST("support: dustbin augmentation by construction (test_support.cpp:92-111)") {
    AugmentedSupport aug = augment_dustbin(build_band_support(4, 4, 1), 2);
    CHECK(aug.mask.n_rows() == 6);
    CHECK(aug.mask.n_cols() == 6);
    CHECK(aug.dustbin_row == 4);
    CHECK(aug.effective_band == 4);
    CHECK(aug.filler_rows == std::vector<Index>{5});
    CHECK(aug.mask.row_active(4));
    CHECK(!aug.mask.row_active(5));
    for (Index i = 0; i < 4; ++i) {
        CHECK(aug.mask.contains(i, aug.dustbin_col));
        CHECK(aug.mask.contains(aug.dustbin_row, i));
    }
    CHECK(aug.mask.contains(aug.dustbin_row, aug.dustbin_col));
}
TEST("support: dustbin augmentation small cases (test_support.cpp:113-135)") {
    {
        AugmentedSupport aug = augment_dustbin(build_band_support(2, 2, 2), 1);
        CHECK(aug.mask.n_rows() == 3);
        CHECK(aug.effective_band == 2);
        CHECK(aug.filler_rows.empty());
        CHECK(aug.mask.active_edge_count() == 9);
    }
    {
        AugmentedSupport aug = augment_dustbin(build_band_support(8, 8, 2), 4);
        std::int64_t count = 0;
        for (Index i = 0; i < aug.mask.n_rows(); ++i)
            for (Index j = 0; j < aug.mask.n_cols(); ++j) {
                const bool active = (i <= 8) && (j <= 8) && std::abs(i - j) <= 8;
                CHECK(aug.mask.contains(i, j) == active);
                if (active) ++count;
            }
        CHECK(count == 81);
        CHECK(aug.mask.active_edge_count() == 81);
    }
}
TEST("support: tile schedule covers each edge once (test_support.cpp:137-156)") {
    SupportMask m = build_band_support(13, 17, 4);
    auto sched = TileSchedule::build(m, 4);
    std::set<std::pair<Index, Index>> covered;
    std::int64_t total = 0;
    for (size_t t = 0; t < sched->tile_count(); ++t) {
        const TileRange& r = sched->tiles()[t];
        for (Index i = 0; i < r.rows(); ++i)
            for (Index j = 0; j < r.cols(); ++j)
                if (sched->tile_activity(t)(i, j)) {
                    CHECK(covered.insert({r.row_begin + i, r.col_begin + j}).second);
                    ++total;
                }
    }
    CHECK(total == m.active_edge_count());
    for (const auto& e : covered) CHECK(m.contains(e.first, e.second));
    CHECK(sched->active_edges() == total);
}
TEST("support: memory ledger long-context figures (test_support.cpp:158-168)") {
    LedgerReport r = estimate_memory_ledger(16384, 1024, 128, 64, 4, 2, 15);
    CHECK(r.active_entries == 32521216);
    CHECK(mib_string(r.direct_plan_bytes, 2) == "496.23");
    CHECK(mib_string(r.one_reference_plan_bytes, 2) == "124.06");
    CHECK(mib_string(r.direct_tile_bytes, 4) == "0.2500");
    CHECK(mib_string(r.one_reference_tile_bytes, 4) == "0.0625");
    CHECK(mib_string(r.tail_dual_bytes, 3) == "0.375");
    CHECK(mib_string(r.base_tail_dual_bytes, 2) == "2.25");
    CHECK(mib_string(r.qkv_bytes, 2) == "12.00");
}
TEST("support: ledger trivial case and 4x ratio (test_support.cpp:170-182)") {
    LedgerReport r = estimate_memory_ledger(1, 0, 1, 1, 4, 2, 0);
    CHECK(r.active_entries == 1);
    CHECK(r.direct_plan_bytes == 16);
    CHECK(r.one_reference_plan_bytes == 4);
    for (Index L : {1, 7, 64, 1000})
        for (Index W : {0, 3, 200}) {
            LedgerReport x = estimate_memory_ledger(L, W, 8, 4, 4, 2, 5);
            CHECK(x.direct_plan_bytes == 4 * x.one_reference_plan_bytes);
            CHECK(x.direct_tile_bytes == 4 * x.one_reference_tile_bytes);
        }
}

// ======================= test_io.cpp (RNG) =======================
TEST("rng: draw-order independent and deterministic (test_io.cpp:68-81)") {
    Mat<double> a = normal_matrix<double>(5, "Q", 8, 4), b = normal_matrix<double>(5, "Q", 8, 4);
    CHECK(max_abs_diff(a, b) == 0.0);
    Mat<double> wide = normal_matrix<double>(5, "Q", 4, 8);
    CHECK(wide(0, 5) == a(1, 1));
    CHECK(max_abs_diff(a, normal_matrix<double>(5, "K", 8, 4)) > 0.0);
    CHECK(max_abs_diff(a, normal_matrix<double>(6, "Q", 8, 4)) > 0.0);
}
TEST("rng: plausible moments (test_io.cpp:83-90)") {
    Mat<double> x = normal_matrix<double>(17, "moments", 20000, 1);
    double mean = 0;
    for (double v : x.a) mean += v;
    mean /= 20000.0;
    double var = 0;
    for (double v : x.a) var += (v - mean) * (v - mean);
    var /= 20000.0;
    CHECK(std::abs(mean) < 0.03);
    CHECK(std::abs(var - 1.0) < 0.05);
}

// ======================= test_sinkhorn.cpp =======================
TEST("sinkhorn: scaled scores absorb the temperature (test_sinkhorn.cpp:33-55)") {
    Mat<double> Q(1, 4), K(1, 4);
    Q(0, 0) = 1;
    K(0, 0) = 1;
    auto s1 = full_sched(1);
    CHECK(approx(scaled_scores<double>(Q, K, 0.5, s1).values.blocks[0](0, 0), 1.0));
    CHECK(scaled_scores<double>(zeros(1, 4), zeros(1, 4), 1.0, s1).values.blocks[0](0, 0) == 0.0);
    Mat<double> Qr = normal_matrix<double>(7, "Q", 6, 4), Kr = normal_matrix<double>(7, "K", 6, 4);
    auto s6 = full_sched(6);
    auto a = scaled_scores<double>(Qr, Kr, 1.0, s6), b = scaled_scores<double>(Qr, Kr, 2.0, s6);
    for (size_t t = 0; t < s6->tile_count(); ++t)
        for (size_t k = 0; k < a.values.blocks[t].a.size(); ++k)
            CHECK(std::abs(a.values.blocks[t].a[k] - 2.0 * b.values.blocks[t].a[k]) < 1e-15);
    CHECK_THROWS_AS(scaled_scores<double>(Qr, Kr, 0.0, s6), InvalidTemperature);
}
TEST("sinkhorn: row half-step tiny supports u=0, -ln2, -2 (test_sinkhorn.cpp:57-86)") {
    {
        auto S = scaled_scores<double>(zeros(1, 1), zeros(1, 1), 1.0, full_sched(1));
        CHECK(std::abs(row_half_step(S, Vec<double>(1, 0.0))[0]) < 1e-15);
    }
    {
        auto sched = TileSchedule::build(build_band_support(1, 2, 2), 8);
        auto S = scaled_scores<double>(zeros(1, 3), zeros(2, 3), 1.0, sched);
        CHECK(approx(row_half_step(S, Vec<double>(2, 0.0))[0], -std::log(2.0), 1e-14));
    }
    {
        auto sched = TileSchedule::build(SupportMask::explicit_edges(1, 1, {{0, 0}}), 4);
        auto S = scaled_scores<double>(zeros(1, 1), zeros(1, 1), 1.0, sched);
        S.values.blocks[0](0, 0) = 3.0;
        CHECK(approx(row_half_step(S, Vec<double>(1, -1.0))[0], -2.0));
    }
}
TEST("sinkhorn: col half-step transpose analogue v=0, -1 (test_sinkhorn.cpp:88-120)") {
    {
        auto sched = TileSchedule::build(build_band_support(2, 1, 2), 8);
        auto S = scaled_scores<double>(zeros(2, 3), zeros(1, 3), 1.0, sched);
        CHECK(std::abs(col_half_step(S, Vec<double>(2, -std::log(2.0)))[0]) < 1e-14);
    }
    {
        auto sched = TileSchedule::build(SupportMask::explicit_edges(1, 1, {{0, 0}}), 4);
        auto S = scaled_scores<double>(zeros(1, 1), zeros(1, 1), 1.0, sched);
        S.values.blocks[0](0, 0) = -1.0;
        CHECK(approx(col_half_step(S, Vec<double>(1, 2.0))[0], -1.0));
    }
    {
        const Index n = 9;
        Mat<double> A = normal_matrix<double>(3, "Q", n, 4);
        auto S = scaled_scores<double>(A, A, 1.0, full_sched(n));
        Mat<double> wm = normal_matrix<double>(5, "w", n, 1);
        Vec<double> w(wm.a.begin(), wm.a.end());
        CHECK(max_abs_diff(row_half_step(S, w), col_half_step(S, w)) < 1e-13);
    }
}
TEST("sinkhorn: centering known answer (test_sinkhorn.cpp:122-145)") {
    Vec<double> u{1, 3}, v{0, 0};
    std::vector<bool> valid{true, true};
    auto c = center(u, v, valid);
    CHECK(approx(c.shift, 2.0));
    CHECK(approx(c.u[0], -1.0));
    CHECK(approx(c.u[1], 1.0));
    CHECK(approx(c.v[0], 2.0));
    CHECK(approx(c.v[1], 2.0));
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j) CHECK(approx(c.u[i] + c.v[j], u[i] + v[j]));
    auto c2 = center(c.u, c.v, valid);
    CHECK(approx(c2.shift, 0.0));
    CHECK(max_abs_diff(c2.u, c.u) == 0.0);
    CHECK_THROWS_AS(center<double>(u, v, std::vector<bool>{false, false}), InfeasibleSupport);
}
TEST("sinkhorn: uniform instance u=0, gauge=-ln n, plan=1/n (test_sinkhorn.cpp:147-162)") {
    const Index n = 5;
    auto raw = raw_scores<double>(zeros(n, 3), zeros(n, 3), full_sched(n));
    auto tr = stopped_base_solve(raw, 1, EpsSchedule<double>::single(1.0, 1));
    CHECK(max_abs(tr.u(1)) < 1e-15);
    CHECK(approx(tr.gauge(1), -std::log(double(n))));
    for (double x : tr.v(1)) CHECK(std::abs(x + std::log(double(n))) < 1e-15);
    auto plan = dense_plan_of(scale_to_temperature(raw, 1.0), tr, 1, 1);
    for (double x : plan.a) CHECK(std::abs(x - 1.0 / n) < 1e-15);
}
TEST("sinkhorn: cold start has empty ledger (test_sinkhorn.cpp:164-174)") {
    auto raw = raw_scores<double>(zeros(3, 2), zeros(3, 2), full_sched(3));
    auto tr = stopped_base_solve(raw, 0, EpsSchedule<double>::single(1.0, 0));
    CHECK(tr.steps() == 0);
    CHECK(tr.split == 0);
    CHECK(max_abs(tr.u(0)) == 0.0);
    CHECK(max_abs(tr.v(0)) == 0.0);
    CHECK(tr.gauge(0) == 0.0);
}
TEST("sinkhorn: column-sum oscillation decays (test_sinkhorn.cpp:176-197)") {
    InstanceSpec spec;
    spec.n_rows = spec.n_cols = 128;
    spec.half_band = 32;
    spec.base_depth = 12;
    spec.tail_depth = 0;
    spec.seed = 0;
    auto inst = make_instance<double>(spec);
    auto raw = raw_scores<double>(inst.Q, inst.K, inst.schedule);
    auto tr = stopped_base_solve(raw, spec.base_depth, inst.eps);
    auto S = scale_to_temperature(raw, 1.0);
    double prev = std::numeric_limits<double>::infinity();
    for (Index h = 1; h <= tr.steps(); ++h) {
        auto p = dense_plan_of(S, tr, h, h - 1);
        double lo = 1e300, hi = -1e300;
        for (Index j = 0; j < p.cols(); ++j) {
            double cs = 0;
            for (Index i = 0; i < p.rows(); ++i) cs += p(i, j);
            lo = std::min(lo, std::log(cs));
            hi = std::max(hi, std::log(cs));
        }
        const double osc = hi - lo;
        if (h > 1) CHECK(osc <= prev + 1e-12);
        prev = osc;
    }
    CHECK(prev < 1e-3);
}
TEST("sinkhorn: tail fixed point, L=2 staircase 0.5, contraction (test_sinkhorn.cpp:199-242)") {
    {
        const Index n = 4;
        auto raw = raw_scores<double>(zeros(n, 2), zeros(n, 2), full_sched(n));
        auto tr = stopped_base_solve(raw, 2, EpsSchedule<double>::single(1.0, 2));
        tail_refine(raw, tr, 2, 1.0);
        for (Index r = 1; r <= 2; ++r) {
            CHECK(max_abs_diff(tr.tail_u(r), tr.tail_u(0)) < 1e-14);
            CHECK(max_abs_diff(tr.tail_v(r), tr.tail_v(0)) < 1e-14);
        }
    }
    {
        auto raw = raw_scores<double>(zeros(2, 2), zeros(2, 2), full_sched(2));
        auto tr = stopped_base_solve(raw, 1, EpsSchedule<double>::single(1.0, 1));
        tail_refine(raw, tr, 2, 1.0);
        auto S = scale_to_temperature(raw, 1.0);
        for (Index a : {1, 2})
            for (Index b : {a - 1, a}) {
                auto p = dense_plan_of(S, tr, tr.tail_step(a), tr.tail_step(b));
                for (double x : p.a) CHECK(std::abs(x - 0.5) < 1e-15);
            }
    }
    {
        InstanceSpec spec;
        spec.n_rows = spec.n_cols = 64;
        spec.half_band = 16;
        spec.base_depth = 6;
        spec.tail_depth = 2;
        spec.seed = 1;
        auto inst = make_instance<double>(spec);
        auto run = run_surrogate(inst.Q, inst.K, inst.V, inst.schedule, 6, 2, inst.eps);
        CHECK(max_abs_diff(run.trace.tail_u(2), run.trace.tail_u(1)) <
              max_abs_diff(run.trace.tail_u(1), run.trace.tail_u(0)));
    }
}
TEST("sinkhorn: unit targets after each half-step (test_sinkhorn.cpp:244-267)") {
    InstanceSpec spec;
    spec.n_rows = spec.n_cols = 48;
    spec.half_band = 12;
    spec.base_depth = 5;
    spec.tail_depth = 2;
    spec.seed = 2;
    auto inst = make_instance<double>(spec);
    auto raw = raw_scores<double>(inst.Q, inst.K, inst.schedule);
    auto tr = stopped_base_solve(raw, 5, inst.eps);
    tail_refine(raw, tr, 2, 1.0);
    auto S = scale_to_temperature(raw, 1.0);
    for (Index h = 1; h <= tr.steps(); ++h) {
        auto mixed = dense_plan_of(S, tr, h, h - 1);
        for (Index i = 0; i < mixed.rows(); ++i) {
            double s = 0;
            for (Index j = 0; j < mixed.cols(); ++j) s += mixed(i, j);
            CHECK(approx(s, 1.0, 1e-12));
        }
        auto same = dense_plan_of(S, tr, h, h);
        for (Index j = 0; j < same.cols(); ++j) {
            double s = 0;
            for (Index i = 0; i < same.rows(); ++i) s += same(i, j);
            CHECK(approx(s, 1.0, 1e-12));
        }
    }
}
TEST("sinkhorn: gauge equivariance centered vs raw (test_sinkhorn.cpp:269-304)") {
    InstanceSpec spec;
    spec.n_rows = spec.n_cols = 24;
    spec.half_band = 8;
    spec.base_depth = 4;
    spec.tail_depth = 2;
    spec.seed = 3;
    auto inst = make_instance<double>(spec);
    auto raw = raw_scores<double>(inst.Q, inst.K, inst.schedule);
    auto cent = stopped_base_solve(raw, 4, inst.eps, true);
    tail_refine(raw, cent, 2, 1.0);
    auto plain = stopped_base_solve(raw, 4, inst.eps, false);
    tail_refine(raw, plain, 2, 1.0);
    auto S = scale_to_temperature(raw, 1.0);
    for (Index h = 1; h <= cent.steps(); ++h) {
        const double c = cent.gauge(h);
        for (Index i = 0; i < 24; ++i) CHECK(approx(cent.u(h)[i], plain.u(h)[i] - c, 1e-12));
        for (Index j = 0; j < 24; ++j) CHECK(approx(cent.v(h)[j], plain.v(h)[j] + c, 1e-12));
        CHECK(max_abs_diff(dense_plan_of(S, cent, h, h), dense_plan_of(S, plain, h, h)) < 1e-12);
    }
}
TEST("sinkhorn: mixed-time plans need the gauge correction (test_sinkhorn.cpp:306-340)") {
    InstanceSpec spec;
    spec.n_rows = spec.n_cols = 16;
    spec.half_band = 16;
    spec.base_depth = 3;
    spec.tail_depth = 2;
    spec.seed = 4;
    auto inst = make_instance<double>(spec);
    auto raw = raw_scores<double>(inst.Q, inst.K, inst.schedule);
    auto S = scale_to_temperature(raw, 1.0);
    auto cent = stopped_base_solve(raw, 3, inst.eps, true);
    tail_refine(raw, cent, 2, 1.0);
    auto plain = stopped_base_solve(raw, 3, inst.eps, false);
    tail_refine(raw, plain, 2, 1.0);
    const Index a = cent.tail_step(1), b = cent.tail_step(0);
    const double gd = cent.gauge(a) - cent.gauge(b);
    CHECK(std::abs(gd) > 1e-6);
    auto corrected = dense_plan_of(S, cent, a, b), ungauged = dense_plan_of(S, plain, a, b);
    CHECK(max_abs_diff(corrected, ungauged) < 1e-12);
    DualTrace<double> nl = cent;
    std::fill(nl.gauge_hist.begin(), nl.gauge_hist.end(), 0.0);
    auto unc = dense_plan_of(S, nl, a, b);
    const double expected_off = std::abs(std::expm1(-gd)) * max_abs(ungauged);
    CHECK(max_abs_diff(unc, ungauged) > 0.5 * expected_off);
}
TEST("sinkhorn: entry points require raw scores (test_sinkhorn.cpp:342-352)") {
    auto sched = full_sched(4);
    auto scaled = scaled_scores<double>(zeros(4, 2), zeros(4, 2), 1.0, sched);
    CHECK_THROWS_AS(stopped_base_solve(scaled, 1, EpsSchedule<double>::single(1.0, 1)), std::invalid_argument);
    CHECK_THROWS_AS(scale_to_temperature(scaled, 2.0), std::invalid_argument);
    auto raw = raw_scores<double>(zeros(4, 2), zeros(4, 2), sched);
    CHECK_THROWS_AS(scale_to_temperature(raw, 0.0), InvalidTemperature);
}
TEST("sinkhorn: epsilon schedule keeps the budget (test_sinkhorn.cpp:354-377)") {
    InstanceSpec spec;
    spec.n_rows = spec.n_cols = 20;
    spec.half_band = 6;
    spec.base_depth = 6;
    spec.tail_depth = 1;
    spec.seed = 5;
    spec.stages = {{4.0, 2}, {2.0, 2}, {1.0, 2}};
    auto inst = make_instance<double>(spec);
    auto raw = raw_scores<double>(inst.Q, inst.K, inst.schedule);
    auto tr = stopped_base_solve(raw, 6, inst.eps);
    CHECK(tr.steps() == 6);
    CHECK(tr.eps_at(1) == 4.0);
    CHECK(tr.eps_at(3) == 2.0);
    CHECK(tr.eps_at(6) == 1.0);
    CHECK(tr.stage_at(1) == 0);
    CHECK(tr.stage_at(6) == 2);
    EpsSchedule<double> bad;
    bad.stages = {{1.0, 2}, {2.0, 2}};
    CHECK_THROWS_AS(bad.validate(4), InvalidTemperature);
    CHECK_THROWS_AS(EpsSchedule<double>::single(1.0, 3).validate(6), std::invalid_argument);
}
TEST("sinkhorn: transport application 0.5 / identity / dense (test_sinkhorn.cpp:379-418)") {
    {
        auto raw = raw_scores<double>(zeros(2, 2), zeros(2, 2), full_sched(2));
        auto tr = stopped_base_solve(raw, 1, EpsSchedule<double>::single(1.0, 1));
        auto O = apply_transport(scale_to_temperature(raw, 1.0), tr.u(1), tr.v(1), identity(2));
        for (double x : O.a) CHECK(std::abs(x - 0.5) < 1e-15);
    }
    {
        auto sched = TileSchedule::build(build_band_support(3, 3, 0), 2);
        auto raw = raw_scores<double>(zeros(3, 2), zeros(3, 2), sched);
        auto tr = stopped_base_solve(raw, 1, EpsSchedule<double>::single(1.0, 1));
        Mat<double> V = normal_matrix<double>(11, "V", 3, 5);
        auto O = apply_transport(scale_to_temperature(raw, 1.0), tr.u(1), tr.v(1), V);
        CHECK(max_abs_diff(O, V) < 1e-14);
    }
    {
        InstanceSpec spec;
        spec.n_rows = spec.n_cols = 32;
        spec.half_band = 8;
        spec.base_depth = 4;
        spec.tail_depth = 2;
        spec.seed = 6;
        auto inst = make_instance<double>(spec);
        auto run = run_surrogate(inst.Q, inst.K, inst.V, inst.schedule, 4, 2, inst.eps);
        const Index h = run.trace.steps();
        auto dense_o = dense::matmul(dense_plan_of(run.scaled, run.trace, h, h), inst.V);
        CHECK(max_abs_diff(dense_o, run.output) < 1e-12);
    }
}
TEST("sinkhorn: blockwise forward equals dense oracle (test_sinkhorn.cpp:420-449)") {
    for (std::uint64_t seed : {0, 1, 2}) {
        InstanceSpec spec;
        spec.n_rows = spec.n_cols = 96;
        spec.half_band = 24;
        spec.base_depth = 8;
        spec.tail_depth = 2;
        spec.seed = seed;
        spec.tile_block = 32;
        auto inst = make_instance<double>(spec);
        auto run = run_surrogate(inst.Q, inst.K, inst.V, inst.schedule, 8, 2, inst.eps);
        DenseProblem dp;
        dp.Q = inst.Q;
        dp.K = inst.K;
        dp.V = inst.V;
        dp.support = dense::dense_support_of(inst.schedule->support());
        dp.epsilon = 1.0;
        dp.base_depth = 8;
        dp.tail_depth = 2;
        dp.loss = LossSpec<double>::linear(zeros(96, spec.head_dim));
        CHECK(max_abs_diff(dense::dense_forward(dp).output, run.output) < 1e-12);
    }
}
TEST("sinkhorn: dustbin fillers inert, equal to explicit (test_sinkhorn.cpp:451-488)") {
    InstanceSpec spec;
    spec.n_rows = spec.n_cols = 12;
    spec.half_band = 3;
    spec.base_depth = 4;
    spec.tail_depth = 2;
    spec.seed = 7;
    spec.dustbin_block = 4;
    auto inst = make_instance<double>(spec);
    auto run = run_surrogate(inst.Q, inst.K, inst.V, inst.schedule, 4, 2, inst.eps);
    const Index h = run.trace.steps();
    auto plan = dense_plan_of(run.scaled, run.trace, h, h);
    for (Index k = 13; k < 16; ++k)
        for (Index x = 0; x < 16; ++x) {
            CHECK(plan(k, x) == 0.0);
            CHECK(plan(x, k) == 0.0);
        }
    const SupportMask& am = inst.schedule->support();
    std::vector<std::pair<Index, Index>> edges;
    for (Index i = 0; i < am.n_rows(); ++i) am.for_each_in_row(i, [&](Index j) { edges.emplace_back(i, j); });
    auto manual = SupportMask::explicit_edges(am.n_rows(), am.n_cols(), edges, am.row_mask(), am.col_mask());
    auto run2 = run_surrogate(inst.Q, inst.K, inst.V, TileSchedule::build(manual, spec.tile_block), 4, 2, inst.eps);
    CHECK(max_abs_diff(run.output, run2.output) <= 1e-12);
    for (Index hh = 0; hh <= run.trace.steps(); ++hh) {
        CHECK(max_abs_diff(run.trace.u(hh), run2.trace.u(hh)) <= 1e-12);
        CHECK(max_abs_diff(run.trace.v(hh), run2.trace.v(hh)) <= 1e-12);
    }
}
TEST("sinkhorn: tile block size invariance (test_sinkhorn.cpp:490-506)") {
    InstanceSpec spec;
    spec.n_rows = spec.n_cols = 40;
    spec.half_band = 10;
    spec.base_depth = 5;
    spec.tail_depth = 2;
    spec.seed = 8;
    spec.tile_block = 8;
    auto a = make_instance<double>(spec);
    spec.tile_block = 64;
    auto b = make_instance<double>(spec);
    auto ra = run_surrogate(a.Q, a.K, a.V, a.schedule, 5, 2, a.eps);
    auto rb = run_surrogate(b.Q, b.K, b.V, b.schedule, 5, 2, b.eps);
    CHECK(max_abs_diff(ra.output, rb.output) < 1e-12);
}

// ======================= test_adjoint.cpp =======================
TEST("adjoint: zero cotangent gives zero (test_adjoint.cpp:34-53)") {
    InstanceSpec spec;
    spec.n_rows = spec.n_cols = 12;
    spec.half_band = 4;
    spec.base_depth = 3;
    spec.tail_depth = 2;
    Ran r = run_linear(spec);
    Mat<double> zero(r.G.rows(), r.G.cols());
    for (BackwardMode mode : {BackwardMode::OneReference, BackwardMode::DirectFourPlan}) {
        auto c = r2_backward(r.run.scaled, r.run.trace, zero, r.inst.Q, r.inst.K, r.inst.V, mode);
        CHECK(max_abs(c.grad_q) == 0.0);
        CHECK(max_abs(c.grad_k) == 0.0);
        CHECK(max_abs(c.grad_v) == 0.0);
        CHECK(c.base_l2() == 0.0);
        CHECK(c.d_eps == 0.0);
    }
    auto g = tail_adjoint_generic(r.run.scaled, r.run.trace, zero, r.inst.Q, r.inst.K, r.inst.V);
    CHECK(max_abs(densify(g.score_bar)) == 0.0);
}
TEST("adjoint: hand-evaluated 2x2 g_v=.5, u2bar=0 (test_adjoint.cpp:55-69)") {
    auto raw = raw_scores<double>(zeros(2, 2), zeros(2, 2), full_sched(2));
    auto tr = stopped_base_solve(raw, 3, EpsSchedule<double>::single(1.0, 3));
    tail_refine(raw, tr, 2, 1.0);
    auto c = tail_adjoint_generic(scale_to_temperature(raw, 1.0), tr, identity(2), zeros(2, 2), zeros(2, 2),
                                  identity(2));
    CHECK(approx(c.v_bar[2][0], 0.5));
    CHECK(approx(c.v_bar[2][1], 0.5));
    CHECK(max_abs(c.u_bar[2]) < 1e-14);
}
TEST("adjoint: one-reference formula collapses when converged (test_adjoint.cpp:71-93)") {
    Mat<double> p(3, 3, 0.25);
    Mat<double> z = normal_matrix<double>(5, "Z", 3, 3);
    auto col = [](std::uint64_t s, const char* t) {
        Mat<double> m = normal_matrix<double>(s, t, 3, 1);
        return Vec<double>(m.a.begin(), m.a.end());
    };
    Vec<double> u2 = col(6, "a"), v2 = col(7, "b"), u1 = col(8, "c"), v1 = col(9, "d"), ones(3, 1.0), zv(3, 0.0);
    auto got = r2_score_cotangent_tile<double>(p, z, u2.data(), v2.data(), u1.data(), v1.data(), ones.data(),
                                               ones.data(), ones.data(), 1.0, 1.0);
    for (Index i = 0; i < 3; ++i)
        for (Index j = 0; j < 3; ++j)
            CHECK(approx(got(i, j), p(i, j) * (z(i, j) - v2[j] - u2[i] - v1[j] - u1[i]), 1e-14));
    auto zero_tile = r2_score_cotangent_tile<double>(p, Mat<double>(3, 3), zv.data(), zv.data(), zv.data(),
                                                     zv.data(), ones.data(), ones.data(), ones.data(), 1.0, 1.0);
    CHECK(max_abs(zero_tile) == 0.0);
}
TEST("adjoint: single-edge score backprop 0.5 (test_adjoint.cpp:95-106)") {
    auto sched = TileSchedule::build(SupportMask::explicit_edges(1, 1, {{0, 0}}), 4);
    BlockField<double> sbar(sched);
    sbar.blocks[0](0, 0) = 1.0;
    Mat<double> Q(1, 4), K(1, 4), gq, gk;
    K(0, 1) = 1.0;
    backprop_scores_to_qkv<double>(sbar, Q, K, 1.0, gq, gk);
    CHECK(approx(gq(0, 1), 0.5));
    CHECK(gq(0, 0) == 0.0);
}
TEST("adjoint: score backprop matches FD (test_adjoint.cpp:108-146)") {
    const Index n = 6, d = 3;
    Mat<double> Q = normal_matrix<double>(21, "Q", n, d), K = normal_matrix<double>(21, "K", n, d);
    auto sched = TileSchedule::build(build_band_support(n, n, 2), 4);
    BlockField<double> sbar(sched);
    for (size_t t = 0; t < sched->tile_count(); ++t) {
        const TileRange& r = sched->tiles()[t];
        sbar.blocks[t] = normal_matrix<double>(33 + t, "S", r.rows(), r.cols());
        for (Index i = 0; i < r.rows(); ++i)
            for (Index j = 0; j < r.cols(); ++j)
                if (!sched->tile_activity(t)(i, j)) sbar.blocks[t](i, j) = 0.0;
    }
    const double eps = 0.7;
    Mat<double> gq, gk;
    backprop_scores_to_qkv<double>(sbar, Q, K, eps, gq, gk);
    auto value = [&](const Mat<double>& q, const Mat<double>& k) {
        auto s = scaled_scores<double>(q, k, eps, sched);
        double acc = 0;
        for (size_t t = 0; t < sched->tile_count(); ++t)
            for (size_t x = 0; x < s.values.blocks[t].a.size(); ++x) acc += s.values.blocks[t].a[x] * sbar.blocks[t].a[x];
        return acc;
    };
    const double h = 1e-6;
    for (Index i = 0; i < n; i += 2)
        for (Index j = 0; j < d; ++j) {
            Mat<double> qp = Q, qm = Q, kp = K, km = K;
            qp(i, j) += h;
            qm(i, j) -= h;
            kp(i, j) += h;
            km(i, j) -= h;
            CHECK(approx(gq(i, j), (value(qp, K) - value(qm, K)) / (2 * h), 1e-7));
            CHECK(approx(gk(i, j), (value(Q, kp) - value(Q, km)) / (2 * h), 1e-7));
        }
}
TEST("adjoint: half-step Jacobian is -mixed plan (test_adjoint.cpp:148-177)") {
    InstanceSpec spec;
    spec.n_rows = spec.n_cols = 10;
    spec.half_band = 3;
    spec.base_depth = 2;
    spec.tail_depth = 0;
    spec.seed = 11;
    auto inst = make_instance<double>(spec);
    auto S = scale_to_temperature(raw_scores<double>(inst.Q, inst.K, inst.schedule), 1.0);
    Mat<double> vm = normal_matrix<double>(12, "v", 10, 1), wm = normal_matrix<double>(13, "w", 10, 1);
    Vec<double> v(vm.a.begin(), vm.a.end()), w(wm.a.begin(), wm.a.end());
    Vec<double> u = row_half_step(S, v);
    const double h = 1e-6;
    Vec<double> vp = v, vn = v;
    for (size_t k = 0; k < v.size(); ++k) { vp[k] += h * w[k]; vn[k] -= h * w[k]; }
    Vec<double> up = row_half_step(S, vp), un = row_half_step(S, vn);
    DualTrace<double> probe;
    probe.centered = false;
    probe.u_hist = {Vec<double>(10, 0.0), u};
    probe.v_hist = {v, v};
    probe.eps_hist = {0.0, 1.0};
    probe.stage_hist = {-1, 0};
    Vec<double> jac(10, 0.0);
    plan_apply(S, probe, 1, 0, w, jac);
    double mx = 0;
    for (size_t k = 0; k < 10; ++k) mx = std::max(mx, std::abs((up[k] - un[k]) / (2 * h) + jac[k]));
    CHECK(mx < 1e-8);
}
TEST("adjoint: orbit identity, staircase = rescaled reference (test_adjoint.cpp:179-210)") {
    InstanceSpec spec;
    spec.n_rows = spec.n_cols = 24;
    spec.half_band = 6;
    spec.base_depth = 4;
    spec.tail_depth = 2;
    spec.seed = 14;
    Ran r = run_linear(spec);
    const auto& tr = r.run.trace;
    const auto& S = r.run.scaled;
    const Index h2 = tr.tail_step(2);
    auto p22 = dense_plan_of(S, tr, h2, h2);
    for (Index a : {2, 1})
        for (Index b : {a, a - 1}) {
            const Index ha = tr.tail_step(a), hb = tr.tail_step(b);
            auto direct = dense_plan_of(S, tr, ha, hb);
            for (Index i = 0; i < 24; ++i)
                for (Index j = 0; j < 24; ++j) {
                    if (p22(i, j) == 0.0) continue;
                    const double lr = tr.u(ha)[i] - tr.u(h2)[i] + tr.gauge(ha) - tr.gauge(h2);
                    const double lc = tr.v(hb)[j] - tr.v(h2)[j] - (tr.gauge(hb) - tr.gauge(h2));
                    const double recon = p22(i, j) * std::exp(lr) * std::exp(lc);
                    CHECK(std::abs(direct(i, j) - recon) <= 1e-12 * std::max(1.0, std::abs(direct(i, j))));
                }
        }
}
TEST("adjoint: equal totals at interior boundaries (test_adjoint.cpp:212-229)") {
    InstanceSpec spec;
    spec.n_rows = spec.n_cols = 32;
    spec.half_band = 8;
    spec.base_depth = 5;
    spec.tail_depth = 4;
    spec.seed = 15;
    Ran r = run_linear(spec);
    auto c = tail_adjoint_generic(r.run.scaled, r.run.trace, r.G, r.inst.Q, r.inst.K, r.inst.V);
    for (Index t = static_cast<Index>(c.u_bar.size()) - 1; t >= 1; --t) {
        double su = 0, sv = 0;
        for (double x : c.u_bar[static_cast<size_t>(t)]) su += x;
        for (double x : c.v_bar[static_cast<size_t>(t) - 1]) sv += x;
        CHECK(std::abs(su) < 1e-10);
        CHECK(std::abs(sv) < 1e-10);
    }
}
TEST("adjoint: surrogate gradient matches FD <=1e-8 (test_adjoint.cpp:231-253)") {
    InstanceSpec spec;
    spec.n_rows = spec.n_cols = 24;
    spec.half_band = 6;
    spec.base_depth = 5;
    spec.tail_depth = 2;
    spec.seed = 16;
    Ran r = run_linear(spec);
    auto dp = dense::make_dense_problem(r.inst, r.loss);
    auto adj = tail_adjoint_generic(r.run.scaled, r.run.trace, r.G, r.inst.Q, r.inst.K, r.inst.V);
    dense::FdOptions opt;
    CHECK(dense::max_abs_diff_on(dense::finite_diff_grad(dp, dense::FdTensor::Q, opt), adj.grad_q) < 1e-8);
    CHECK(dense::max_abs_diff_on(dense::finite_diff_grad(dp, dense::FdTensor::K, opt), adj.grad_k) < 1e-8);
    CHECK(dense::max_abs_diff_on(dense::finite_diff_grad(dp, dense::FdTensor::V, opt), adj.grad_v) < 1e-8);
}
TEST("adjoint: generic R=1 and R=3 vs FD (test_adjoint.cpp:255-275)") {
    for (Index R : {1, 3}) {
        InstanceSpec spec;
        spec.n_rows = spec.n_cols = 16;
        spec.half_band = 5;
        spec.base_depth = 4;
        spec.tail_depth = R;
        spec.seed = 17 + static_cast<std::uint64_t>(R);
        Ran r = run_linear(spec);
        auto dp = dense::make_dense_problem(r.inst, r.loss);
        auto adj = tail_adjoint_generic(r.run.scaled, r.run.trace, r.G, r.inst.Q, r.inst.K, r.inst.V);
        dense::FdOptions opt;
        CHECK(dense::max_abs_diff_on(dense::finite_diff_grad(dp, dense::FdTensor::Q, opt), adj.grad_q) < 1e-8);
        CHECK(dense::max_abs_diff_on(dense::finite_diff_grad(dp, dense::FdTensor::K, opt), adj.grad_k) < 1e-8);
    }
}
TEST("adjoint: R=0 is the terminal application (test_adjoint.cpp:277-292)") {
    InstanceSpec spec;
    spec.n_rows = spec.n_cols = 16;
    spec.half_band = 5;
    spec.base_depth = 4;
    spec.tail_depth = 0;
    spec.seed = 19;
    Ran r = run_linear(spec);
    auto dp = dense::make_dense_problem(r.inst, r.loss);
    auto adj = tail_adjoint_generic(r.run.scaled, r.run.trace, r.G, r.inst.Q, r.inst.K, r.inst.V);
    dense::FdOptions opt;
    CHECK(dense::max_abs_diff_on(dense::finite_diff_grad(dp, dense::FdTensor::Q, opt), adj.grad_q) < 1e-8);
    CHECK(max_abs_diff(adj.base_u, adj.u_bar[0]) == 0.0);
    CHECK(max_abs_diff(adj.base_v, adj.v_bar[0]) == 0.0);
    CHECK(adj.base_l2() > 0.0);
}
TEST("adjoint: r2 modes agree with each other and generic <=1e-12 (test_adjoint.cpp:294-318)") {
    for (std::uint64_t seed : {20, 21, 22}) {
        InstanceSpec spec;
        spec.n_rows = spec.n_cols = 48;
        spec.half_band = 12;
        spec.base_depth = 6;
        spec.tail_depth = 2;
        spec.seed = seed;
        spec.tile_block = 16;
        Ran r = run_linear(spec);
        auto one = r2_backward(r.run.scaled, r.run.trace, r.G, r.inst.Q, r.inst.K, r.inst.V, BackwardMode::OneReference);
        auto four = r2_backward(r.run.scaled, r.run.trace, r.G, r.inst.Q, r.inst.K, r.inst.V, BackwardMode::DirectFourPlan);
        auto gen = tail_adjoint_generic(r.run.scaled, r.run.trace, r.G, r.inst.Q, r.inst.K, r.inst.V);
        CHECK(max_abs_diff(densify(one.score_bar), densify(four.score_bar)) < 1e-12);
        CHECK(max_abs_diff(one.grad_q, four.grad_q) < 1e-12);
        CHECK(max_abs_diff(one.grad_k, four.grad_k) < 1e-12);
        CHECK(max_abs_diff(one.grad_v, four.grad_v) < 1e-12);
        CHECK(max_abs_diff(densify(one.score_bar), densify(gen.score_bar)) < 1e-12);
        CHECK(max_abs_diff(one.grad_q, gen.grad_q) < 1e-12);
        CHECK(max_abs_diff(one.base_v, gen.base_v) < 1e-12);
    }
}
TEST("adjoint: r2 fast path rejects other depths (test_adjoint.cpp:320-329)") {
    InstanceSpec spec;
    spec.n_rows = spec.n_cols = 8;
    spec.half_band = 3;
    spec.base_depth = 2;
    spec.tail_depth = 1;
    Ran r = run_linear(spec);
    CHECK_THROWS_AS(r2_backward(r.run.scaled, r.run.trace, r.G, r.inst.Q, r.inst.K, r.inst.V), UnsupportedDepth);
}
TEST("adjoint: backward consumes only the stopped state (test_adjoint.cpp:331-353)") {
    InstanceSpec spec;
    spec.n_rows = spec.n_cols = 20;
    spec.half_band = 6;
    spec.base_depth = 5;
    spec.tail_depth = 2;
    spec.seed = 23;
    Ran r = run_linear(spec);
    auto ref = r2_backward(r.run.scaled, r.run.trace, r.G, r.inst.Q, r.inst.K, r.inst.V);
    DualTrace<double> scr = r.run.trace;
    for (Index h = 0; h < scr.split; ++h) {
        std::fill(scr.u_hist[static_cast<size_t>(h)].begin(), scr.u_hist[static_cast<size_t>(h)].end(), 42.0);
        std::fill(scr.v_hist[static_cast<size_t>(h)].begin(), scr.v_hist[static_cast<size_t>(h)].end(), -7.0);
    }
    auto got = r2_backward(r.run.scaled, scr, r.G, r.inst.Q, r.inst.K, r.inst.V);
    CHECK(max_abs_diff(ref.grad_q, got.grad_q) == 0.0);
    CHECK(max_abs_diff(ref.grad_k, got.grad_k) == 0.0);
    CHECK(max_abs_diff(ref.base_v, got.base_v) == 0.0);
}
TEST("adjoint: centered and uncentered give the same gradient (test_adjoint.cpp:355-376)") {
    InstanceSpec spec;
    spec.n_rows = spec.n_cols = 20;
    spec.half_band = 20;
    spec.base_depth = 2;
    spec.tail_depth = 2;
    spec.seed = 24;
    auto inst = make_instance<double>(spec);
    auto cent = run_surrogate(inst.Q, inst.K, inst.V, inst.schedule, 2, 2, inst.eps, true);
    auto plain = run_surrogate(inst.Q, inst.K, inst.V, inst.schedule, 2, 2, inst.eps, false);
    CHECK(max_abs_diff(cent.output, plain.output) < 1e-11);
    auto loss = random_linear_loss(inst);
    auto G = loss.output_cotangent(cent.output, inst.V, inst.schedule->support().row_mask());
    auto a = r2_backward(cent.scaled, cent.trace, G, inst.Q, inst.K, inst.V);
    auto b = r2_backward(plain.scaled, plain.trace, G, inst.Q, inst.K, inst.V);
    CHECK(max_abs_diff(a.grad_q, b.grad_q) < 1e-10);
    CHECK(max_abs_diff(a.grad_k, b.grad_k) < 1e-10);
    CHECK(max_abs_diff(a.grad_v, b.grad_v) < 1e-10);
}
TEST("adjoint: rectangular supports end to end (test_adjoint.cpp:378-409)") {
    const Index rows = 18, cols = 26, d = 4;
    Mat<double> Q = normal_matrix<double>(90, "Q", rows, d), K = normal_matrix<double>(90, "K", cols, d),
                V = normal_matrix<double>(90, "V", cols, d);
    auto sched = TileSchedule::build(build_band_support(rows, cols, 9), 8);
    auto run = run_surrogate(Q, K, V, sched, 4, 2, EpsSchedule<double>::single(1.0, 4));
    Mat<double> G = normal_matrix<double>(91, "G", rows, d);
    auto one = r2_backward(run.scaled, run.trace, G, Q, K, V);
    auto gen = tail_adjoint_generic(run.scaled, run.trace, G, Q, K, V);
    CHECK(max_abs_diff(one.grad_q, gen.grad_q) < 1e-12);
    CHECK(max_abs_diff(one.grad_k, gen.grad_k) < 1e-12);
    DenseProblem dp;
    dp.Q = Q;
    dp.K = K;
    dp.V = V;
    dp.support = dense::dense_support_of(sched->support());
    dp.base_depth = 4;
    dp.tail_depth = 2;
    dp.loss = LossSpec<double>::linear(G);
    CHECK(max_abs_diff(dense::dense_forward(dp).output, run.output) < 1e-12);
    dense::FdOptions opt;
    CHECK(dense::max_abs_diff_on(dense::finite_diff_grad(dp, dense::FdTensor::Q, opt), one.grad_q) < 1e-8);
    CHECK(dense::max_abs_diff_on(dense::finite_diff_grad(dp, dense::FdTensor::K, opt), one.grad_k) < 1e-8);
    CHECK(dense::max_abs_diff_on(dense::finite_diff_grad(dp, dense::FdTensor::V, opt), one.grad_v) < 1e-8);
}
TEST("adjoint: float32 tracks f64 <=1e-4 (test_adjoint.cpp:411-434)") {
    InstanceSpec spec;
    spec.n_rows = spec.n_cols = 32;
    spec.half_band = 8;
    spec.base_depth = 5;
    spec.tail_depth = 2;
    spec.seed = 25;
    auto i64 = make_instance<double>(spec);
    auto i32 = make_instance<float>(spec);
    auto r32 = run_surrogate(i32.Q, i32.K, i32.V, i32.schedule, 5, 2, i32.eps);
    auto loss = random_linear_loss(i64);
    Mat<float> G32 = loss.fixed.cast<float>();
    auto c32 = r2_backward(r32.scaled, r32.trace, G32, i32.Q, i32.K, i32.V);
    auto r64 = run_surrogate(i64.Q, i64.K, i64.V, i64.schedule, 5, 2, i64.eps);
    auto c64 = r2_backward(r64.scaled, r64.trace, loss.fixed, i64.Q, i64.K, i64.V);
    CHECK(max_abs_diff(c32.grad_q, c64.grad_q) < 1e-4);
    CHECK(max_abs_diff(c32.grad_k, c64.grad_k) < 1e-4);
    CHECK(max_abs_diff(c32.grad_v, c64.grad_v) < 1e-4);
}

// ======================= test_oracle.cpp =======================
Instance<double> make_inst(Index n, Index w, Index t, Index r, std::uint64_t seed, Index block = 32) {
    InstanceSpec spec;
    spec.n_rows = spec.n_cols = n;
    spec.half_band = w;
    spec.base_depth = t;
    spec.tail_depth = r;
    spec.seed = seed;
    spec.tile_block = block;
    return make_instance<double>(spec);
}
TEST("oracle: dense forward uniform 1/3 (test_oracle.cpp:30-42)") {
    DenseProblem p;
    p.Q = zeros(3, 2);
    p.K = zeros(3, 2);
    p.V = identity(3);
    p.support = BoolMat(3, 3, 1);
    p.base_depth = 2;
    p.tail_depth = 1;
    p.loss = LossSpec<double>::linear(zeros(3, 3));
    for (double x : dense::dense_forward(p).output.a) CHECK(std::abs(x - 1.0 / 3.0) < 1e-15);
}
TEST("oracle: blockwise vs dense on 50 random instances (test_oracle.cpp:44-58)") {
    for (std::uint64_t seed = 0; seed < 50; ++seed) {
        const Index L = 40 + 43 * (seed % 6), W = 6 + 9 * (seed % 4);
        auto inst = make_inst(L, W, 6, 2, seed, 16);
        auto run = run_surrogate(inst.Q, inst.K, inst.V, inst.schedule, 6, 2, inst.eps);
        auto dp = dense::make_dense_problem(inst, random_linear_loss(inst));
        CHECK(max_abs_diff(dense::dense_forward(dp).output, run.output) < 1e-12);
    }
}
TEST("oracle: dustbin dense equals explicit (test_oracle.cpp:60-84)") {
    InstanceSpec spec;
    spec.n_rows = spec.n_cols = 10;
    spec.half_band = 3;
    spec.base_depth = 4;
    spec.tail_depth = 2;
    spec.seed = 31;
    spec.dustbin_block = 3;
    auto inst = make_instance<double>(spec);
    auto dp = dense::make_dense_problem(inst, random_linear_loss(inst));
    auto f1 = dense::dense_forward(dp);
    const SupportMask& am = inst.schedule->support();
    std::vector<std::pair<Index, Index>> edges;
    for (Index i = 0; i < am.n_rows(); ++i) am.for_each_in_row(i, [&](Index j) { edges.emplace_back(i, j); });
    auto manual = SupportMask::explicit_edges(am.n_rows(), am.n_cols(), edges, am.row_mask(), am.col_mask());
    DenseProblem dp2 = dp;
    dp2.support = dense::dense_support_of(manual);
    CHECK(max_abs_diff(f1.output, dense::dense_forward(dp2).output) == 0.0);
}
TEST("oracle: FD reduces to plan product for a frozen plan (test_oracle.cpp:86-102)") {
    auto inst = make_inst(12, 4, 3, 0, 32);
    auto run = run_surrogate(inst.Q, inst.K, inst.V, inst.schedule, 3, 0, inst.eps);
    auto loss = random_linear_loss(inst);
    auto dp = dense::make_dense_problem(inst, loss);
    dense::FdOptions opt;
    auto fd = dense::finite_diff_grad(dp, dense::FdTensor::V, opt);
    const Index h = run.trace.steps();
    auto an = dense::matmul(dense::transpose(dense_plan_of(run.scaled, run.trace, h, h)), loss.fixed);
    CHECK(dense::max_abs_diff_on(fd, an) < 1e-9);
}
TEST("oracle: surrogate FD keeps the frozen base (test_oracle.cpp:104-120)") {
    auto inst = make_inst(16, 5, 4, 2, 33);
    auto dp = dense::make_dense_problem(inst, random_linear_loss(inst));
    DenseProblem base_only = dp;
    base_only.tail_depth = 0;
    auto base = dense::dense_forward(base_only);
    DenseProblem bumped = dp;
    for (auto& x : bumped.Q.a) x += 0.37;
    dense::FrozenBase fb{base.trace.u_hist.back(), base.trace.v_hist.back(), base.trace.gauge_hist.back()};
    auto f = dense::dense_forward_impl(bumped, fb);
    CHECK(max_abs_diff(f.trace.u_hist.front(), fb.u) == 0.0);
    CHECK(max_abs_diff(f.trace.v_hist.front(), fb.v) == 0.0);
}
TEST("oracle: full BPTT T=0 equals surrogate (test_oracle.cpp:147-154)") {
    auto inst = make_inst(16, 6, 0, 2, 35);
    auto dp = dense::make_dense_problem(inst, random_linear_loss(inst));
    auto full = dense::full_bptt_grad(dp), surr = dense::dense_surrogate_grad(dp);
    CHECK(max_abs_diff(full.grad_q, surr.grad_q) == 0.0);
    CHECK(max_abs_diff(full.grad_k, surr.grad_k) == 0.0);
}
TEST("oracle: full BPTT vs full-variant FD (test_oracle.cpp:156-168)") {
    auto inst = make_inst(20, 6, 4, 2, 36);
    auto dp = dense::make_dense_problem(inst, random_linear_loss(inst));
    auto full = dense::full_bptt_grad(dp);
    dense::FdOptions opt;
    opt.variant = dense::FdVariant::Full;
    CHECK(dense::max_abs_diff_on(dense::finite_diff_grad(dp, dense::FdTensor::Q, opt), full.grad_q) < 1e-7);
    CHECK(dense::max_abs_diff_on(dense::finite_diff_grad(dp, dense::FdTensor::K, opt), full.grad_k) < 1e-7);
    CHECK(dense::max_abs_diff_on(dense::finite_diff_grad(dp, dense::FdTensor::V, opt), full.grad_v) < 1e-7);
}
TEST("oracle: supervised value loss (test_oracle.cpp:170-196)") {
    InstanceSpec spec;
    spec.n_rows = spec.n_cols = 14;
    spec.half_band = 5;
    spec.base_depth = 3;
    spec.tail_depth = 2;
    spec.seed = 37;
    auto inst = make_instance<double>(spec);
    std::vector<Index> cols(14);
    for (Index i = 0; i < 14; ++i) cols[static_cast<size_t>(i)] = i;
    auto loss = LossSpec<double>::supervised_value_mse(cols);
    auto dp = dense::make_dense_problem(inst, loss);
    auto run = run_surrogate(inst.Q, inst.K, inst.V, inst.schedule, 3, 2, inst.eps);
    const auto& rows = inst.schedule->support().row_mask();
    auto G = loss.output_cotangent(run.output, inst.V, rows);
    auto adj = tail_adjoint_generic(run.scaled, run.trace, G, inst.Q, inst.K, inst.V);
    Mat<double> tv = adj.grad_v;
    auto D = loss.direct_value_cotangent(run.output, inst.V, rows);
    for (size_t k = 0; k < tv.a.size(); ++k) tv.a[k] += D.a[k];
    dense::FdOptions opt;
    CHECK(dense::max_abs_diff_on(dense::finite_diff_grad(dp, dense::FdTensor::V, opt), tv) < 1e-8);
    CHECK(dense::max_abs_diff_on(dense::finite_diff_grad(dp, dense::FdTensor::Q, opt), adj.grad_q) < 1e-8);
}
TEST("oracle: frobenius loss vs FD (test_oracle.cpp:198-216)") {
    auto inst = make_inst(12, 4, 3, 2, 38);
    const SupportMask& m = inst.schedule->support();
    auto loss = LossSpec<double>::frobenius_to_target(normal_matrix<double>(39, "T", m.n_rows(), inst.spec.head_dim));
    auto dp = dense::make_dense_problem(inst, loss);
    auto run = run_surrogate(inst.Q, inst.K, inst.V, inst.schedule, 3, 2, inst.eps);
    auto G = loss.output_cotangent(run.output, inst.V, m.row_mask());
    auto adj = tail_adjoint_generic(run.scaled, run.trace, G, inst.Q, inst.K, inst.V);
    dense::FdOptions opt;
    CHECK(dense::max_abs_diff_on(dense::finite_diff_grad(dp, dense::FdTensor::Q, opt), adj.grad_q) < 1e-8);
    CHECK(dense::max_abs_diff_on(dense::finite_diff_grad(dp, dense::FdTensor::V, opt), adj.grad_v) < 1e-8);
}
TEST("oracle: size caps are hard errors (test_oracle.cpp:218-240)") {
    DenseProblem p;
    p.Q = zeros(600, 2);
    p.K = zeros(600, 2);
    p.V = zeros(600, 2);
    p.support = BoolMat(600, 600, 1);
    p.base_depth = 1;
    p.loss = LossSpec<double>::linear(zeros(600, 2));
    CHECK_THROWS_AS(dense::dense_forward(p), SizeCapExceeded);
    DenseProblem q;
    q.Q = zeros(300, 2);
    q.K = zeros(300, 2);
    q.V = zeros(300, 2);
    q.support = BoolMat(300, 300, 1);
    q.base_depth = 1;
    q.loss = LossSpec<double>::linear(zeros(300, 2));
    CHECK_THROWS_AS(dense::full_bptt_grad(q), SizeCapExceeded);
}
TEST("oracle: too-small FD steps flagged (test_oracle.cpp:242-249)") {
    auto inst = make_inst(8, 3, 2, 1, 40);
    auto dp = dense::make_dense_problem(inst, random_linear_loss(inst));
    dense::FdOptions opt;
    opt.step = 1e-12;
    CHECK_THROWS_AS(dense::finite_diff_grad(dp, dense::FdTensor::Q, opt), std::invalid_argument);
}
TEST("oracle: eps-scaling dense vs tiled, FD (test_oracle.cpp:251-269)") {
    InstanceSpec spec;
    spec.n_rows = spec.n_cols = 28;
    spec.half_band = 9;
    spec.base_depth = 6;
    spec.tail_depth = 2;
    spec.seed = 41;
    spec.stages = {{3.0, 2}, {1.5, 2}, {1.0, 2}};
    auto inst = make_instance<double>(spec);
    auto run = run_surrogate(inst.Q, inst.K, inst.V, inst.schedule, 6, 2, inst.eps);
    auto dp = dense::make_dense_problem(inst, random_linear_loss(inst));
    CHECK(max_abs_diff(dense::dense_forward(dp).output, run.output) < 1e-12);
    auto G = dp.loss.output_cotangent(run.output, inst.V, inst.schedule->support().row_mask());
    auto adj = tail_adjoint_generic(run.scaled, run.trace, G, inst.Q, inst.K, inst.V);
    dense::FdOptions opt;
    CHECK(dense::max_abs_diff_on(dense::finite_diff_grad(dp, dense::FdTensor::Q, opt), adj.grad_q) < 1e-8);
}

// ======================= EXT: pins for the extensions =======================
TEST("ext: d_eps matches FD through the frozen-base surrogate") {
    for (std::uint64_t seed : {50, 51}) {
        InstanceSpec spec;
        spec.n_rows = spec.n_cols = 24;
        spec.half_band = 6;
        spec.base_depth = 5;
        spec.tail_depth = 2;
        spec.epsilon = 0.7;
        spec.seed = seed;
        Ran r = run_linear(spec);
        auto dp = dense::make_dense_problem(r.inst, r.loss);
        auto one = r2_backward(r.run.scaled, r.run.trace, r.G, r.inst.Q, r.inst.K, r.inst.V);
        auto four = r2_backward(r.run.scaled, r.run.trace, r.G, r.inst.Q, r.inst.K, r.inst.V, BackwardMode::DirectFourPlan);
        dense::FdOptions opt;
        const double fd = dense::finite_diff_grad(dp, dense::FdTensor::Eps, opt)(0, 0);
        CHECK(std::abs(fd - one.d_eps) < 1e-7 * std::max(1.0, std::abs(fd)));
        CHECK(std::abs(one.d_eps - four.d_eps) < 1e-12 * std::max(1.0, std::abs(one.d_eps)));
        // identity without dustbin: d_eps = -(1/eps) <Q, dQ>
        double qdq = 0;
        for (size_t k = 0; k < r.inst.Q.a.size(); ++k) qdq += r.inst.Q.a[k] * one.grad_q.a[k];
        CHECK(std::abs(one.d_eps + qdq / 0.7) < 1e-10 * std::max(1.0, std::abs(one.d_eps)));
        auto dg = dense::dense_surrogate_grad(dp);
        CHECK(std::abs(dg.d_eps - one.d_eps) < 1e-10 * std::max(1.0, std::abs(fd)));
    }
}
TEST("ext: masked band surrogate vs dense oracle and FD") {
    const Index L = 40, d = 6, w = 5;
    Mat<double> Q = normal_matrix<double>(60, "Q", L, d), K = normal_matrix<double>(60, "K", L, d),
                V = normal_matrix<double>(60, "V", L, d), G = normal_matrix<double>(60, "G", L, d);
    std::vector<bool> rm(L, true), cm(L, true);
    for (Index i = 29; i < L; ++i) rm[i] = cm[i] = false;  // valid length 29
    auto sup = build_band_support(L, L, w, rm, cm);
    for (Index i = 0; i < L; ++i)
        if (!rm[i]) for (Index x = 0; x < d; ++x) G(i, x) = 0;
    auto sched = TileSchedule::build(sup, 16);
    auto run = run_surrogate(Q, K, V, sched, 6, 2, EpsSchedule<double>::single(0.5, 6));
    auto one = r2_backward(run.scaled, run.trace, G, Q, K, V);
    DenseProblem dp;
    dp.Q = Q;
    dp.K = K;
    dp.V = V;
    dp.support = dense::dense_support_of(sup);
    dp.epsilon = 0.5;
    dp.base_depth = 6;
    dp.tail_depth = 2;
    dp.loss = LossSpec<double>::linear(G);
    CHECK(max_abs_diff(dense::dense_forward(dp).output, run.output) < 1e-12);
    dense::FdOptions opt;
    CHECK(dense::max_abs_diff_on(dense::finite_diff_grad(dp, dense::FdTensor::Q, opt), one.grad_q) < 1e-8);
    CHECK(dense::max_abs_diff_on(dense::finite_diff_grad(dp, dense::FdTensor::V, opt), one.grad_v) < 1e-8);
    for (Index i = 29; i < L; ++i)
        for (Index x = 0; x < d; ++x) {
            CHECK(run.output(i, x) == 0.0);
            CHECK(one.grad_q(i, x) == 0.0);
            CHECK(one.grad_k(i, x) == 0.0);
            CHECK(one.grad_v(i, x) == 0.0);
        }
}
TEST("ext: spoke dustbin constant cost == reference-semantics embedding (SURVEY App. A)") {
    const Index L = 30, d = 6, w = 4;
    const double eps = 0.4, cost = 1.0;
    Mat<double> Q = normal_matrix<double>(70, "Q", L + 1, d), K = normal_matrix<double>(70, "K", L + 1, d),
                V = normal_matrix<double>(70, "V", L + 1, d), G = normal_matrix<double>(70, "G", L + 1, d);
    std::vector<bool> rm(L, true), cm(L, true);
    for (Index i = 22; i < L; ++i) rm[i] = cm[i] = false;
    auto sup = spoke_dustbin_support(L, w, rm, cm);
    for (Index i = 0; i <= L; ++i)
        if (!sup.row_active(i)) for (Index x = 0; x < d; ++x) G(i, x) = 0;
    auto sched = TileSchedule::build(sup, 8);
    ConstantEdges<double> cst{L, L, -cost};
    auto es = EpsSchedule<double>::single(eps, 7);
    auto run = run_surrogate(Q, K, V, sched, 7, 2, es, true, &cst);
    auto one = r2_backward(run.scaled, run.trace, G, Q, K, V, BackwardMode::OneReference, &cst);
    // embedding trick: head dim d+2 reproduces q.k/sqrt(d) on band edges and -cost on dustbin edges
    const double s = std::pow((d + 2.0) / d, 0.25), r2 = std::sqrt(d + 2.0);
    Mat<double> Qe(L + 1, d + 2), Ke(L + 1, d + 2);
    for (Index i = 0; i < L; ++i) {
        for (Index x = 0; x < d; ++x) { Qe(i, x) = s * Q(i, x); Ke(i, x) = s * K(i, x); }
        Qe(i, d) = 1.0 * cost;
        Ke(i, d + 1) = 1.0;
    }
    Qe(L, d + 1) = -r2 * cost;
    Ke(L, d) = -r2;
    Ke(L, d + 1) = 1.0;
    auto run_e = run_surrogate(Qe, Ke, V, sched, 7, 2, es);
    auto one_e = r2_backward(run_e.scaled, run_e.trace, G, Qe, Ke, V);
    CHECK(max_abs_diff(run.output, run_e.output) < 1e-11);
    CHECK(max_abs_diff(one.grad_v, one_e.grad_v) < 1e-10);
    double mq = 0, mk = 0;
    for (Index i = 0; i < L; ++i)
        for (Index x = 0; x < d; ++x) {
            mq = std::max(mq, std::abs(one.grad_q(i, x) - s * one_e.grad_q(i, x)));
            mk = std::max(mk, std::abs(one.grad_k(i, x) - s * one_e.grad_k(i, x)));
        }
    CHECK(mq < 1e-10);
    CHECK(mk < 1e-10);
    for (Index x = 0; x < d; ++x) {
        CHECK(one.grad_q(L, x) == 0.0);
        CHECK(one.grad_k(L, x) == 0.0);
    }
    // dense oracle with the same constant edges agrees, incl. FD in V and eps
    DenseProblem dp;
    dp.Q = Q;
    dp.K = K;
    dp.V = V;
    dp.support = dense::dense_support_of(sup);
    dp.epsilon = eps;
    dp.base_depth = 7;
    dp.tail_depth = 2;
    dp.loss = LossSpec<double>::linear(G);
    dp.cst = &cst;
    CHECK(max_abs_diff(dense::dense_forward(dp).output, run.output) < 1e-12);
    dense::FdOptions opt;
    CHECK(dense::max_abs_diff_on(dense::finite_diff_grad(dp, dense::FdTensor::Q, opt), one.grad_q) < 1e-8);
    CHECK(dense::max_abs_diff_on(dense::finite_diff_grad(dp, dense::FdTensor::V, opt), one.grad_v) < 1e-8);
    const double fde = dense::finite_diff_grad(dp, dense::FdTensor::Eps, opt)(0, 0);
    CHECK(std::abs(fde - one.d_eps) < 1e-7 * std::max(1.0, std::abs(fde)));
}

// ---- certificates (test_certificates.cpp) -------------------------------------------------------
CertificateProblem cert_problem(Index n, Index w, Index t, std::uint64_t seed, double loss_scale = 1.0) {
    auto inst = make_inst(n, w, t, 2, seed, 64);
    CertificateProblem p;
    p.Q = inst.Q;
    p.K = inst.K;
    p.V = inst.V;
    p.schedule = inst.schedule;
    p.base_depth = t;
    p.eps = inst.eps;
    p.loss = random_linear_loss(inst, loss_scale);
    return p;
}
double mat_max_abs(const Mat<double>& m) {
    double x = 0.0;
    for (double v : m.a) x = std::max(x, std::abs(v));
    return x;
}
TEST("certificates: base-solve VJP edge cases (test_certificates.cpp:38-54)") {
    auto p = cert_problem(16, 5, 4, 50);
    auto run = run_surrogate<double>(p.Q, p.K, p.V, p.schedule, p.base_depth, 2, p.eps);
    Vec<double> z(16, 0.0), one(16, 1.0);
    auto c0 = base_solve_vjp(run.raw, run.trace, z, z, p.Q, p.K);
    CHECK(mat_max_abs(c0.grad_q) == 0.0);
    CHECK(mat_max_abs(c0.grad_k) == 0.0);
    auto cold = run_surrogate<double>(p.Q, p.K, p.V, p.schedule, 0, 2, EpsSchedule<double>::single(1.0, 0));
    auto cz = base_solve_vjp(cold.raw, cold.trace, one, one, p.Q, p.K);
    CHECK(mat_max_abs(cz.grad_q) == 0.0);
    CHECK(mat_max_abs(cz.grad_k) == 0.0);
}
TEST("certificates: remainder identity full - stopped = c_R (test_certificates.cpp:56-65)") {
    for (std::uint64_t seed : {0, 1}) {
        auto p = cert_problem(48, 16, 8, seed);
        for (Index r : {0, 1, 2}) {
            auto cert = bias_certificate(p, r);
            CHECK(cert.residual_computed);
            CHECK(cert.residual < 1e-12);
        }
    }
}
TEST("certificates: output-independent loss zeroes every field (test_certificates.cpp:67-74)") {
    auto p = cert_problem(16, 5, 4, 51, 0.0);
    auto cert = bias_certificate(p, 2);
    CHECK(cert.eta_norm == 0.0);
    CHECK(cert.c_inf == 0.0);
    CHECK(cert.max_gap == 0.0);
    CHECK(cert.residual == 0.0);
}
TEST("certificates: eta decays strictly with the tail depth (test_certificates.cpp:76-86)") {
    for (std::uint64_t seed = 0; seed < 20; ++seed) {
        auto p = cert_problem(32, 32, 10, 100 + seed);
        double prev = std::numeric_limits<double>::infinity();
        for (Index r = 0; r <= 3; ++r) {
            const double e = bias_certificate(p, r, false).eta_norm;
            CHECK(e < prev);
            prev = e;
        }
    }
}
TEST("certificates: selector returns the first feasible depth (test_certificates.cpp:106-133)") {
    auto p = cert_problem(32, 32, 10, 8);
    CHECK(select_tail_depth(p, 1e3, 4).selected == 0);
    auto s1 = select_tail_depth(p, 1e-30, 3);
    CHECK(s1.selected == -1);
    CHECK(s1.trail.size() == 4);
    const double tau = bias_certificate(p, 2, false).c_inf * 1.5;
    Index expected = -1;
    for (Index r = 0; r <= 5; ++r)
        if (bias_certificate(p, r, false).c_inf <= tau) { expected = r; break; }
    CHECK(select_tail_depth(p, tau, 5).selected == expected);
    CHECK_THROWS_AS(select_tail_depth(p, -1.0, 3), std::invalid_argument);
    CHECK_THROWS_AS(select_tail_depth(p, 1.0, 3, [](Index r) { return -static_cast<double>(r); }),
                    std::invalid_argument);
    const double bound = 1.0;
    const double tau1 = bound * bias_certificate(p, 1, false).eta_norm * 1.01;
    auto s = select_tail_depth(p, tau1, 4, [](Index r) { return static_cast<double>(r); }, &bound);
    CHECK(s.used_sufficient_bound);
    CHECK(s.selected == 1);
}

}  // namespace

int main(int argc, char** argv) {
    const char* filter = argc > 1 ? argv[1] : nullptr;
    int ran = 0;
    for (const auto& t : registry()) {
        if (filter && std::string(t.name).find(filter) == std::string::npos) continue;
        g_current = t.name;
        const int before = g_fail;
        try {
            t.fn();
        } catch (const std::exception& e) {
            ++g_fail;
            std::printf("  EXCEPTION [%s]: %s\n", t.name, e.what());
        }
        std::printf("%s %s\n", g_fail == before ? "PASS" : "FAIL", t.name);
        ++ran;
    }
    std::printf("%d tests, %d checks, %d failures\n", ran, g_checks, g_fail);
    return g_fail == 0 ? 0 : 1;
}
