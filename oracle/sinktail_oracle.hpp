// ============================================================================
// sinktail_oracle.hpp -- CPU restatement of the reference's banded balanced
// entropic-OT attention path (arxiv 2605.08123, /root/reference/proj).
//
// TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2605_08123_b200/)
// includes, links or calls this file.  Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference leg use it, as the checker
// and as the timed "reference CPU path".
//
// Why a restatement: the reference is header-only C++20 over Eigen3
// (proj/CMakeLists.txt:10, include/sinktail/types.hpp:3) plus vendored
// json.hpp/CLI11.hpp/doctest.h (proj/CMakeLists.txt:18) -- none of which is
// present in this image, so the reference cannot be compiled here.  Eigen is
// the third-party dependency holding the path's arithmetic (GEMMs, matvecs,
// elementwise exp); its version is unpinned ("Eigen3 3.3 REQUIRED",
// proj/CMakeLists.txt:10).  Here every Eigen expression is spelled out as the
// plain loop it denotes (row-major storage, inc/types.hpp:10-11).
//
// Pinning: the restatement is checked against every known-answer test of the
// reference's own suites for this path (proj/tests/test_support.cpp,
// test_sinkhorn.cpp, test_adjoint.cpp, test_oracle.cpp, test_io.cpp) --
// ported one-for-one in oracle/kat_tests.cpp -- and against the analytic pins
// those tests hold (u=-ln2, 2x2 staircase plans 0.5, band count 32,521,216,
// RNG flat-index identity, ...).  There are no stored golden vectors in the
// reference.
//
// Extensions the reference lacks (each marked EXT below): batch/head loop,
// sparse-spoke dustbin support with a constant dustbin cost, d(epsilon),
// bf16 input rounding.
// ============================================================================
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <limits>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

namespace stoc {

using Index = std::int64_t;

// ---------------------------------------------------------------------------
// Errors -- include/sinktail/errors.hpp:10-39
// ---------------------------------------------------------------------------
struct InfeasibleSupport : std::runtime_error {
    explicit InfeasibleSupport(const std::string& w) : std::runtime_error(w) {}
};
struct InvalidTemperature : std::runtime_error {
    explicit InvalidTemperature(const std::string& w) : std::runtime_error(w) {}
};
struct UnsupportedDepth : std::runtime_error {
    explicit UnsupportedDepth(const std::string& w) : std::runtime_error(w) {}
};
struct SizeCapExceeded : std::runtime_error {
    explicit SizeCapExceeded(const std::string& w) : std::runtime_error(w) {}
};
struct MissingBaseTrace : std::runtime_error {
    explicit MissingBaseTrace(const std::string& w) : std::runtime_error(w) {}
};

// ---------------------------------------------------------------------------
// Minimal row-major matrix / vector (stand-ins for inc/types.hpp:10-21)
// ---------------------------------------------------------------------------
template <class T>
struct Mat {
    Index r = 0, c = 0;
    std::vector<T> a;
    Mat() = default;
    Mat(Index rows, Index cols, T fill = T(0))
        : r(rows), c(cols), a(static_cast<size_t>(rows * cols), fill) {}
    Index rows() const { return r; }
    Index cols() const { return c; }
    T& operator()(Index i, Index j) { return a[static_cast<size_t>(i * c + j)]; }
    const T& operator()(Index i, Index j) const { return a[static_cast<size_t>(i * c + j)]; }
    T* row(Index i) { return a.data() + i * c; }
    const T* row(Index i) const { return a.data() + i * c; }
    void set_zero() { std::fill(a.begin(), a.end(), T(0)); }
    template <class U>
    Mat<U> cast() const {
        Mat<U> m(r, c);
        for (size_t k = 0; k < a.size(); ++k) m.a[k] = static_cast<U>(a[k]);
        return m;
    }
};
template <class T>
using Vec = std::vector<T>;
using BoolMat = Mat<unsigned char>;

template <class T>
double max_abs(const Mat<T>& m) {
    double mx = 0;
    for (const T& x : m.a) mx = std::max(mx, std::abs(static_cast<double>(x)));
    return mx;
}
template <class T>
double max_abs(const Vec<T>& v) {
    double mx = 0;
    for (const T& x : v) mx = std::max(mx, std::abs(static_cast<double>(x)));
    return mx;
}
template <class A, class B>
double max_abs_diff(const Mat<A>& x, const Mat<B>& y) {
    double mx = 0;
    for (size_t k = 0; k < x.a.size(); ++k)
        mx = std::max(mx, std::abs(static_cast<double>(x.a[k]) - static_cast<double>(y.a[k])));
    return mx;
}
template <class A, class B>
double max_abs_diff(const Vec<A>& x, const Vec<B>& y) {
    double mx = 0;
    for (size_t k = 0; k < x.size(); ++k)
        mx = std::max(mx, std::abs(static_cast<double>(x[k]) - static_cast<double>(y[k])));
    return mx;
}

// ---------------------------------------------------------------------------
// Counter RNG -- include/sinktail/rng.hpp:14-56 (bit-exact restatement)
// ---------------------------------------------------------------------------
inline std::uint64_t splitmix64(std::uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
// rng.hpp:21-27
inline std::uint64_t fold_tag(std::uint64_t seed, std::string_view tag) {
    std::uint64_t h = splitmix64(seed ^ 0x5bf03635d78d672dULL);
    for (char ch : tag) h = splitmix64(h ^ static_cast<std::uint64_t>(static_cast<unsigned char>(ch)));
    return h;
}
// rng.hpp:30-35 -- uniform in [2^-53, 1)
inline double counter_uniform(std::uint64_t key) {
    const std::uint64_t bits = splitmix64(key);
    double u = static_cast<double>(bits >> 11) * 0x1.0p-53;
    if (u <= 0.0) u = 0x1.0p-53;
    return u;
}
// rng.hpp:38-43 -- Box-Muller on the (2n, 2n+1) pair of the stream
inline double counter_normal_base(std::uint64_t base, std::uint64_t index) {
    const double u1 = counter_uniform(base + 2 * index);
    const double u2 = counter_uniform(base + 2 * index + 1);
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
}
inline double counter_normal(std::uint64_t seed, std::string_view tag, std::uint64_t index) {
    return counter_normal_base(fold_tag(seed, tag), index);
}
// rng.hpp:45-56 -- flat row-major index, scale applied in double then cast
template <class T>
Mat<T> normal_matrix(std::uint64_t seed, std::string_view tag, Index rows, Index cols,
                     double scale = 1.0) {
    Mat<T> m(rows, cols);
    const std::uint64_t base = fold_tag(seed, tag);
    for (Index i = 0; i < rows; ++i)
        for (Index j = 0; j < cols; ++j)
            m(i, j) = static_cast<T>(scale * counter_normal_base(base, static_cast<std::uint64_t>(i * cols + j)));
    return m;
}

// ---------------------------------------------------------------------------
// Support -- include/sinktail/support.hpp:15-172, proj/src/support.cpp:1-216
// ---------------------------------------------------------------------------
enum class SupportKind { Banded, Explicit, Augmented };

class SupportMask {
public:
    SupportMask() = default;

    // support.cpp:20-32
    static SupportMask banded(Index n_rows, Index n_cols, Index half_band,
                              std::vector<bool> row_active = {}, std::vector<bool> col_active = {}) {
        if (n_rows < 1 || n_cols < 1) throw std::invalid_argument("support dimensions must be >= 1");
        if (half_band < 0) throw std::invalid_argument("half band width must be >= 0");
        SupportMask m;
        m.kind_ = SupportKind::Banded;
        m.n_rows_ = n_rows;
        m.n_cols_ = n_cols;
        m.half_band_ = half_band;
        m.row_active_ = resolve(std::move(row_active), n_rows, "row");
        m.col_active_ = resolve(std::move(col_active), n_cols, "col");
        return m;
    }
    // support.cpp:34-60 -- sorted, deduplicated CSR; edges on inactive rows/cols dropped
    static SupportMask explicit_edges(Index n_rows, Index n_cols,
                                      std::vector<std::pair<Index, Index>> edges,
                                      std::vector<bool> row_active = {},
                                      std::vector<bool> col_active = {}) {
        if (n_rows < 1 || n_cols < 1) throw std::invalid_argument("support dimensions must be >= 1");
        SupportMask m;
        m.kind_ = SupportKind::Explicit;
        m.n_rows_ = n_rows;
        m.n_cols_ = n_cols;
        m.row_active_ = resolve(std::move(row_active), n_rows, "row");
        m.col_active_ = resolve(std::move(col_active), n_cols, "col");
        std::sort(edges.begin(), edges.end());
        edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
        m.row_ptr_.assign(static_cast<size_t>(n_rows) + 1, 0);
        m.col_idx_.reserve(edges.size());
        for (const auto& e : edges) {
            const Index i = e.first, j = e.second;
            if (i < 0 || i >= n_rows || j < 0 || j >= n_cols) throw std::invalid_argument("edge index out of range");
            if (!m.row_active_[static_cast<size_t>(i)] || !m.col_active_[static_cast<size_t>(j)]) continue;
            m.row_ptr_[static_cast<size_t>(i) + 1]++;
            m.col_idx_.push_back(j);
        }
        for (size_t i = 1; i < m.row_ptr_.size(); ++i) m.row_ptr_[i] += m.row_ptr_[i - 1];
        return m;
    }

    SupportKind kind() const { return kind_; }
    Index n_rows() const { return n_rows_; }
    Index n_cols() const { return n_cols_; }
    Index half_band() const { return half_band_; }
    Index dustbin_block() const { return dustbin_block_; }
    bool row_active(Index i) const { return row_active_[static_cast<size_t>(i)]; }
    bool col_active(Index j) const { return col_active_[static_cast<size_t>(j)]; }
    const std::vector<bool>& row_mask() const { return row_active_; }
    const std::vector<bool>& col_mask() const { return col_active_; }

    // support.cpp:62-73
    bool contains(Index i, Index j) const {
        if (i < 0 || i >= n_rows_ || j < 0 || j >= n_cols_) return false;
        if (!row_active(i) || !col_active(j)) return false;
        if (kind_ == SupportKind::Explicit) {
            const size_t lo = row_ptr_[static_cast<size_t>(i)], hi = row_ptr_[static_cast<size_t>(i) + 1];
            return std::binary_search(col_idx_.begin() + static_cast<std::ptrdiff_t>(lo),
                                      col_idx_.begin() + static_cast<std::ptrdiff_t>(hi), j);
        }
        const Index diff = i > j ? i - j : j - i;
        return diff <= half_band_;
    }

    // support.hpp:49-63 -- active columns of row i in ascending order
    template <class Fn>
    void for_each_in_row(Index i, Fn&& fn) const {
        if (!row_active(i)) return;
        if (kind_ == SupportKind::Explicit) {
            const size_t lo = row_ptr_[static_cast<size_t>(i)], hi = row_ptr_[static_cast<size_t>(i) + 1];
            for (size_t k = lo; k < hi; ++k) fn(col_idx_[k]);
        } else {
            const Index lo = std::max<Index>(0, i - half_band_);
            const Index hi = std::min<Index>(n_cols_ - 1, i + half_band_);
            for (Index j = lo; j <= hi; ++j)
                if (col_active(j)) fn(j);
        }
    }

    std::int64_t active_edge_count() const {
        std::int64_t n = 0;
        for (Index i = 0; i < n_rows_; ++i) for_each_in_row(i, [&](Index) { ++n; });
        return n;
    }

    // support.cpp:91-109
    void validate() const {
        std::vector<bool> col_hit(static_cast<size_t>(n_cols_), false);
        for (Index i = 0; i < n_rows_; ++i) {
            if (!row_active(i)) continue;
            Index deg = 0;
            for_each_in_row(i, [&](Index j) {
                ++deg;
                col_hit[static_cast<size_t>(j)] = true;
            });
            if (deg == 0) throw InfeasibleSupport("active row " + std::to_string(i) + " has no active edge");
        }
        for (Index j = 0; j < n_cols_; ++j)
            if (col_active(j) && !col_hit[static_cast<size_t>(j)])
                throw InfeasibleSupport("active column " + std::to_string(j) + " has no active edge");
    }

    SupportKind kind_ = SupportKind::Banded;
    Index n_rows_ = 0, n_cols_ = 0, half_band_ = 0, dustbin_block_ = 0;
    std::vector<bool> row_active_, col_active_;
    std::vector<size_t> row_ptr_;
    std::vector<Index> col_idx_;

private:
    static std::vector<bool> resolve(std::vector<bool> mask, Index n, const char* side) {
        if (mask.empty()) return std::vector<bool>(static_cast<size_t>(n), true);
        if (static_cast<Index>(mask.size()) != n)
            throw std::invalid_argument(std::string(side) + " mask size does not match dimension");
        return mask;
    }
};

// support.cpp:111-117
inline SupportMask build_band_support(Index n_rows, Index n_cols, Index half_band,
                                      std::vector<bool> row_mask = {}, std::vector<bool> col_mask = {}) {
    SupportMask m = SupportMask::banded(n_rows, n_cols, half_band, std::move(row_mask), std::move(col_mask));
    m.validate();
    return m;
}

// support.hpp:92-103, support.cpp:119-148 -- the reference's dustbin realization:
// one active slack token per side + (B-1) inert fillers, band widened to max(W, L).
struct AugmentedSupport {
    SupportMask mask, base;
    Index dustbin_row = 0, dustbin_col = 0, effective_band = 0;
    std::vector<Index> filler_rows, filler_cols;
};

inline AugmentedSupport augment_dustbin(const SupportMask& base, Index dustbin_block) {
    if (dustbin_block < 1) throw std::invalid_argument("dustbin block must be >= 1");
    base.validate();
    AugmentedSupport aug;
    aug.base = base;
    const Index rows = base.n_rows() + dustbin_block, cols = base.n_cols() + dustbin_block;
    aug.dustbin_row = base.n_rows();
    aug.dustbin_col = base.n_cols();
    aug.effective_band = std::max(base.half_band(), std::max(base.n_rows(), base.n_cols()));
    std::vector<bool> ra(static_cast<size_t>(rows), false), ca(static_cast<size_t>(cols), false);
    for (Index i = 0; i < base.n_rows(); ++i) ra[static_cast<size_t>(i)] = base.row_active(i);
    for (Index j = 0; j < base.n_cols(); ++j) ca[static_cast<size_t>(j)] = base.col_active(j);
    ra[static_cast<size_t>(aug.dustbin_row)] = true;
    ca[static_cast<size_t>(aug.dustbin_col)] = true;
    for (Index k = 1; k < dustbin_block; ++k) {
        aug.filler_rows.push_back(aug.dustbin_row + k);
        aug.filler_cols.push_back(aug.dustbin_col + k);
    }
    aug.mask = SupportMask::banded(rows, cols, aug.effective_band, std::move(ra), std::move(ca));
    aug.mask.kind_ = SupportKind::Augmented;
    aug.mask.dustbin_block_ = dustbin_block;
    aug.mask.validate();
    return aug;
}

// EXT (BASELINE config 3): sparse-spoke support
//   band(half_band) on [0,L) x [0,L)  U  {(i, L)}  U  {(L, j)}  U  {(L, L)}
// on active rows/cols, realized through the reference's explicit_edges.
inline SupportMask spoke_dustbin_support(Index L, Index half_band, const std::vector<bool>& row_mask,
                                         const std::vector<bool>& col_mask) {
    std::vector<bool> ra(static_cast<size_t>(L + 1), true), ca(static_cast<size_t>(L + 1), true);
    for (Index i = 0; i < L; ++i) {
        ra[static_cast<size_t>(i)] = row_mask.empty() ? true : row_mask[static_cast<size_t>(i)];
        ca[static_cast<size_t>(i)] = col_mask.empty() ? true : col_mask[static_cast<size_t>(i)];
    }
    std::vector<std::pair<Index, Index>> edges;
    for (Index i = 0; i < L; ++i) {
        const Index lo = std::max<Index>(0, i - half_band), hi = std::min<Index>(L - 1, i + half_band);
        for (Index j = lo; j <= hi; ++j) edges.emplace_back(i, j);
        edges.emplace_back(i, L);
        edges.emplace_back(L, i);
    }
    edges.emplace_back(L, L);
    SupportMask m = SupportMask::explicit_edges(L + 1, L + 1, std::move(edges), ra, ca);
    m.validate();
    return m;
}

struct TileRange {
    Index row_begin = 0, row_end = 0, col_begin = 0, col_end = 0;
    Index rows() const { return row_end - row_begin; }
    Index cols() const { return col_end - col_begin; }
};

// support.cpp:150-186 -- row-major BxB cover, empty tiles dropped
class TileSchedule {
public:
    static std::shared_ptr<const TileSchedule> build(SupportMask support, Index block) {
        if (block < 1) throw std::invalid_argument("tile block must be >= 1");
        support.validate();
        auto s = std::make_shared<TileSchedule>();
        s->block_ = block;
        s->support_ = std::move(support);
        const SupportMask& m = s->support_;
        const Index rt = (m.n_rows() + block - 1) / block, ct = (m.n_cols() + block - 1) / block;
        for (Index bi = 0; bi < rt; ++bi) {
            for (Index bj = 0; bj < ct; ++bj) {
                TileRange r;
                r.row_begin = bi * block;
                r.row_end = std::min(m.n_rows(), r.row_begin + block);
                r.col_begin = bj * block;
                r.col_end = std::min(m.n_cols(), r.col_begin + block);
                BoolMat act(r.rows(), r.cols(), 0);
                std::int64_t edges = 0;
                for (Index i = r.row_begin; i < r.row_end; ++i) {
                    if (!m.row_active(i)) continue;
                    m.for_each_in_row(i, [&](Index j) {
                        if (j >= r.col_begin && j < r.col_end) {
                            act(i - r.row_begin, j - r.col_begin) = 1;
                            ++edges;
                        }
                    });
                }
                if (edges > 0) {
                    s->tiles_.push_back(r);
                    s->activity_.push_back(std::move(act));
                    s->active_edges_ += edges;
                }
            }
        }
        return s;
    }
    Index block() const { return block_; }
    const SupportMask& support() const { return support_; }
    const std::vector<TileRange>& tiles() const { return tiles_; }
    size_t tile_count() const { return tiles_.size(); }
    const BoolMat& tile_activity(size_t t) const { return activity_[t]; }
    std::int64_t active_edges() const { return active_edges_; }

private:
    Index block_ = 0;
    SupportMask support_;
    std::vector<TileRange> tiles_;
    std::vector<BoolMat> activity_;
    std::int64_t active_edges_ = 0;
};

// support.cpp:188-192
inline std::int64_t banded_entry_count(Index L, Index half_band) {
    const std::int64_t W = std::min<std::int64_t>(half_band, L - 1);
    return L * (2 * W + 1) - W * (W + 1);
}

// support.cpp:194-216 (analytic storage ledger)
struct LedgerReport {
    std::int64_t active_entries = 0, direct_plan_bytes = 0, one_reference_plan_bytes = 0,
                 direct_tile_bytes = 0, one_reference_tile_bytes = 0, tail_dual_bytes = 0,
                 base_tail_dual_bytes = 0, qkv_bytes = 0;
};
inline LedgerReport estimate_memory_ledger(Index L, Index W, Index B, Index d, Index bps, Index R, Index T) {
    if (L < 1 || B < 1 || d < 1 || bps < 1) throw std::invalid_argument("ledger parameters must be >= 1");
    LedgerReport r;
    r.active_entries = banded_entry_count(L, W);
    r.direct_plan_bytes = 4 * r.active_entries * bps;
    r.one_reference_plan_bytes = r.active_entries * bps;
    r.direct_tile_bytes = 4 * B * B * bps;
    r.one_reference_tile_bytes = B * B * bps;
    r.tail_dual_bytes = 2 * (R + 1) * L * bps;
    r.base_tail_dual_bytes = 2 * (T + R + 1) * L * bps;
    r.qkv_bytes = 3 * L * d * bps;
    return r;
}
inline std::string mib_string(std::int64_t bytes, int decimals) {
    char buf[64];
    std::snprintf(buf, sizeof(buf), "%.*f", decimals, static_cast<double>(bytes) / (1024.0 * 1024.0));
    return buf;
}

// ---------------------------------------------------------------------------
// Score field -- include/sinktail/score.hpp:14-85
// ---------------------------------------------------------------------------
template <class T>
struct BlockField {
    std::shared_ptr<const TileSchedule> schedule;
    std::vector<Mat<T>> blocks;
    BlockField() = default;
    explicit BlockField(std::shared_ptr<const TileSchedule> s) : schedule(std::move(s)) {
        blocks.reserve(schedule->tile_count());
        for (const TileRange& t : schedule->tiles()) blocks.emplace_back(t.rows(), t.cols());
    }
};

template <class T>
struct ScoreField {
    T epsilon = T(1);
    bool raw = false;
    BlockField<T> values;
    const TileSchedule& sched() const { return *values.schedule; }
    const SupportMask& support() const { return values.schedule->support(); }
};

// EXT: constant-score edges for the spoke dustbin (config 3).  Edges in row
// `row` or column `col` carry the raw score `value` instead of QK^T/sqrt(d).
template <class T>
struct ConstantEdges {
    Index row = -1, col = -1;
    T value = T(0);
    bool hit(Index i, Index j) const { return i == row || j == col; }
};

// score.hpp:40-63 (+ EXT constant edges)
template <class T>
ScoreField<T> scaled_scores(const Mat<T>& Q, const Mat<T>& K, T epsilon,
                            std::shared_ptr<const TileSchedule> schedule,
                            const ConstantEdges<T>* cst = nullptr) {
    if (!(epsilon > T(0))) throw InvalidTemperature("epsilon must be > 0");
    if (Q.cols() != K.cols()) throw std::invalid_argument("Q and K head dimensions differ");
    const SupportMask& m = schedule->support();
    if (Q.rows() != m.n_rows() || K.rows() != m.n_cols())
        throw std::invalid_argument("Q/K row counts do not match the support");
    const Index d = Q.cols();
    const T inv = T(1) / (std::sqrt(static_cast<T>(d)) * epsilon);
    ScoreField<T> s;
    s.epsilon = epsilon;
    s.raw = false;
    s.values = BlockField<T>(schedule);
    for (size_t t = 0; t < schedule->tile_count(); ++t) {
        const TileRange& r = schedule->tiles()[t];
        const BoolMat& act = schedule->tile_activity(t);
        Mat<T>& blk = s.values.blocks[t];
        for (Index i = 0; i < r.rows(); ++i) {
            const T* q = Q.row(r.row_begin + i);
            for (Index j = 0; j < r.cols(); ++j) {
                if (!act(i, j)) { blk(i, j) = T(0); continue; }
                T acc = 0;
                const T* k = K.row(r.col_begin + j);
                for (Index x = 0; x < d; ++x) acc += q[x] * k[x];
                blk(i, j) = acc * inv;
                if (cst && cst->hit(r.row_begin + i, r.col_begin + j)) blk(i, j) = cst->value / epsilon;
            }
        }
    }
    return s;
}
// score.hpp:65-72
template <class T>
ScoreField<T> raw_scores(const Mat<T>& Q, const Mat<T>& K, std::shared_ptr<const TileSchedule> s,
                         const ConstantEdges<T>* cst = nullptr) {
    ScoreField<T> f = scaled_scores<T>(Q, K, T(1), std::move(s), cst);
    f.raw = true;
    return f;
}
// score.hpp:74-85
template <class T>
ScoreField<T> scale_to_temperature(const ScoreField<T>& raw, T epsilon) {
    if (!(epsilon > T(0))) throw InvalidTemperature("epsilon must be > 0");
    if (!raw.raw) throw std::invalid_argument("scale_to_temperature expects a raw score field");
    ScoreField<T> s;
    s.epsilon = epsilon;
    s.raw = false;
    s.values.schedule = raw.values.schedule;
    s.values.blocks.reserve(raw.values.blocks.size());
    for (const auto& blk : raw.values.blocks) {
        Mat<T> b = blk;
        for (auto& x : b.a) x = x / epsilon;
        s.values.blocks.push_back(std::move(b));
    }
    return s;
}

// ---------------------------------------------------------------------------
// Epsilon schedule and dual trace -- include/sinktail/trace.hpp:12-86
// ---------------------------------------------------------------------------
template <class T>
struct EpsSchedule {
    struct Stage { T epsilon; Index iterations; };
    std::vector<Stage> stages;
    static EpsSchedule single(T eps, Index iters) {
        EpsSchedule s;
        s.stages.push_back({eps, iters});
        return s;
    }
    Index total_iterations() const {
        Index n = 0;
        for (const Stage& s : stages) n += s.iterations;
        return n;
    }
    T final_epsilon() const {
        if (stages.empty()) throw InvalidTemperature("empty epsilon schedule");
        return stages.back().epsilon;
    }
    void validate(Index base_depth) const {
        if (stages.empty()) throw InvalidTemperature("empty epsilon schedule");
        T prev = stages.front().epsilon;
        for (const Stage& s : stages) {
            if (!(s.epsilon > T(0))) throw InvalidTemperature("stage epsilon must be > 0");
            if (s.epsilon > prev) throw InvalidTemperature("stage epsilons must be non-increasing");
            if (s.iterations < 0) throw std::invalid_argument("stage iterations must be >= 0");
            prev = s.epsilon;
        }
        if (total_iterations() != base_depth) throw std::invalid_argument("epsilon schedule iterations do not sum to T");
    }
};

template <class T>
struct DualTrace {
    std::vector<Vec<T>> u_hist, v_hist;
    std::vector<T> gauge_hist, eps_hist;
    std::vector<int> stage_hist;
    Index split = 0;
    bool centered = true;
    Index steps() const { return static_cast<Index>(u_hist.size()) - 1; }
    Index tail_depth() const { return steps() - split; }
    const Vec<T>& u(Index h) const { return u_hist[static_cast<size_t>(h)]; }
    const Vec<T>& v(Index h) const { return v_hist[static_cast<size_t>(h)]; }
    T gauge(Index h) const {
        if (!centered || gauge_hist.empty()) return T(0);
        return gauge_hist[static_cast<size_t>(h)];
    }
    T eps_at(Index h) const { return eps_hist[static_cast<size_t>(h)]; }
    int stage_at(Index h) const { return stage_hist[static_cast<size_t>(h)]; }
    Index tail_step(Index r) const { return split + r; }
    const Vec<T>& tail_u(Index r) const { return u(split + r); }
    const Vec<T>& tail_v(Index r) const { return v(split + r); }
    T tail_gauge(Index r) const { return gauge(split + r) - gauge(split); }
};

// ---------------------------------------------------------------------------
// Sinkhorn core -- include/sinktail/sinkhorn.hpp:15-302
// ---------------------------------------------------------------------------
// sinkhorn.hpp:15-61 -- two-pass (max, then exp-sum) row log-sum-exp
template <class T>
Vec<T> row_half_step(const ScoreField<T>& S, const Vec<T>& v) {
    const TileSchedule& sched = S.sched();
    const SupportMask& m = sched.support();
    const Index n = m.n_rows();
    const T ninf = -std::numeric_limits<T>::infinity();
    Vec<T> row_max(static_cast<size_t>(n), ninf);
    for (size_t t = 0; t < sched.tile_count(); ++t) {
        const TileRange& r = sched.tiles()[t];
        const Mat<T>& blk = S.values.blocks[t];
        const BoolMat& act = sched.tile_activity(t);
        for (Index i = 0; i < r.rows(); ++i) {
            T mx = row_max[static_cast<size_t>(r.row_begin + i)];
            for (Index j = 0; j < r.cols(); ++j) {
                if (!act(i, j)) continue;
                const T x = blk(i, j) + v[static_cast<size_t>(r.col_begin + j)];
                if (x > mx) mx = x;
            }
            row_max[static_cast<size_t>(r.row_begin + i)] = mx;
        }
    }
    Vec<T> acc(static_cast<size_t>(n), T(0));
    for (size_t t = 0; t < sched.tile_count(); ++t) {
        const TileRange& r = sched.tiles()[t];
        const Mat<T>& blk = S.values.blocks[t];
        const BoolMat& act = sched.tile_activity(t);
        for (Index i = 0; i < r.rows(); ++i) {
            const T mx = row_max[static_cast<size_t>(r.row_begin + i)];
            T sum = 0;
            for (Index j = 0; j < r.cols(); ++j) {
                if (!act(i, j)) continue;
                sum += std::exp(blk(i, j) + v[static_cast<size_t>(r.col_begin + j)] - mx);
            }
            acc[static_cast<size_t>(r.row_begin + i)] += sum;
        }
    }
    Vec<T> u(static_cast<size_t>(n), T(0));
    for (Index i = 0; i < n; ++i) {
        if (!m.row_active(i)) continue;
        const size_t k = static_cast<size_t>(i);
        if (!(acc[k] > T(0)) || !std::isfinite(row_max[k]))
            throw InfeasibleSupport("active row " + std::to_string(i) + " has empty reduction");
        u[k] = -(row_max[k] + std::log(acc[k]));
    }
    return u;
}

// sinkhorn.hpp:64-107 -- transpose analogue
template <class T>
Vec<T> col_half_step(const ScoreField<T>& S, const Vec<T>& u) {
    const TileSchedule& sched = S.sched();
    const SupportMask& m = sched.support();
    const Index n = m.n_cols();
    const T ninf = -std::numeric_limits<T>::infinity();
    Vec<T> col_max(static_cast<size_t>(n), ninf);
    for (size_t t = 0; t < sched.tile_count(); ++t) {
        const TileRange& r = sched.tiles()[t];
        const Mat<T>& blk = S.values.blocks[t];
        const BoolMat& act = sched.tile_activity(t);
        for (Index i = 0; i < r.rows(); ++i) {
            const T ui = u[static_cast<size_t>(r.row_begin + i)];
            for (Index j = 0; j < r.cols(); ++j) {
                if (!act(i, j)) continue;
                const T x = blk(i, j) + ui;
                T& cm = col_max[static_cast<size_t>(r.col_begin + j)];
                if (x > cm) cm = x;
            }
        }
    }
    Vec<T> acc(static_cast<size_t>(n), T(0));
    for (size_t t = 0; t < sched.tile_count(); ++t) {
        const TileRange& r = sched.tiles()[t];
        const Mat<T>& blk = S.values.blocks[t];
        const BoolMat& act = sched.tile_activity(t);
        for (Index i = 0; i < r.rows(); ++i) {
            const T ui = u[static_cast<size_t>(r.row_begin + i)];
            for (Index j = 0; j < r.cols(); ++j) {
                if (!act(i, j)) continue;
                const size_t c = static_cast<size_t>(r.col_begin + j);
                acc[c] += std::exp(blk(i, j) + ui - col_max[c]);
            }
        }
    }
    Vec<T> v(static_cast<size_t>(n), T(0));
    for (Index j = 0; j < n; ++j) {
        if (!m.col_active(j)) continue;
        const size_t k = static_cast<size_t>(j);
        if (!(acc[k] > T(0)) || !std::isfinite(col_max[k]))
            throw InfeasibleSupport("active column " + std::to_string(j) + " has empty reduction");
        v[k] = -(col_max[k] + std::log(acc[k]));
    }
    return v;
}

template <class T>
struct CenterResult { Vec<T> u, v; T shift; };

// sinkhorn.hpp:118-140 -- subtract mean of u over valid rows, add it to all of v
template <class T>
CenterResult<T> center(const Vec<T>& u, const Vec<T>& v, const std::vector<bool>& valid) {
    T sum = 0;
    Index count = 0;
    for (size_t i = 0; i < u.size(); ++i)
        if (valid[i]) { sum += u[i]; ++count; }
    if (count == 0) throw InfeasibleSupport("centering requires at least one valid query");
    const T c = sum / static_cast<T>(count);
    CenterResult<T> out{u, v, c};
    for (size_t i = 0; i < u.size(); ++i)
        if (valid[i]) out.u[i] -= c;
    for (auto& x : out.v) x += c;
    return out;
}

// sinkhorn.hpp:146-164
template <class T>
void advance_full_step(const ScoreField<T>& S, DualTrace<T>& trace, int stage_id) {
    const SupportMask& m = S.support();
    Vec<T> u_next = row_half_step(S, trace.v_hist.back());
    Vec<T> v_next = col_half_step(S, u_next);
    T shift = 0;
    if (trace.centered) {
        CenterResult<T> c = center(u_next, v_next, m.row_mask());
        u_next = std::move(c.u);
        v_next = std::move(c.v);
        shift = c.shift;
    }
    trace.u_hist.push_back(std::move(u_next));
    trace.v_hist.push_back(std::move(v_next));
    if (trace.centered) trace.gauge_hist.push_back(trace.gauge_hist.back() + shift);
    trace.eps_hist.push_back(S.epsilon);
    trace.stage_hist.push_back(stage_id);
}

// sinkhorn.hpp:171-198 -- cold start u = v = 0
template <class T>
DualTrace<T> stopped_base_solve(const ScoreField<T>& raw, Index base_depth, const EpsSchedule<T>& schedule,
                                bool centered = true) {
    if (!raw.raw) throw std::invalid_argument("stopped_base_solve expects raw (unscaled) scores");
    schedule.validate(base_depth);
    const SupportMask& m = raw.support();
    DualTrace<T> tr;
    tr.centered = centered;
    tr.u_hist.push_back(Vec<T>(static_cast<size_t>(m.n_rows()), T(0)));
    tr.v_hist.push_back(Vec<T>(static_cast<size_t>(m.n_cols()), T(0)));
    if (centered) tr.gauge_hist.push_back(T(0));
    tr.eps_hist.push_back(T(0));
    tr.stage_hist.push_back(-1);
    int stage_id = 0;
    for (const auto& stage : schedule.stages) {
        if (stage.iterations > 0) {
            const ScoreField<T> S = scale_to_temperature(raw, stage.epsilon);
            for (Index k = 0; k < stage.iterations; ++k) advance_full_step(S, tr, stage_id);
        }
        ++stage_id;
    }
    tr.split = tr.steps();
    return tr;
}

// sinkhorn.hpp:203-221
template <class T>
void tail_refine(const ScoreField<T>& raw, DualTrace<T>& tr, Index tail_depth, T final_eps) {
    if (!raw.raw) throw std::invalid_argument("tail_refine expects raw (unscaled) scores");
    if (tail_depth < 0) throw std::invalid_argument("tail depth must be >= 0");
    if (tr.steps() != tr.split) throw std::invalid_argument("trace already has a tail");
    int tail_stage = 0;
    if (tr.split > 0) {
        tail_stage = tr.stage_at(tr.split);
        if (tr.eps_at(tr.split) != final_eps) ++tail_stage;
    }
    if (tail_depth > 0) {
        const ScoreField<T> S = scale_to_temperature(raw, final_eps);
        for (Index r = 0; r < tail_depth; ++r) advance_full_step(S, tr, tail_stage);
    }
}

// sinkhorn.hpp:226-240 -- P_ij = exp(S_ij + u_i + v_j + log_gauge) on support
template <class T>
Mat<T> plan_tile(const ScoreField<T>& S, size_t tile, const Vec<T>& u, const Vec<T>& v, T log_gauge = T(0)) {
    const TileRange& r = S.sched().tiles()[tile];
    const BoolMat& act = S.sched().tile_activity(tile);
    const Mat<T>& blk = S.values.blocks[tile];
    Mat<T> p(r.rows(), r.cols());
    for (Index i = 0; i < r.rows(); ++i) {
        const T ui = u[static_cast<size_t>(r.row_begin + i)] + log_gauge;
        for (Index j = 0; j < r.cols(); ++j)
            p(i, j) = act(i, j) ? std::exp(blk(i, j) + ui + v[static_cast<size_t>(r.col_begin + j)]) : T(0);
    }
    return p;
}

// sinkhorn.hpp:244-255
template <class T>
BlockField<T> staircase_plan(const ScoreField<T>& S, const DualTrace<T>& tr, Index hu, Index hv) {
    const T lg = tr.gauge(hu) - tr.gauge(hv);
    BlockField<T> out;
    out.schedule = S.values.schedule;
    for (size_t t = 0; t < S.sched().tile_count(); ++t) out.blocks.push_back(plan_tile(S, t, tr.u(hu), tr.v(hv), lg));
    return out;
}

template <class T>
Mat<T> densify(const BlockField<T>& f) {
    const SupportMask& m = f.schedule->support();
    Mat<T> out(m.n_rows(), m.n_cols());
    for (size_t t = 0; t < f.schedule->tile_count(); ++t) {
        const TileRange& r = f.schedule->tiles()[t];
        for (Index i = 0; i < r.rows(); ++i)
            for (Index j = 0; j < r.cols(); ++j) out(r.row_begin + i, r.col_begin + j) = f.blocks[t](i, j);
    }
    return out;
}

// sinkhorn.hpp:262-277 -- O = P V, no row renormalization
template <class T>
Mat<T> apply_transport(const ScoreField<T>& S, const Vec<T>& u, const Vec<T>& v, const Mat<T>& V) {
    const TileSchedule& sched = S.sched();
    if (V.rows() != S.support().n_cols()) throw std::invalid_argument("V row count mismatch");
    Mat<T> O(S.support().n_rows(), V.cols());
    for (size_t t = 0; t < sched.tile_count(); ++t) {
        const TileRange& r = sched.tiles()[t];
        const Mat<T> p = plan_tile(S, t, u, v);
        for (Index i = 0; i < r.rows(); ++i) {
            T* o = O.row(r.row_begin + i);
            for (Index j = 0; j < r.cols(); ++j) {
                const T pij = p(i, j);
                if (pij == T(0)) continue;
                const T* vv = V.row(r.col_begin + j);
                for (Index x = 0; x < V.cols(); ++x) o[x] += pij * vv[x];
            }
        }
    }
    return O;
}

template <class T>
struct SurrogateRun {
    DualTrace<T> trace;
    ScoreField<T> raw, scaled;
    Mat<T> output;
};

// sinkhorn.hpp:288-302 -- forward entry point
template <class T>
SurrogateRun<T> run_surrogate(const Mat<T>& Q, const Mat<T>& K, const Mat<T>& V,
                              std::shared_ptr<const TileSchedule> schedule, Index base_depth, Index tail_depth,
                              const EpsSchedule<T>& eps, bool centered = true,
                              const ConstantEdges<T>* cst = nullptr) {
    SurrogateRun<T> run;
    run.raw = raw_scores(Q, K, schedule, cst);
    run.trace = stopped_base_solve(run.raw, base_depth, eps, centered);
    tail_refine(run.raw, run.trace, tail_depth, eps.final_epsilon());
    run.scaled = scale_to_temperature(run.raw, eps.final_epsilon());
    const Index h = run.trace.steps();
    run.output = apply_transport(run.scaled, run.trace.u(h), run.trace.v(h), V);
    return run;
}

// ---------------------------------------------------------------------------
// Adjoint -- include/sinktail/adjoint.hpp:9-373
// ---------------------------------------------------------------------------
template <class T>
struct CotangentSet {
    BlockField<T> score_bar;
    Mat<T> grad_q, grad_k, grad_v;
    std::vector<Vec<T>> u_bar, v_bar;
    Vec<T> base_u, base_v;  // BaseCotangent (adjoint.hpp:11-17)
    T d_eps = T(0);         // EXT: dL/d(epsilon), sec. A21 of SURVEY.md
    double base_l2() const {
        double s = 0;
        for (T x : base_u) s += double(x) * double(x);
        for (T x : base_v) s += double(x) * double(x);
        return std::sqrt(s);
    }
};

// adjoint.hpp:30-51
template <class T>
struct ModifierVectors {
    Vec<T> u_step_ratio, v_step_ratio, v_base_ratio;
    T gauge_21 = T(1), gauge_10 = T(1);
    static ModifierVectors from_trace(const DualTrace<T>& tr) {
        if (tr.tail_depth() != 2) throw UnsupportedDepth("modifier vectors need a depth-2 tail");
        ModifierVectors m;
        const auto& u1 = tr.tail_u(1);
        const auto& u2 = tr.tail_u(2);
        const auto& v0 = tr.tail_v(0);
        const auto& v1 = tr.tail_v(1);
        const auto& v2 = tr.tail_v(2);
        m.u_step_ratio.resize(u1.size());
        m.v_step_ratio.resize(v1.size());
        m.v_base_ratio.resize(v1.size());
        for (size_t i = 0; i < u1.size(); ++i) m.u_step_ratio[i] = std::exp(u1[i] - u2[i]);
        for (size_t j = 0; j < v1.size(); ++j) {
            m.v_step_ratio[j] = std::exp(v1[j] - v2[j]);
            m.v_base_ratio[j] = std::exp(v0[j] - v2[j]);
        }
        m.gauge_21 = std::exp(tr.tail_gauge(2) - tr.tail_gauge(1));
        m.gauge_10 = std::exp(tr.tail_gauge(1) - tr.tail_gauge(0));
        return m;
    }
};

enum class BackwardMode { OneReference, DirectFourPlan };

// adjoint.hpp:57-68 -- y += P^(hu,hv) x
template <class T>
void plan_apply(const ScoreField<T>& S, const DualTrace<T>& tr, Index hu, Index hv, const Vec<T>& x, Vec<T>& y) {
    const T lg = tr.gauge(hu) - tr.gauge(hv);
    const TileSchedule& sched = S.sched();
    for (size_t t = 0; t < sched.tile_count(); ++t) {
        const TileRange& r = sched.tiles()[t];
        const Mat<T> p = plan_tile(S, t, tr.u(hu), tr.v(hv), lg);
        for (Index i = 0; i < r.rows(); ++i) {
            T acc = 0;
            for (Index j = 0; j < r.cols(); ++j) acc += p(i, j) * x[static_cast<size_t>(r.col_begin + j)];
            y[static_cast<size_t>(r.row_begin + i)] += acc;
        }
    }
}
// adjoint.hpp:72-82 -- y += P^(hu,hv)^T x
template <class T>
void plan_apply_transpose(const ScoreField<T>& S, const DualTrace<T>& tr, Index hu, Index hv, const Vec<T>& x,
                          Vec<T>& y) {
    const T lg = tr.gauge(hu) - tr.gauge(hv);
    const TileSchedule& sched = S.sched();
    for (size_t t = 0; t < sched.tile_count(); ++t) {
        const TileRange& r = sched.tiles()[t];
        const Mat<T> p = plan_tile(S, t, tr.u(hu), tr.v(hv), lg);
        for (Index j = 0; j < r.cols(); ++j) {
            T acc = 0;
            for (Index i = 0; i < r.rows(); ++i) acc += p(i, j) * x[static_cast<size_t>(r.row_begin + i)];
            y[static_cast<size_t>(r.col_begin + j)] += acc;
        }
    }
}
// adjoint.hpp:87-106
template <class T>
void subtract_plan_outer(const ScoreField<T>& S, const DualTrace<T>& tr, Index hu, Index hv, const Vec<T>* row,
                         const Vec<T>* col, BlockField<T>& sbar, T weight = T(1)) {
    const T lg = tr.gauge(hu) - tr.gauge(hv);
    const TileSchedule& sched = S.sched();
    for (size_t t = 0; t < sched.tile_count(); ++t) {
        const TileRange& r = sched.tiles()[t];
        Mat<T> p = plan_tile(S, t, tr.u(hu), tr.v(hv), lg);
        Mat<T>& out = sbar.blocks[t];
        for (Index i = 0; i < r.rows(); ++i)
            for (Index j = 0; j < r.cols(); ++j) {
                const T pij = p(i, j) * weight;
                if (col) out(i, j) -= pij * (*col)[static_cast<size_t>(r.col_begin + j)];
                if (row) out(i, j) -= (*row)[static_cast<size_t>(r.row_begin + i)] * pij;
            }
    }
}

// adjoint.hpp:109-126 -- grad_Q = Sbar K /(sqrt(d) eps), grad_K = Sbar^T Q /(sqrt(d) eps).
// EXT: constant-score (dustbin) cells carry no Q/K dependence and are skipped.
template <class T>
void backprop_scores_to_qkv(const BlockField<T>& sbar, const Mat<T>& Q, const Mat<T>& K, T epsilon, Mat<T>& gq,
                            Mat<T>& gk, const ConstantEdges<T>* cst = nullptr) {
    const TileSchedule& sched = *sbar.schedule;
    const Index d = Q.cols();
    const T inv = T(1) / (std::sqrt(static_cast<T>(d)) * epsilon);
    gq = Mat<T>(Q.rows(), d);
    gk = Mat<T>(K.rows(), d);
    for (size_t t = 0; t < sched.tile_count(); ++t) {
        const TileRange& r = sched.tiles()[t];
        const Mat<T>& blk = sbar.blocks[t];
        for (Index i = 0; i < r.rows(); ++i)
            for (Index j = 0; j < r.cols(); ++j) {
                const T s = blk(i, j);
                if (s == T(0)) continue;
                if (cst && cst->hit(r.row_begin + i, r.col_begin + j)) continue;
                const T* k = K.row(r.col_begin + j);
                const T* q = Q.row(r.row_begin + i);
                T* dq = gq.row(r.row_begin + i);
                T* dk = gk.row(r.col_begin + j);
                for (Index x = 0; x < d; ++x) {
                    dq[x] += inv * (s * k[x]);
                    dk[x] += inv * (s * q[x]);
                }
            }
    }
}

// EXT: dL/d(eps) = -(1/eps) sum_ij Sbar_ij S_ij over the
// tail-temperature score field (S = raw/eps on every edge, dustbin included).
template <class T>
T d_epsilon_from_score_bar(const BlockField<T>& sbar, const ScoreField<T>& S) {
    T acc = 0;
    for (size_t t = 0; t < sbar.blocks.size(); ++t)
        for (size_t k = 0; k < sbar.blocks[t].a.size(); ++k) acc += sbar.blocks[t].a[k] * S.values.blocks[t].a[k];
    return -acc / S.epsilon;
}

// adjoint.hpp:132-200 -- exact reverse pass of the tail surrogate for any R
template <class T>
CotangentSet<T> tail_adjoint_generic(const ScoreField<T>& S, const DualTrace<T>& tr, const Mat<T>& G,
                                     const Mat<T>& Q, const Mat<T>& K, const Mat<T>& V,
                                     const ConstantEdges<T>* cst = nullptr) {
    const TileSchedule& sched = S.sched();
    const SupportMask& m = sched.support();
    const Index R = tr.tail_depth();
    const Index hR = tr.steps();
    const Index d = V.cols();
    const size_t nr = static_cast<size_t>(m.n_rows()), nc = static_cast<size_t>(m.n_cols());
    CotangentSet<T> out;
    out.score_bar = BlockField<T>(S.values.schedule);
    out.grad_v = Mat<T>(V.rows(), d);
    out.u_bar.assign(static_cast<size_t>(R) + 1, Vec<T>(nr, T(0)));
    out.v_bar.assign(static_cast<size_t>(R) + 1, Vec<T>(nc, T(0)));
    Vec<T> g_u(nr, T(0)), g_v(nc, T(0));
    for (size_t t = 0; t < sched.tile_count(); ++t) {
        const TileRange& r = sched.tiles()[t];
        const Mat<T> p = plan_tile(S, t, tr.u(hR), tr.v(hR));
        for (Index i = 0; i < r.rows(); ++i)
            for (Index j = 0; j < r.cols(); ++j) {
                const T* gi = G.row(r.row_begin + i);
                const T* vj = V.row(r.col_begin + j);
                T z = 0;
                for (Index x = 0; x < d; ++x) z += gi[x] * vj[x];
                const T w = p(i, j) * z;
                out.score_bar.blocks[t](i, j) += w;
                g_u[static_cast<size_t>(r.row_begin + i)] += w;
                g_v[static_cast<size_t>(r.col_begin + j)] += w;
                T* dv = out.grad_v.row(r.col_begin + j);
                for (Index x = 0; x < d; ++x) dv[x] += p(i, j) * gi[x];
            }
    }
    if (R == 0) {
        out.u_bar[0] = g_u;
        out.v_bar[0] = g_v;
        out.base_u = g_u;
        out.base_v = g_v;
        backprop_scores_to_qkv(out.score_bar, Q, K, S.epsilon, out.grad_q, out.grad_k, cst);
        out.d_eps = d_epsilon_from_score_bar(out.score_bar, S);
        return out;
    }
    out.v_bar[static_cast<size_t>(R)] = g_v;
    Vec<T> pv(nr, T(0));
    plan_apply(S, tr, hR, hR, out.v_bar[static_cast<size_t>(R)], pv);
    for (size_t i = 0; i < nr; ++i) out.u_bar[static_cast<size_t>(R)][i] = g_u[i] - pv[i];
    for (Index t = R; t >= 1; --t) {
        const Index h = tr.tail_step(t);
        const Vec<T>& ub = out.u_bar[static_cast<size_t>(t)];
        const Vec<T>& vb = out.v_bar[static_cast<size_t>(t)];
        subtract_plan_outer<T>(S, tr, h, h, nullptr, &vb, out.score_bar);
        subtract_plan_outer<T>(S, tr, h, h - 1, &ub, nullptr, out.score_bar);
        Vec<T> vprev(nc, T(0));
        plan_apply_transpose(S, tr, h, h - 1, ub, vprev);
        for (size_t j = 0; j < nc; ++j) out.v_bar[static_cast<size_t>(t) - 1][j] = -vprev[j];
        if (t >= 2) {
            Vec<T> un(nr, T(0));
            plan_apply(S, tr, h - 1, h - 1, out.v_bar[static_cast<size_t>(t) - 1], un);
            for (size_t i = 0; i < nr; ++i) out.u_bar[static_cast<size_t>(t) - 1][i] = -un[i];
        }
    }
    out.u_bar[0] = Vec<T>(nr, T(0));
    out.base_u = out.u_bar[0];
    out.base_v = out.v_bar[0];
    backprop_scores_to_qkv(out.score_bar, Q, K, S.epsilon, out.grad_q, out.grad_k, cst);
    out.d_eps = d_epsilon_from_score_bar(out.score_bar, S);
    return out;
}

// certificates.hpp:25-70 -- pull a base-state cotangent (u-bar, v-bar at step T) back through the
// stopped base solve to (Q, K): the tail recurrences extended over h = T..1, each step's plans at its
// stage temperature, the raw-score cotangent weighted by 1/eps_h.
template <class T>
struct BaseVjpResult {
    Mat<T> grad_q, grad_k;
};

template <class T>
BaseVjpResult<T> base_solve_vjp(const ScoreField<T>& raw, const DualTrace<T>& tr, const Vec<T>& eta_u,
                                const Vec<T>& eta_v, const Mat<T>& Q, const Mat<T>& K) {
    if (!raw.raw) throw std::invalid_argument("base_solve_vjp expects raw (unscaled) scores");
    if (static_cast<Index>(tr.u_hist.size()) <= tr.split) throw MissingBaseTrace("trace does not retain all base duals");
    const SupportMask& m = raw.support();
    const size_t nr = static_cast<size_t>(m.n_rows()), nc = static_cast<size_t>(m.n_cols());
    if (eta_u.size() != nr || eta_v.size() != nc)
        throw std::invalid_argument("base-state cotangent sized to the wrong support");
    BaseVjpResult<T> out;
    out.grad_q = Mat<T>(Q.rows(), Q.cols());
    out.grad_k = Mat<T>(K.rows(), K.cols());
    if (tr.split == 0) return out;  // the cold start does not depend on the parameters
    BlockField<T> raw_bar(raw.values.schedule);
    Vec<T> ub = eta_u, vb = eta_v;
    int stage = tr.stage_at(tr.split);
    ScoreField<T> S = scale_to_temperature(raw, tr.eps_at(tr.split));
    for (Index h = tr.split; h >= 1; --h) {
        if (tr.stage_at(h) != stage) {
            stage = tr.stage_at(h);
            S = scale_to_temperature(raw, tr.eps_at(h));
        }
        const T inv_eps = T(1) / tr.eps_at(h);
        Vec<T> pv(nr, T(0));
        plan_apply(S, tr, h, h, vb, pv);
        Vec<T> ab(nr);
        for (size_t i = 0; i < nr; ++i) ab[i] = ub[i] - pv[i];
        subtract_plan_outer<T>(S, tr, h, h, nullptr, &vb, raw_bar, inv_eps);
        Vec<T> vprev(nc, T(0));
        plan_apply_transpose(S, tr, h, h - 1, ab, vprev);
        subtract_plan_outer<T>(S, tr, h, h - 1, &ab, nullptr, raw_bar, inv_eps);
        for (size_t j = 0; j < nc; ++j) vb[j] = -vprev[j];
        std::fill(ub.begin(), ub.end(), T(0));
    }
    backprop_scores_to_qkv(raw_bar, Q, K, T(1), out.grad_q, out.grad_k);
    return out;
}

// adjoint.hpp:202-226 -- one-reference-tile score cotangent
//   Sbar_ij = P22_ij (Z_ij - v2b_j - g21 b_j u2b_i - a_i b_j v1b_j - g10 a_i d_j u1b_i)
template <class T>
Mat<T> r2_score_cotangent_tile(const Mat<T>& p22, const Mat<T>& z, const T* u2b, const T* v2b, const T* u1b,
                               const T* v1b, const T* a, const T* b, const T* dl, T g21, T g10) {
    Mat<T> out(p22.rows(), p22.cols());
    for (Index i = 0; i < p22.rows(); ++i) {
        const T ai = a[i], u2 = u2b[i], au1 = g10 * ai * u1b[i];
        for (Index j = 0; j < p22.cols(); ++j) {
            const T mod = z(i, j) - v2b[j] - g21 * b[j] * u2 - ai * b[j] * v1b[j] - au1 * dl[j];
            out(i, j) = p22(i, j) * mod;
        }
    }
    return out;
}

namespace detail {
// Z tile = G_I V_J^T (adjoint.hpp:263-264)
template <class T>
Mat<T> z_tile(const Mat<T>& G, const Mat<T>& V, const TileRange& r) {
    const Index d = V.cols();
    Mat<T> z(r.rows(), r.cols());
    for (Index i = 0; i < r.rows(); ++i) {
        const T* gi = G.row(r.row_begin + i);
        for (Index j = 0; j < r.cols(); ++j) {
            const T* vj = V.row(r.col_begin + j);
            T acc = 0;
            for (Index x = 0; x < d; ++x) acc += gi[x] * vj[x];
            z(i, j) = acc;
        }
    }
    return z;
}
// dQ += inv Sbar K, dK += inv Sbar^T Q (adjoint.hpp:305-308), constant edges skipped (EXT)
template <class T>
void accumulate_qk(const Mat<T>& sb, const TileRange& r, const Mat<T>& Q, const Mat<T>& K, T inv, Mat<T>& gq,
                   Mat<T>& gk, const ConstantEdges<T>* cst) {
    const Index d = Q.cols();
    for (Index i = 0; i < r.rows(); ++i)
        for (Index j = 0; j < r.cols(); ++j) {
            const T s = sb(i, j);
            if (s == T(0)) continue;
            if (cst && cst->hit(r.row_begin + i, r.col_begin + j)) continue;
            const T* k = K.row(r.col_begin + j);
            const T* q = Q.row(r.row_begin + i);
            T* dq = gq.row(r.row_begin + i);
            T* dk = gk.row(r.col_begin + j);
            for (Index x = 0; x < d; ++x) {
                dq[x] += inv * (s * k[x]);
                dk[x] += inv * (s * q[x]);
            }
        }
}
// terminal sweep: W = P22 .* Z, g_u, g_v, dV += P22^T G (adjoint.hpp:258-270)
template <class T>
void terminal_sweep(const ScoreField<T>& S, const DualTrace<T>& tr, Index h2, const Mat<T>& G, const Mat<T>& V,
                    Vec<T>& g_u, Vec<T>& g_v, Mat<T>& gv) {
    const TileSchedule& sched = S.sched();
    const Index d = V.cols();
    for (size_t t = 0; t < sched.tile_count(); ++t) {
        const TileRange& r = sched.tiles()[t];
        const Mat<T> p = plan_tile(S, t, tr.u(h2), tr.v(h2));
        const Mat<T> z = z_tile(G, V, r);
        for (Index i = 0; i < r.rows(); ++i)
            for (Index j = 0; j < r.cols(); ++j) {
                const T w = p(i, j) * z(i, j);
                g_u[static_cast<size_t>(r.row_begin + i)] += w;
                g_v[static_cast<size_t>(r.col_begin + j)] += w;
            }
        for (Index j = 0; j < r.cols(); ++j) {
            T* dv = gv.row(r.col_begin + j);
            for (Index i = 0; i < r.rows(); ++i) {
                const T pij = p(i, j);
                if (pij == T(0)) continue;
                const T* gi = G.row(r.row_begin + i);
                for (Index x = 0; x < d; ++x) dv[x] += pij * gi[x];
            }
        }
    }
}
}  // namespace detail

// adjoint.hpp:232-373 -- full R=2 backward, both schedules
template <class T>
CotangentSet<T> r2_backward(const ScoreField<T>& S, const DualTrace<T>& tr, const Mat<T>& G, const Mat<T>& Q,
                            const Mat<T>& K, const Mat<T>& V, BackwardMode mode = BackwardMode::OneReference,
                            const ConstantEdges<T>* cst = nullptr) {
    if (tr.tail_depth() != 2) throw UnsupportedDepth("r2_backward requires a tail of depth 2");
    const TileSchedule& sched = S.sched();
    const SupportMask& m = sched.support();
    const Index h0 = tr.tail_step(0), h1 = tr.tail_step(1), h2 = tr.tail_step(2);
    const T inv_qk = T(1) / (std::sqrt(static_cast<T>(Q.cols())) * S.epsilon);
    const size_t nr = static_cast<size_t>(m.n_rows()), nc = static_cast<size_t>(m.n_cols());
    CotangentSet<T> out;
    out.score_bar = BlockField<T>(S.values.schedule);
    out.grad_q = Mat<T>(Q.rows(), Q.cols());
    out.grad_k = Mat<T>(K.rows(), K.cols());
    out.grad_v = Mat<T>(V.rows(), V.cols());
    out.u_bar.assign(3, Vec<T>(nr, T(0)));
    out.v_bar.assign(3, Vec<T>(nc, T(0)));

    Vec<T> g_u(nr, T(0)), g_v(nc, T(0));
    detail::terminal_sweep(S, tr, h2, G, V, g_u, g_v, out.grad_v);
    out.v_bar[2] = g_v;
    Vec<T> pv(nr, T(0));
    plan_apply(S, tr, h2, h2, out.v_bar[2], pv);
    for (size_t i = 0; i < nr; ++i) out.u_bar[2][i] = g_u[i] - pv[i];

    if (mode == BackwardMode::OneReference) {
        const ModifierVectors<T> mv = ModifierVectors<T>::from_trace(tr);
        // adjoint.hpp:279-291 -- recurrences as reference-plan products with modifiers
        Vec<T> tmp_v(nc, T(0));
        plan_apply_transpose(S, tr, h2, h2, out.u_bar[2], tmp_v);
        for (size_t j = 0; j < nc; ++j) out.v_bar[1][j] = -mv.gauge_21 * mv.v_step_ratio[j] * tmp_v[j];
        Vec<T> tmp_u(nr, T(0)), bv1(nc);
        for (size_t j = 0; j < nc; ++j) bv1[j] = mv.v_step_ratio[j] * out.v_bar[1][j];
        plan_apply(S, tr, h2, h2, bv1, tmp_u);
        for (size_t i = 0; i < nr; ++i) out.u_bar[1][i] = -mv.u_step_ratio[i] * tmp_u[i];
        std::fill(tmp_v.begin(), tmp_v.end(), T(0));
        Vec<T> au1(nr);
        for (size_t i = 0; i < nr; ++i) au1[i] = mv.u_step_ratio[i] * out.u_bar[1][i];
        plan_apply_transpose(S, tr, h2, h2, au1, tmp_v);
        for (size_t j = 0; j < nc; ++j) out.v_bar[0][j] = -mv.gauge_10 * mv.v_base_ratio[j] * tmp_v[j];
        // adjoint.hpp:293-310 -- score cotangent from one reference tile per block
        for (size_t t = 0; t < sched.tile_count(); ++t) {
            const TileRange& r = sched.tiles()[t];
            const Mat<T> p22 = plan_tile(S, t, tr.u(h2), tr.v(h2));
            const Mat<T> z = detail::z_tile(G, V, r);
            const size_t rb = static_cast<size_t>(r.row_begin), cb = static_cast<size_t>(r.col_begin);
            Mat<T> sb = r2_score_cotangent_tile<T>(p22, z, out.u_bar[2].data() + rb, out.v_bar[2].data() + cb,
                                                   out.u_bar[1].data() + rb, out.v_bar[1].data() + cb,
                                                   mv.u_step_ratio.data() + rb, mv.v_step_ratio.data() + cb,
                                                   mv.v_base_ratio.data() + cb, mv.gauge_21, mv.gauge_10);
            detail::accumulate_qk(sb, r, Q, K, inv_qk, out.grad_q, out.grad_k, cst);
            out.score_bar.blocks[t] = std::move(sb);
        }
    } else {
        // adjoint.hpp:333-368 -- direct route through the mixed staircase plans
        Vec<T> tmp_v(nc, T(0));
        plan_apply_transpose(S, tr, h2, h1, out.u_bar[2], tmp_v);
        for (size_t j = 0; j < nc; ++j) out.v_bar[1][j] = -tmp_v[j];
        Vec<T> tmp_u(nr, T(0));
        plan_apply(S, tr, h1, h1, out.v_bar[1], tmp_u);
        for (size_t i = 0; i < nr; ++i) out.u_bar[1][i] = -tmp_u[i];
        std::fill(tmp_v.begin(), tmp_v.end(), T(0));
        plan_apply_transpose(S, tr, h1, h0, out.u_bar[1], tmp_v);
        for (size_t j = 0; j < nc; ++j) out.v_bar[0][j] = -tmp_v[j];
        for (size_t t = 0; t < sched.tile_count(); ++t) {
            const TileRange& r = sched.tiles()[t];
            const Index rb = r.row_begin, cb = r.col_begin;
            const Mat<T> p22 = plan_tile(S, t, tr.u(h2), tr.v(h2));
            const Mat<T> p21 = plan_tile(S, t, tr.u(h2), tr.v(h1), tr.gauge(h2) - tr.gauge(h1));
            const Mat<T> p11 = plan_tile(S, t, tr.u(h1), tr.v(h1));
            const Mat<T> p10 = plan_tile(S, t, tr.u(h1), tr.v(h0), tr.gauge(h1) - tr.gauge(h0));
            const Mat<T> z = detail::z_tile(G, V, r);
            Mat<T> sb(r.rows(), r.cols());
            for (Index i = 0; i < r.rows(); ++i)
                for (Index j = 0; j < r.cols(); ++j) {
                    T s = p22(i, j) * z(i, j);
                    s -= p22(i, j) * out.v_bar[2][static_cast<size_t>(cb + j)];
                    s -= out.u_bar[2][static_cast<size_t>(rb + i)] * p21(i, j);
                    s -= p11(i, j) * out.v_bar[1][static_cast<size_t>(cb + j)];
                    s -= out.u_bar[1][static_cast<size_t>(rb + i)] * p10(i, j);
                    sb(i, j) = s;
                }
            detail::accumulate_qk(sb, r, Q, K, inv_qk, out.grad_q, out.grad_k, cst);
            out.score_bar.blocks[t] = std::move(sb);
        }
    }
    out.u_bar[0] = Vec<T>(nr, T(0));
    out.base_u = out.u_bar[0];
    out.base_v = out.v_bar[0];
    out.d_eps = d_epsilon_from_score_bar(out.score_bar, S);
    return out;
}

// ---------------------------------------------------------------------------
// Losses -- include/sinktail/loss.hpp:10-113
// ---------------------------------------------------------------------------
enum class LossKind { FrobeniusToTarget, Linear, SupervisedValueMse };

template <class T>
struct LossSpec {
    LossKind kind = LossKind::Linear;
    Mat<T> fixed;
    std::vector<Index> target_cols;
    static LossSpec linear(Mat<T> g) { LossSpec l; l.kind = LossKind::Linear; l.fixed = std::move(g); return l; }
    static LossSpec frobenius_to_target(Mat<T> t) {
        LossSpec l; l.kind = LossKind::FrobeniusToTarget; l.fixed = std::move(t); return l;
    }
    static LossSpec supervised_value_mse(std::vector<Index> c) {
        LossSpec l; l.kind = LossKind::SupervisedValueMse; l.target_cols = std::move(c); return l;
    }
    Index active_rows(const std::vector<bool>& rv) const {
        Index n = 0;
        for (bool b : rv) n += b ? 1 : 0;
        return n;
    }
    // loss.hpp:50-72
    T value(const Mat<T>& O, const Mat<T>& V, const std::vector<bool>& rv) const {
        T acc = 0;
        const Index d = O.cols();
        switch (kind) {
            case LossKind::Linear:
                for (Index i = 0; i < O.rows(); ++i)
                    if (rv[static_cast<size_t>(i)]) for (Index x = 0; x < d; ++x) acc += fixed(i, x) * O(i, x);
                return acc;
            case LossKind::FrobeniusToTarget:
                for (Index i = 0; i < O.rows(); ++i)
                    if (rv[static_cast<size_t>(i)])
                        for (Index x = 0; x < d; ++x) { const T e = O(i, x) - fixed(i, x); acc += e * e; }
                return T(0.5) * acc;
            case LossKind::SupervisedValueMse: {
                const Index n = active_rows(rv);
                for (Index i = 0; i < O.rows(); ++i) {
                    if (!rv[static_cast<size_t>(i)]) continue;
                    const Index c = target_cols.at(static_cast<size_t>(i));
                    for (Index x = 0; x < d; ++x) { const T e = O(i, x) - V(c, x); acc += e * e; }
                }
                return acc / static_cast<T>(n);
            }
        }
        return acc;
    }
    // loss.hpp:74-98
    Mat<T> output_cotangent(const Mat<T>& O, const Mat<T>& V, const std::vector<bool>& rv) const {
        Mat<T> G(O.rows(), O.cols());
        const Index d = O.cols();
        for (Index i = 0; i < O.rows(); ++i) {
            if (!rv[static_cast<size_t>(i)]) continue;
            for (Index x = 0; x < d; ++x) {
                switch (kind) {
                    case LossKind::Linear: G(i, x) = fixed(i, x); break;
                    case LossKind::FrobeniusToTarget: G(i, x) = O(i, x) - fixed(i, x); break;
                    case LossKind::SupervisedValueMse:
                        G(i, x) = T(2) / static_cast<T>(active_rows(rv)) *
                                  (O(i, x) - V(target_cols.at(static_cast<size_t>(i)), x));
                        break;
                }
            }
        }
        return G;
    }
    // loss.hpp:101-113
    Mat<T> direct_value_cotangent(const Mat<T>& O, const Mat<T>& V, const std::vector<bool>& rv) const {
        Mat<T> D(V.rows(), V.cols());
        if (kind != LossKind::SupervisedValueMse) return D;
        const T w = T(2) / static_cast<T>(active_rows(rv));
        for (Index i = 0; i < O.rows(); ++i) {
            if (!rv[static_cast<size_t>(i)]) continue;
            const Index c = target_cols.at(static_cast<size_t>(i));
            for (Index x = 0; x < V.cols(); ++x) D(c, x) -= w * (O(i, x) - V(c, x));
        }
        return D;
    }
};

// ---------------------------------------------------------------------------
// Instances -- include/sinktail/problem.hpp:19-88
// ---------------------------------------------------------------------------
struct InstanceSpec {
    Index n_rows = 64, n_cols = 64, head_dim = 8, half_band = 16, base_depth = 15, tail_depth = 2;
    double epsilon = 1.0;
    std::vector<std::pair<double, Index>> stages;
    std::uint64_t seed = 0;
    Index dustbin_block = 0;
    Index tile_block = 64;
};

template <class T>
struct Instance {
    InstanceSpec spec;
    Mat<T> Q, K, V;
    std::shared_ptr<const TileSchedule> schedule;
    EpsSchedule<T> eps;
};

template <class T>
EpsSchedule<T> make_eps_schedule(const InstanceSpec& spec) {
    if (spec.stages.empty()) return EpsSchedule<T>::single(static_cast<T>(spec.epsilon), spec.base_depth);
    EpsSchedule<T> s;
    for (const auto& st : spec.stages) s.stages.push_back({static_cast<T>(st.first), st.second});
    return s;
}

// problem.hpp:56-88
template <class T>
Instance<T> make_instance(const InstanceSpec& spec) {
    Instance<T> inst;
    inst.spec = spec;
    inst.Q = normal_matrix<T>(spec.seed, "Q", spec.n_rows, spec.head_dim);
    inst.K = normal_matrix<T>(spec.seed, "K", spec.n_cols, spec.head_dim);
    inst.V = normal_matrix<T>(spec.seed, "V", spec.n_cols, spec.head_dim);
    SupportMask mask = build_band_support(spec.n_rows, spec.n_cols, spec.half_band);
    if (spec.dustbin_block > 0) {
        AugmentedSupport aug = augment_dustbin(mask, spec.dustbin_block);
        auto append = [&](const Mat<T>& base, const char* tag) {
            Mat<T> out(base.rows() + spec.dustbin_block, spec.head_dim);
            std::copy(base.a.begin(), base.a.end(), out.a.begin());
            Mat<T> row = normal_matrix<T>(spec.seed, tag, 1, spec.head_dim);
            std::copy(row.a.begin(), row.a.end(), out.a.begin() + base.a.size());
            return out;
        };
        inst.Q = append(inst.Q, "dustbin_q");
        inst.K = append(inst.K, "dustbin_k");
        inst.V = append(inst.V, "dustbin_v");
        inst.schedule = TileSchedule::build(aug.mask, spec.tile_block);
    } else {
        inst.schedule = TileSchedule::build(mask, spec.tile_block);
    }
    inst.eps = make_eps_schedule<T>(spec);
    return inst;
}

// test_util.hpp:54-61 -- linear loss with G drawn from tag "G", inactive rows zeroed
inline LossSpec<double> random_linear_loss(const Instance<double>& inst, double scale = 1.0) {
    const SupportMask& m = inst.schedule->support();
    Mat<double> g = normal_matrix<double>(inst.spec.seed, "G", m.n_rows(), inst.spec.head_dim, scale);
    for (Index i = 0; i < m.n_rows(); ++i)
        if (!m.row_active(i)) for (Index x = 0; x < g.cols(); ++x) g(i, x) = 0;
    return LossSpec<double>::linear(std::move(g));
}

// ---------------------------------------------------------------------------
// Dense f64 oracle -- include/sinktail/oracle.hpp:14-333
// ---------------------------------------------------------------------------
namespace dense {

inline constexpr Index kDenseCap = 512;
inline constexpr Index kBpttCap = 256;

struct DenseProblem {
    Mat<double> Q, K, V;
    BoolMat support;
    double epsilon = 1.0;
    Index base_depth = 0, tail_depth = 0;
    EpsSchedule<double> schedule;
    LossSpec<double> loss;
    const ConstantEdges<double>* cst = nullptr;  // EXT: constant-score dustbin edges
    Index rows() const { return support.rows(); }
    Index cols() const { return support.cols(); }
    std::vector<bool> row_valid() const {
        std::vector<bool> r(static_cast<size_t>(rows()), false);
        for (Index i = 0; i < rows(); ++i)
            for (Index j = 0; j < cols(); ++j) if (support(i, j)) { r[static_cast<size_t>(i)] = true; break; }
        return r;
    }
    EpsSchedule<double> resolved_schedule() const {
        if (schedule.stages.empty()) return EpsSchedule<double>::single(epsilon, base_depth);
        return schedule;
    }
    void check_cap(Index cap) const {
        if (rows() > cap || cols() > cap)
            throw SizeCapExceeded("dense oracle cap exceeded: " + std::to_string(rows()) + "x" +
                                  std::to_string(cols()) + " > " + std::to_string(cap));
    }
};

struct DenseTrace {
    std::vector<Vec<double>> u_hist, v_hist;
    std::vector<double> gauge_hist, eps_hist;
    Index split = 0;
    Index steps() const { return static_cast<Index>(u_hist.size()) - 1; }
};

struct DenseForward {
    Mat<double> raw_scores;
    DenseTrace trace;
    Mat<double> output;
    double loss_value = 0.0;
};

// oracle.hpp:73-76
inline Mat<double> dense_raw_scores(const DenseProblem& p) {
    const Index d = p.Q.cols();
    Mat<double> s(p.rows(), p.cols());
    const double inv = 1.0 / std::sqrt(static_cast<double>(d));
    for (Index i = 0; i < p.rows(); ++i)
        for (Index j = 0; j < p.cols(); ++j) {
            if (!p.support(i, j)) continue;
            if (p.cst && p.cst->hit(i, j)) { s(i, j) = p.cst->value; continue; }
            double acc = 0;
            for (Index x = 0; x < d; ++x) acc += p.Q(i, x) * p.K(j, x);
            s(i, j) = acc * inv;
        }
    return s;
}
inline Mat<double> scale(const Mat<double>& m, double eps) {
    Mat<double> o = m;
    for (auto& x : o.a) x /= eps;
    return o;
}
// oracle.hpp:78-96
inline Vec<double> dense_row_half_step(const Mat<double>& S, const BoolMat& sp, const Vec<double>& v) {
    Vec<double> u(static_cast<size_t>(S.rows()), 0.0);
    for (Index i = 0; i < S.rows(); ++i) {
        double mx = -std::numeric_limits<double>::infinity();
        for (Index j = 0; j < S.cols(); ++j) if (sp(i, j)) mx = std::max(mx, S(i, j) + v[static_cast<size_t>(j)]);
        if (!std::isfinite(mx)) continue;
        double acc = 0;
        for (Index j = 0; j < S.cols(); ++j) if (sp(i, j)) acc += std::exp(S(i, j) + v[static_cast<size_t>(j)] - mx);
        u[static_cast<size_t>(i)] = -(mx + std::log(acc));
    }
    return u;
}
// oracle.hpp:98-115
inline Vec<double> dense_col_half_step(const Mat<double>& S, const BoolMat& sp, const Vec<double>& u) {
    Vec<double> v(static_cast<size_t>(S.cols()), 0.0);
    for (Index j = 0; j < S.cols(); ++j) {
        double mx = -std::numeric_limits<double>::infinity();
        for (Index i = 0; i < S.rows(); ++i) if (sp(i, j)) mx = std::max(mx, S(i, j) + u[static_cast<size_t>(i)]);
        if (!std::isfinite(mx)) continue;
        double acc = 0;
        for (Index i = 0; i < S.rows(); ++i) if (sp(i, j)) acc += std::exp(S(i, j) + u[static_cast<size_t>(i)] - mx);
        v[static_cast<size_t>(j)] = -(mx + std::log(acc));
    }
    return v;
}
// oracle.hpp:117-126
inline Mat<double> dense_plan(const Mat<double>& S, const BoolMat& sp, const Vec<double>& u, const Vec<double>& v,
                              double lg = 0.0) {
    Mat<double> p(S.rows(), S.cols());
    for (Index i = 0; i < S.rows(); ++i)
        for (Index j = 0; j < S.cols(); ++j)
            if (sp(i, j)) p(i, j) = std::exp(S(i, j) + u[static_cast<size_t>(i)] + v[static_cast<size_t>(j)] + lg);
    return p;
}
inline Mat<double> matmul(const Mat<double>& A, const Mat<double>& B) {
    Mat<double> C(A.rows(), B.cols());
    for (Index i = 0; i < A.rows(); ++i)
        for (Index k = 0; k < A.cols(); ++k) {
            const double a = A(i, k);
            if (a == 0.0) continue;
            for (Index j = 0; j < B.cols(); ++j) C(i, j) += a * B(k, j);
        }
    return C;
}
inline Mat<double> transpose(const Mat<double>& A) {
    Mat<double> t(A.cols(), A.rows());
    for (Index i = 0; i < A.rows(); ++i) for (Index j = 0; j < A.cols(); ++j) t(j, i) = A(i, j);
    return t;
}

struct FrozenBase { Vec<double> u, v; double gauge = 0.0; };

// oracle.hpp:134-193
inline DenseForward dense_forward_impl(const DenseProblem& p, const std::optional<FrozenBase>& frozen) {
    p.check_cap(kDenseCap);
    const auto rv = p.row_valid();
    DenseForward fwd;
    fwd.raw_scores = dense_raw_scores(p);
    const EpsSchedule<double> sched = p.resolved_schedule();
    sched.validate(p.base_depth);
    DenseTrace& tr = fwd.trace;
    tr.u_hist.push_back(Vec<double>(static_cast<size_t>(p.rows()), 0.0));
    tr.v_hist.push_back(Vec<double>(static_cast<size_t>(p.cols()), 0.0));
    tr.gauge_hist.push_back(0.0);
    tr.eps_hist.push_back(0.0);
    auto advance = [&](const Mat<double>& S, double eps) {
        Vec<double> a = dense_row_half_step(S, p.support, tr.v_hist.back());
        Vec<double> b = dense_col_half_step(S, p.support, a);
        double sum = 0;
        Index cnt = 0;
        for (Index i = 0; i < p.rows(); ++i) if (rv[static_cast<size_t>(i)]) { sum += a[static_cast<size_t>(i)]; ++cnt; }
        const double c = sum / static_cast<double>(cnt);
        for (Index i = 0; i < p.rows(); ++i) if (rv[static_cast<size_t>(i)]) a[static_cast<size_t>(i)] -= c;
        for (auto& x : b) x += c;
        tr.u_hist.push_back(std::move(a));
        tr.v_hist.push_back(std::move(b));
        tr.gauge_hist.push_back(tr.gauge_hist.back() + c);
        tr.eps_hist.push_back(eps);
    };
    if (frozen.has_value()) {
        tr.u_hist = {frozen->u};
        tr.v_hist = {frozen->v};
        tr.gauge_hist = {frozen->gauge};
        tr.split = 0;
    } else {
        for (const auto& st : sched.stages) {
            const Mat<double> S = scale(fwd.raw_scores, st.epsilon);
            for (Index k = 0; k < st.iterations; ++k) advance(S, st.epsilon);
        }
        tr.split = tr.steps();
    }
    const double ef = sched.final_epsilon();
    const Mat<double> Sf = scale(fwd.raw_scores, ef);
    for (Index r = 0; r < p.tail_depth; ++r) advance(Sf, ef);
    const Index h = tr.steps();
    const Mat<double> plan = dense_plan(Sf, p.support, tr.u_hist[static_cast<size_t>(h)], tr.v_hist[static_cast<size_t>(h)]);
    fwd.output = matmul(plan, p.V);
    fwd.loss_value = p.loss.value(fwd.output, p.V, rv);
    return fwd;
}
inline DenseForward dense_forward(const DenseProblem& p) { return dense_forward_impl(p, std::nullopt); }

struct DenseGradients {
    Mat<double> grad_q, grad_k, grad_v;
    Vec<double> eta_u, eta_v;
    double d_eps = 0.0;  // EXT (single-stage schedules only)
};

// oracle.hpp:206-262 -- analytic reverse pass with explicit centering pullbacks
inline DenseGradients dense_reverse(const DenseProblem& p, const DenseForward& fwd, bool through_base) {
    const auto rv = p.row_valid();
    const Index n_valid = static_cast<Index>(std::count(rv.begin(), rv.end(), true));
    const DenseTrace& tr = fwd.trace;
    const Index H = tr.steps();
    const Index stop = through_base ? 0 : tr.split;
    const double ef = p.resolved_schedule().final_epsilon();
    const Index nr = p.rows(), nc = p.cols();
    DenseGradients g;
    Mat<double> rsb(nr, nc);  // raw_score_bar
    const Mat<double> Sf = scale(fwd.raw_scores, ef);
    const Mat<double> plan = dense_plan(Sf, p.support, tr.u_hist[static_cast<size_t>(H)], tr.v_hist[static_cast<size_t>(H)]);
    const Mat<double> G = p.loss.output_cotangent(fwd.output, p.V, rv);
    const Mat<double> Z = matmul(G, transpose(p.V));
    Mat<double> W(nr, nc);
    for (size_t k = 0; k < W.a.size(); ++k) W.a[k] = plan.a[k] * Z.a[k];
    for (size_t k = 0; k < W.a.size(); ++k) rsb.a[k] += W.a[k] / ef;
    g.grad_v = matmul(transpose(plan), G);
    {
        const Mat<double> D = p.loss.direct_value_cotangent(fwd.output, p.V, rv);
        for (size_t k = 0; k < D.a.size(); ++k) g.grad_v.a[k] += D.a[k];
    }
    Vec<double> ub(static_cast<size_t>(nr), 0.0), vb(static_cast<size_t>(nc), 0.0);
    for (Index i = 0; i < nr; ++i) for (Index j = 0; j < nc; ++j) { ub[static_cast<size_t>(i)] += W(i, j); vb[static_cast<size_t>(j)] += W(i, j); }
    for (Index h = H; h > stop; --h) {
        const double eh = tr.eps_hist[static_cast<size_t>(h)];
        const Mat<double> Sh = scale(fwd.raw_scores, eh);
        double sv = 0, su = 0;
        for (double x : vb) sv += x;
        for (double x : ub) su += x;
        const double delta = sv - su;
        for (Index i = 0; i < nr; ++i) if (rv[static_cast<size_t>(i)]) ub[static_cast<size_t>(i)] += delta / static_cast<double>(n_valid);
        const Mat<double> ps = dense_plan(Sh, p.support, tr.u_hist[static_cast<size_t>(h)], tr.v_hist[static_cast<size_t>(h)]);
        for (Index i = 0; i < nr; ++i) {
            double acc = 0;
            for (Index j = 0; j < nc; ++j) acc += ps(i, j) * vb[static_cast<size_t>(j)];
            ub[static_cast<size_t>(i)] -= acc;
        }
        for (Index i = 0; i < nr; ++i) for (Index j = 0; j < nc; ++j) rsb(i, j) -= ps(i, j) * vb[static_cast<size_t>(j)] / eh;
        const double lg = tr.gauge_hist[static_cast<size_t>(h)] - tr.gauge_hist[static_cast<size_t>(h - 1)];
        const Mat<double> pm = dense_plan(Sh, p.support, tr.u_hist[static_cast<size_t>(h)], tr.v_hist[static_cast<size_t>(h - 1)], lg);
        Vec<double> vprev(static_cast<size_t>(nc), 0.0);
        for (Index j = 0; j < nc; ++j) {
            double acc = 0;
            for (Index i = 0; i < nr; ++i) acc += pm(i, j) * ub[static_cast<size_t>(i)];
            vprev[static_cast<size_t>(j)] = -acc;
        }
        for (Index i = 0; i < nr; ++i) for (Index j = 0; j < nc; ++j) rsb(i, j) -= pm(i, j) * ub[static_cast<size_t>(i)] / eh;
        vb = std::move(vprev);
        ub.assign(static_cast<size_t>(nr), 0.0);
    }
    g.eta_u = ub;
    g.eta_v = vb;
    const double inv = 1.0 / std::sqrt(static_cast<double>(p.Q.cols()));
    // EXT: d(eps) on the surrogate (single-stage): S = raw/eps everywhere in the tail
    if (!through_base) {
        double acc = 0;
        for (Index i = 0; i < nr; ++i) for (Index j = 0; j < nc; ++j) acc += rsb(i, j) * fwd.raw_scores(i, j);
        g.d_eps = -acc / ef;
    }
    Mat<double> rq = rsb;
    if (p.cst)
        for (Index i = 0; i < nr; ++i) for (Index j = 0; j < nc; ++j) if (p.cst->hit(i, j)) rq(i, j) = 0.0;
    g.grad_q = matmul(rq, p.K);
    g.grad_k = matmul(transpose(rq), p.Q);
    for (auto& x : g.grad_q.a) x *= inv;
    for (auto& x : g.grad_k.a) x *= inv;
    return g;
}

inline DenseGradients full_bptt_grad(const DenseProblem& p) {
    p.check_cap(kBpttCap);
    return dense_reverse(p, dense_forward(p), true);
}
inline DenseGradients dense_surrogate_grad(const DenseProblem& p) { return dense_reverse(p, dense_forward(p), false); }

enum class FdVariant { Surrogate, Full };
enum class FdTensor { Q, K, V, Eps };

struct FdOptions {
    double step = 1e-5;
    FdVariant variant = FdVariant::Surrogate;
    std::vector<std::pair<Index, Index>> entries;
};

// oracle.hpp:290-333 -- central differences with stop-gradient semantics.
// EXT: FdTensor::Eps perturbs the tail temperature with the base frozen.
inline Mat<double> finite_diff_grad(const DenseProblem& p, FdTensor wrt, const FdOptions& opt) {
    p.check_cap(kDenseCap);
    if (!(opt.step > 0)) throw std::invalid_argument("finite-difference step must be > 0");
    if (opt.step < 1e-9) throw std::invalid_argument("finite-difference step too small for double precision");
    std::optional<FrozenBase> frozen;
    if (opt.variant == FdVariant::Surrogate) {
        DenseProblem base_only = p;
        base_only.tail_depth = 0;
        const DenseForward base = dense_forward(base_only);
        frozen = FrozenBase{base.trace.u_hist.back(), base.trace.v_hist.back(), base.trace.gauge_hist.back()};
    }
    DenseProblem work = p;
    if (wrt == FdTensor::Eps) {
        Mat<double> g(1, 1, 0.0);
        // perturb the tail temperature = the schedule's final stage (base frozen)
        const double x = p.resolved_schedule().final_epsilon(), h = opt.step * (1.0 + std::abs(x));
        auto set_eps = [&](double e) {
            work.epsilon = e;
            if (!work.schedule.stages.empty()) work.schedule.stages.back().epsilon = e;
        };
        set_eps(x + h);
        const double lp = dense_forward_impl(work, frozen).loss_value;
        set_eps(x - h);
        const double lm = dense_forward_impl(work, frozen).loss_value;
        g(0, 0) = (lp - lm) / (2.0 * h);
        return g;
    }
    const Mat<double>* src = wrt == FdTensor::Q ? &p.Q : (wrt == FdTensor::K ? &p.K : &p.V);
    Mat<double> grad(src->rows(), src->cols(), std::numeric_limits<double>::quiet_NaN());
    std::vector<std::pair<Index, Index>> entries = opt.entries;
    if (entries.empty())
        for (Index i = 0; i < src->rows(); ++i) for (Index j = 0; j < src->cols(); ++j) entries.emplace_back(i, j);
    Mat<double>* dst = wrt == FdTensor::Q ? &work.Q : (wrt == FdTensor::K ? &work.K : &work.V);
    for (const auto& e : entries) {
        const double x = (*src)(e.first, e.second), h = opt.step * (1.0 + std::abs(x));
        (*dst)(e.first, e.second) = x + h;
        const double lp = dense_forward_impl(work, frozen).loss_value;
        (*dst)(e.first, e.second) = x - h;
        const double lm = dense_forward_impl(work, frozen).loss_value;
        (*dst)(e.first, e.second) = x;
        grad(e.first, e.second) = (lp - lm) / (2.0 * h);
    }
    return grad;
}

inline double max_abs_diff_on(const Mat<double>& fd, const Mat<double>& an) {
    double mx = 0;
    for (size_t k = 0; k < fd.a.size(); ++k) {
        if (std::isnan(fd.a[k])) continue;
        mx = std::max(mx, std::abs(fd.a[k] - an.a[k]));
    }
    return mx;
}

inline BoolMat dense_support_of(const SupportMask& m) {
    BoolMat b(m.n_rows(), m.n_cols(), 0);
    for (Index i = 0; i < m.n_rows(); ++i) m.for_each_in_row(i, [&](Index j) { b(i, j) = 1; });
    return b;
}

inline DenseProblem make_dense_problem(const Instance<double>& inst, LossSpec<double> loss) {
    DenseProblem p;
    p.Q = inst.Q;
    p.K = inst.K;
    p.V = inst.V;
    p.support = dense_support_of(inst.schedule->support());
    p.epsilon = inst.spec.epsilon;
    p.base_depth = inst.spec.base_depth;
    p.tail_depth = inst.spec.tail_depth;
    p.schedule = make_eps_schedule<double>(inst.spec);
    p.loss = std::move(loss);
    return p;
}

}  // namespace dense

// certificates.hpp:72-150 -- the omitted-gradient certificate of a tail depth: eta_R from the generic
// tail adjoint, pulled back through the base solve (c_R); with the dense oracle in reach, the exact
// remainder identity (full BPTT - stopped) = c_R is checked
struct BiasCertificate {
    Index tail_depth = 0;
    double eta_norm = 0.0, c_inf = 0.0, c_l2 = 0.0;
    Mat<double> c_q, c_k;
    double max_gap = std::numeric_limits<double>::quiet_NaN();
    double residual = std::numeric_limits<double>::quiet_NaN();
    bool residual_computed = false;
};

struct CertificateProblem {
    Mat<double> Q, K, V;
    std::shared_ptr<const TileSchedule> schedule;
    Index base_depth = 0;
    EpsSchedule<double> eps;
    LossSpec<double> loss;
};

inline dense::DenseProblem to_dense_problem(const CertificateProblem& p, Index tail_depth) {
    dense::DenseProblem d;
    d.Q = p.Q;
    d.K = p.K;
    d.V = p.V;
    d.support = dense::dense_support_of(p.schedule->support());
    d.epsilon = p.eps.final_epsilon();
    d.base_depth = p.base_depth;
    d.tail_depth = tail_depth;
    d.schedule = p.eps;
    d.loss = p.loss;
    return d;
}

inline BiasCertificate bias_certificate(const CertificateProblem& p, Index tail_depth, bool want_residual = true) {
    SurrogateRun<double> run = run_surrogate<double>(p.Q, p.K, p.V, p.schedule, p.base_depth, tail_depth, p.eps);
    const auto rv = p.schedule->support().row_mask();
    const Mat<double> G = p.loss.output_cotangent(run.output, p.V, rv);
    const CotangentSet<double> adj = tail_adjoint_generic(run.scaled, run.trace, G, p.Q, p.K, p.V);
    const BaseVjpResult<double> c = base_solve_vjp(run.raw, run.trace, adj.base_u, adj.base_v, p.Q, p.K);
    BiasCertificate cert;
    cert.tail_depth = tail_depth;
    cert.eta_norm = adj.base_l2();
    cert.c_q = c.grad_q;
    cert.c_k = c.grad_k;
    double l2 = 0.0;
    for (double x : c.grad_q.a) { cert.c_inf = std::max(cert.c_inf, std::abs(x)); l2 += x * x; }
    for (double x : c.grad_k.a) { cert.c_inf = std::max(cert.c_inf, std::abs(x)); l2 += x * x; }
    cert.c_l2 = std::sqrt(l2);
    const SupportMask& m = p.schedule->support();
    if (want_residual && m.n_rows() <= dense::kBpttCap && m.n_cols() <= dense::kBpttCap) {
        const dense::DenseGradients full = dense::full_bptt_grad(to_dense_problem(p, tail_depth));
        double gap = 0.0, res = 0.0;
        for (size_t k = 0; k < full.grad_q.a.size(); ++k) {
            const double g = full.grad_q.a[k] - adj.grad_q.a[k];
            gap = std::max(gap, std::abs(g));
            res = std::max(res, std::abs(g - c.grad_q.a[k]));
        }
        for (size_t k = 0; k < full.grad_k.a.size(); ++k) {
            const double g = full.grad_k.a[k] - adj.grad_k.a[k];
            gap = std::max(gap, std::abs(g));
            res = std::max(res, std::abs(g - c.grad_k.a[k]));
        }
        cert.max_gap = gap;
        cert.residual = res;
        cert.residual_computed = true;
    }
    return cert;
}

// certificates.hpp:152-179 -- smallest R <= r_max whose certified omitted gradient is <= tau
// (cost nondecreasing, so the first feasible depth is the min-cost one); with an operator-norm
// bound the sufficient test bound * ||eta_R|| <= tau replaces c_inf
struct TailDepthSelection {
    Index selected = -1;
    bool used_sufficient_bound = false;
    std::vector<BiasCertificate> trail;
};

inline TailDepthSelection select_tail_depth(const CertificateProblem& p, double tau, Index r_max,
                                            const std::function<double(Index)>& cost =
                                                [](Index r) { return static_cast<double>(r); },
                                            const double* operator_norm_bound = nullptr) {
    if (!(tau > 0)) throw std::invalid_argument("tolerance must be > 0");
    if (r_max < 0) throw std::invalid_argument("R_max must be >= 0");
    double prev = -std::numeric_limits<double>::infinity();
    for (Index r = 0; r <= r_max; ++r) {
        const double c = cost(r);
        if (c < prev) throw std::invalid_argument("cost function must be nondecreasing");
        prev = c;
    }
    TailDepthSelection sel;
    sel.used_sufficient_bound = operator_norm_bound != nullptr;
    for (Index r = 0; r <= r_max; ++r) {
        BiasCertificate cert = bias_certificate(p, r, false);
        const bool ok = operator_norm_bound ? (*operator_norm_bound * cert.eta_norm <= tau) : (cert.c_inf <= tau);
        sel.trail.push_back(std::move(cert));
        if (ok) {
            sel.selected = r;
            break;
        }
    }
    return sel;
}

}  // namespace stoc
