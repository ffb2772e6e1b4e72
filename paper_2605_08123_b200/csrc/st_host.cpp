// st_host.cpp -- host-side pieces of the C-ABI: the counter RNG used to build
// seeded inputs (make_instance's generator, rng.hpp:14-56, bit-exact) and the
// host support validation (SupportMask::validate, src/support.cpp:91-109).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>
#include <thread>
#include <vector>

#include "../../include/sinkattn.h"

namespace {

inline uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
inline uint64_t fold_tag(uint64_t seed, const char* tag) {
    uint64_t h = splitmix64(seed ^ 0x5bf03635d78d672dULL);
    for (const char* c = tag; *c; ++c) h = splitmix64(h ^ (uint64_t)(unsigned char)*c);
    return h;
}
inline double uniform(uint64_t key) {
    double u = (double)(splitmix64(key) >> 11) * 0x1.0p-53;
    return u <= 0.0 ? 0x1.0p-53 : u;
}
inline double normal(uint64_t base, uint64_t n) {
    const double u1 = uniform(base + 2 * n), u2 = uniform(base + 2 * n + 1);
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
}

template <class F>
void parallel_chunks(int64_t n, F&& f) {
    const int64_t kMin = 1 << 16;
    int nt = (int)std::min<int64_t>(std::max(1u, std::thread::hardware_concurrency()), (n + kMin - 1) / kMin);
    if (nt <= 1) {
        f(0, n);
        return;
    }
    std::vector<std::thread> th;
    const int64_t per = (n + nt - 1) / nt;
    for (int t = 0; t < nt; ++t) {
        const int64_t lo = t * per, hi = std::min(n, lo + per);
        if (lo < hi) th.emplace_back([&, lo, hi] { f(lo, hi); });
    }
    for (auto& x : th) x.join();
}

thread_local std::string g_host_err;

}  // namespace

extern "C" {

void st_normal_fill(uint64_t seed, const char* tag, uint64_t start, int64_t n, double scale, double* out) {
    const uint64_t base = fold_tag(seed, tag);
    parallel_chunks(n, [&](int64_t lo, int64_t hi) {
        for (int64_t k = lo; k < hi; ++k) out[k] = scale * normal(base, start + (uint64_t)k);
    });
}

void st_uniform_fill(uint64_t seed, const char* tag, uint64_t start, int64_t n, double* out) {
    const uint64_t base = fold_tag(seed, tag);
    parallel_chunks(n, [&](int64_t lo, int64_t hi) {
        for (int64_t k = lo; k < hi; ++k) out[k] = uniform(base + start + (uint64_t)k);
    });
}

// SupportMask::validate on the (optionally spoke-augmented) band support of
// every example.  O(B * L * W) worst case, with a prefix-count shortcut.
st_status st_validate_support(const st_desc* d, const uint8_t* rm, const uint8_t* cm) {
    if (d == nullptr || d->batch < 1 || d->seq_q < 1 || d->seq_k < 1 || d->half_band < 0)
        return ST_INVALID_ARGUMENT;
    const int64_t Lq = d->seq_q, Lk = d->seq_k, w = d->half_band;
    std::vector<int64_t> pre_c(Lk + 1), pre_r(Lq + 1);
    for (int64_t b = 0; b < d->batch; ++b) {
        const uint8_t* r = rm ? rm + b * Lq : nullptr;
        const uint8_t* c = cm ? cm + b * Lk : nullptr;
        pre_c[0] = 0;
        for (int64_t j = 0; j < Lk; ++j) pre_c[j + 1] = pre_c[j] + ((c == nullptr || c[j]) ? 1 : 0);
        pre_r[0] = 0;
        for (int64_t i = 0; i < Lq; ++i) pre_r[i + 1] = pre_r[i] + ((r == nullptr || r[i]) ? 1 : 0);
        if (d->dustbin) continue;  // every active row/col reaches the always-active dustbin
        for (int64_t i = 0; i < Lq; ++i) {
            if (r && !r[i]) continue;
            const int64_t lo = std::max<int64_t>(0, i - w), hi = std::min<int64_t>(Lk - 1, i + w);
            if (lo > hi || pre_c[hi + 1] - pre_c[lo] == 0) return ST_INFEASIBLE_SUPPORT;
        }
        for (int64_t j = 0; j < Lk; ++j) {
            if (c && !c[j]) continue;
            const int64_t lo = std::max<int64_t>(0, j - w), hi = std::min<int64_t>(Lq - 1, j + w);
            if (lo > hi || pre_r[hi + 1] - pre_r[lo] == 0) return ST_INFEASIBLE_SUPPORT;
        }
    }
    return ST_OK;
}

}  // extern "C"
