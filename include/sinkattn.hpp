// sinkattn.hpp -- the include-swap C++ drop-in for the reference's hot path.
//
// The reference's two calls (proj/include/sinktail):
//   SurrogateRun<S> run_surrogate(Q, K, V, schedule, T, R, EpsSchedule, centered)   sinkhorn.hpp:288-302
//   CotangentSet<S> r2_backward(run.scaled, run.trace, G, Q, K, V, BackwardMode)      adjoint.hpp:232-236
// take host row-major matrices (Matrix<S> = Eigen::Matrix<S, Dynamic, Dynamic, RowMajor>,
// types.hpp:10-21) and return results by value.  This header keeps those names, argument order
// and exception types over the C-ABI of libsinkattn.so (include/sinkattn.h).  `Mat` is any
// row-major float matrix with rows(), cols(), data() and a (rows, cols) constructor -- the
// reference's Matrix<float> included.
//
// Differences, by design:
//  * the support is described by (half_band, optional row / column masks) -- the arguments of
//    build_band_support (src/support.cpp:111-117) -- instead of a TileSchedule (results are
//    tile-size invariant, test_sinkhorn.cpp:490-506);
//  * a `Context` owns the device buffers and the stream and is reused across calls, so no
//    allocation happens once it is sized (pass device-resident data through the C-ABI directly
//    to also skip the host copies);
//  * SurrogateRun carries the O(L) saved tail state (device) instead of the trace and score
//    fields; r2_backward takes the run.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "sinkattn.h"

namespace sinkattn {

// inc/errors.hpp:10-39 -- same names, std::runtime_error bases
struct InfeasibleSupport : std::runtime_error { using std::runtime_error::runtime_error; };
struct InvalidTemperature : std::runtime_error { using std::runtime_error::runtime_error; };
struct UnsupportedDepth : std::runtime_error { using std::runtime_error::runtime_error; };
struct MissingBaseTrace : std::runtime_error { using std::runtime_error::runtime_error; };
struct SizeCapExceeded : std::runtime_error { using std::runtime_error::runtime_error; };
struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };

inline void check(st_status s) {
    const std::string m = st_last_error();
    switch (s) {
        case ST_OK: return;
        case ST_INFEASIBLE_SUPPORT: throw InfeasibleSupport(m);
        case ST_INVALID_TEMPERATURE: throw InvalidTemperature(m);
        case ST_UNSUPPORTED_DEPTH: throw UnsupportedDepth(m);
        case ST_MISSING_BASE_TRACE: throw MissingBaseTrace(m);
        case ST_SIZE_CAP_EXCEEDED: throw SizeCapExceeded(m);
        case ST_CUDA_ERROR: throw CudaError(m);
        default: throw std::invalid_argument(m);
    }
}
inline void cuda_check(cudaError_t e) {
    if (e != cudaSuccess) throw CudaError(cudaGetErrorString(e));
}

enum class BackwardMode { OneReference, DirectFourPlan };  // adjoint.hpp:54

// Device buffers and stream reused across calls (grown on demand, never shrunk).
class Context {
   public:
    explicit Context(cudaStream_t s = nullptr) : stream(s) {}
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    ~Context() {
        for (auto& b : bufs_) cudaFree(b.p);
    }
    void* buffer(size_t slot, size_t bytes) {
        if (bufs_.size() <= slot) bufs_.resize(slot + 1);
        Buf& b = bufs_[slot];
        if (b.n < bytes) {
            if (b.p) cuda_check(cudaFree(b.p));
            b.p = nullptr;
            cuda_check(cudaMalloc(&b.p, bytes));
            b.n = bytes;
        }
        return b.p;
    }
    cudaStream_t stream;

   private:
    struct Buf {
        void* p = nullptr;
        size_t n = 0;
    };
    std::vector<Buf> bufs_;
};

enum Slot : size_t { kQ, kK, kV, kG, kO, kSaved, kWs, kRowMask, kColMask, kDQ, kDK, kDV, kDeps };

template <class Mat>
struct SurrogateRun {          // sinkhorn.hpp:279-286, minus the trace / score fields
    Mat output;                // O = P^(T+R) V
    st_desc desc{};
    void* saved = nullptr;     // device: tail duals + status (owned by the Context)
    void* workspace = nullptr;
    size_t workspace_bytes = 0;
    const uint8_t* row_mask = nullptr;  // device copies (nullptr: all active)
    const uint8_t* col_mask = nullptr;
    Context* ctx = nullptr;
};

template <class Mat>
struct CotangentSet {          // adjoint.hpp:19-28 (grads) plus d_eps (EXT)
    Mat grad_q, grad_k, grad_v;
    float d_eps = 0.f;
};

namespace detail {
template <class Mat>
const float* upload(Context& c, size_t slot, const Mat& m) {
    const size_t n = sizeof(float) * (size_t)m.rows() * (size_t)m.cols();
    void* d = c.buffer(slot, n);
    cuda_check(cudaMemcpyAsync(d, m.data(), n, cudaMemcpyHostToDevice, c.stream));
    return static_cast<const float*>(d);
}
inline const uint8_t* upload_mask(Context& c, size_t slot, const std::vector<bool>* mask) {
    if (mask == nullptr || mask->empty()) return nullptr;
    std::vector<uint8_t> h(mask->begin(), mask->end());
    void* d = c.buffer(slot, h.size());
    cuda_check(cudaMemcpyAsync(d, h.data(), h.size(), cudaMemcpyHostToDevice, c.stream));
    cuda_check(cudaStreamSynchronize(c.stream));  // h is a temporary
    return static_cast<const uint8_t*>(d);
}
template <class Mat>
Mat download(Context& c, const void* d, int64_t rows, int64_t cols) {
    Mat m(rows, cols);
    cuda_check(cudaMemcpyAsync(m.data(), d, sizeof(float) * rows * cols, cudaMemcpyDeviceToHost, c.stream));
    return m;
}
}  // namespace detail

// run_surrogate (sinkhorn.hpp:288-302) over build_band_support(L_q, L_k, half_band, masks):
// stopped T-step base solve from the cold start, R-step tail, O = P^(T+R) V; fp32.
template <class Mat>
SurrogateRun<Mat> run_surrogate(const Mat& Q, const Mat& K, const Mat& V, int64_t half_band, int64_t base_depth,
                                int64_t tail_depth, double epsilon, Context& ctx,
                                const std::vector<bool>* row_mask = nullptr,
                                const std::vector<bool>* col_mask = nullptr, bool centered = true) {
    if (Q.cols() != K.cols() || K.rows() != V.rows()) throw std::invalid_argument("Q / K / V shapes differ");
    SurrogateRun<Mat> r;
    r.ctx = &ctx;
    r.desc = st_desc{};
    r.desc.batch = 1;
    r.desc.heads = 1;
    r.desc.seq_q = Q.rows();
    r.desc.seq_k = K.rows();
    r.desc.head_dim = Q.cols();
    r.desc.half_band = half_band;
    r.desc.base_depth = base_depth;
    r.desc.tail_depth = tail_depth;
    r.desc.epsilon = epsilon;
    r.desc.dtype = ST_F32;
    r.desc.dustbin_cost = 1.0;
    r.desc.centered = centered ? 1 : 0;
    const uint8_t* rm = detail::upload_mask(ctx, kRowMask, row_mask);
    const uint8_t* cm = detail::upload_mask(ctx, kColMask, col_mask);
    if (rm || cm) {  // SupportMask::validate (src/support.cpp:91-109) on the host, like build_band_support
        std::vector<uint8_t> hr, hc;
        if (row_mask) hr.assign(row_mask->begin(), row_mask->end());
        if (col_mask) hc.assign(col_mask->begin(), col_mask->end());
        check(st_validate_support(&r.desc, hr.empty() ? nullptr : hr.data(), hc.empty() ? nullptr : hc.data()));
    }
    r.row_mask = rm;
    r.col_mask = cm;
    const float* dQ = detail::upload(ctx, kQ, Q);
    const float* dK = detail::upload(ctx, kK, K);
    const float* dV = detail::upload(ctx, kV, V);
    r.saved = ctx.buffer(kSaved, st_saved_bytes(&r.desc));
    r.workspace_bytes = st_workspace_bytes(&r.desc);
    r.workspace = ctx.buffer(kWs, r.workspace_bytes);
    float* O = static_cast<float*>(ctx.buffer(kO, sizeof(float) * Q.rows() * V.cols()));
    check(st_forward(&r.desc, dQ, dK, dV, rm, cm, O, r.saved, r.workspace, r.workspace_bytes, ctx.stream));
    r.output = detail::download<Mat>(ctx, O, Q.rows(), V.cols());
    check(st_check_status(&r.desc, r.saved, ctx.stream));  // synchronizes; the reference throws here
    return r;
}

// r2_backward (adjoint.hpp:232-373) for the run's forward and the output cotangent G (linear loss).
template <class Mat>
CotangentSet<Mat> r2_backward(const SurrogateRun<Mat>& run, const Mat& G, const Mat& Q, const Mat& K, const Mat& V,
                              BackwardMode mode = BackwardMode::OneReference) {
    Context& ctx = *run.ctx;
    if (run.desc.tail_depth != 2) throw UnsupportedDepth("r2_backward requires a tail of depth 2");
    const float* dQ = detail::upload(ctx, kQ, Q);
    const float* dK = detail::upload(ctx, kK, K);
    const float* dV = detail::upload(ctx, kV, V);
    const float* dG = detail::upload(ctx, kG, G);
    const size_t nq = sizeof(float) * Q.rows() * Q.cols(), nk = sizeof(float) * K.rows() * K.cols();
    float* gq = static_cast<float*>(ctx.buffer(kDQ, nq));
    float* gk = static_cast<float*>(ctx.buffer(kDK, nk));
    float* gv = static_cast<float*>(ctx.buffer(kDV, sizeof(float) * V.rows() * V.cols()));
    float* de = static_cast<float*>(ctx.buffer(kDeps, sizeof(float)));
    check(st_backward(&run.desc, run.saved, dQ, dK, dV, dG, run.row_mask, run.col_mask, gq, gk, gv, de, nullptr,
                      mode == BackwardMode::OneReference ? ST_ONE_REFERENCE : ST_DIRECT_FOUR_PLAN, run.workspace,
                      run.workspace_bytes, ctx.stream));
    CotangentSet<Mat> c;
    c.grad_q = detail::download<Mat>(ctx, gq, Q.rows(), Q.cols());
    c.grad_k = detail::download<Mat>(ctx, gk, K.rows(), K.cols());
    c.grad_v = detail::download<Mat>(ctx, gv, V.rows(), V.cols());
    cuda_check(cudaMemcpyAsync(&c.d_eps, de, sizeof(float), cudaMemcpyDeviceToHost, ctx.stream));
    cuda_check(cudaStreamSynchronize(ctx.stream));
    return c;
}

}  // namespace sinkattn
