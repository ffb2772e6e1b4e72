/*
 * sinkattn.h -- C-ABI of the B200-native banded balanced entropic-OT
 * ("Sinkhorn") attention operator: stopped T-step log-domain base solve,
 * depth-2 differentiable tail, exact R=2 adjoint in the one-reference-tile
 * form, single-active-dustbin (spoke) variant.
 *
 * Plain C: pointers, sizes and status codes only (no torch / no C++ types).
 * Every entry point is stream-ordered on `stream` (a cudaStream_t passed as
 * void*), never allocates, never synchronizes, and never falls back to the
 * CPU.  Device buffers are owned by the caller.
 *
 * Reference interface each entry point replaces (paths under
 * /root/reference/proj/include/sinktail/):
 *   st_forward   <- run_surrogate<Scalar>(Q, K, V, schedule, T, R, EpsSchedule, centered)
 *                   sinkhorn.hpp:288-302 (support built by build_band_support
 *                   src/support.cpp:111-117 / augment_dustbin src/support.cpp:119-148)
 *   st_backward  <- r2_backward<Scalar>(S, trace, G, Q, K, V, BackwardMode)
 *                   adjoint.hpp:232-373 (OneReference :255-310, DirectFourPlan :311-368)
 *   st_status    <- the exception types of errors.hpp:10-39
 *   st_validate_support <- SupportMask::validate, src/support.cpp:91-109
 *   st_normal_fill      <- normal_matrix / counter_normal, rng.hpp:38-56
 *
 * Tensor layout: [B, H, L', d] contiguous row-major; each (b, h) slice is the
 * reference's row-major Matrix (types.hpp:10-11).  L' = L + 1 when
 * dustbin = 1: row L holds the dustbin token (its Q/K rows are unused under
 * the constant dustbin cost; its V row is the dustbin value).
 * Masks: uint8 [B, L] (1 = active) shared by all heads of an example, or NULL
 * for all-active.  The dustbin row/column is always active.
 */
#ifndef SINKATTN_H_
#define SINKATTN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum st_status {
    ST_OK = 0,
    ST_INVALID_ARGUMENT = 1,     /* std::invalid_argument (shapes, masks) */
    ST_INFEASIBLE_SUPPORT = 2,   /* InfeasibleSupport: active row/col without an active edge */
    ST_INVALID_TEMPERATURE = 3,  /* InvalidTemperature: epsilon <= 0 */
    ST_UNSUPPORTED_DEPTH = 4,    /* UnsupportedDepth: r2 path with tail_depth != 2 */
    ST_MISSING_BASE_TRACE = 5,   /* MissingBaseTrace: backward without a forward's saved state */
    ST_SIZE_CAP_EXCEEDED = 6,    /* SizeCapExceeded */
    ST_CUDA_ERROR = 7,           /* a CUDA runtime error (message in st_last_error) */
    ST_WORKSPACE_TOO_SMALL = 8,
    ST_NOT_SUPPORTED = 9         /* shape outside what the sm_100a kernels implement */
} st_status;

typedef enum st_dtype { ST_F32 = 0, ST_BF16 = 1 } st_dtype;

typedef enum st_backward_mode {
    ST_ONE_REFERENCE = 0,    /* BackwardMode::OneReference (adjoint.hpp:255-310) */
    ST_DIRECT_FOUR_PLAN = 1, /* BackwardMode::DirectFourPlan (adjoint.hpp:311-368), ablation */
    ST_GENERIC_TAIL = 2      /* tail_adjoint_generic (adjoint.hpp:132-200): any tail depth R <= 8,
                                materialised score cotangent; no dustbin, d in {32, 64, 128} */
} st_backward_mode;

typedef struct st_desc {
    int64_t batch;        /* B */
    int64_t heads;        /* H */
    int64_t seq_q;        /* L_q (rows, queries), without the dustbin token */
    int64_t seq_k;        /* L_k (cols, keys), without the dustbin token */
    int64_t head_dim;     /* d */
    int64_t half_band;    /* reference W: (i, j) active iff |i - j| <= half_band (support.hpp:20-23) */
    int64_t base_depth;   /* T: stopped base steps from the cold start u = v = 0 */
    int64_t tail_depth;   /* R: differentiable tail steps (r2_backward modes require 2) */
    double epsilon;       /* entropic temperature, > 0 */
    int32_t dtype;        /* st_dtype of Q, K, V, dO (outputs and gradients are always f32) */
    int32_t dustbin;      /* 0, or 1 = one active dustbin token per side on the spoke support */
    double dustbin_cost;  /* constant cost on every dustbin edge (score = -cost / epsilon) */
    int32_t centered;     /* 1 = reference default: report the centered gauge ledger in saved */
    int32_t flags;        /* 0 = auto; ST_FLAG_GENERIC forces the generic (non-tensor-core) kernels,
                             ST_FLAG_REUSE_BAND (backward) reuses the forward's score band */
    /* epsilon-continuation schedule of the base solve (EpsSchedule, trace.hpp:12-50): stage q runs
     * stage_iters[q] full steps at temperature stage_eps[q]; temperatures non-increasing, iterations
     * summing to base_depth, the last stage at `epsilon` (the tail temperature, as
     * EpsSchedule::final_epsilon).  n_stages = 0: one stage of base_depth steps at `epsilon`.
     * Host pointers, read during the call only; at most ST_MAX_STAGES stages. */
    int32_t n_stages;
    const double* stage_eps;
    const int64_t* stage_iters;
} st_desc;

#define ST_MAX_STAGES 8

#define ST_FLAG_GENERIC 1
/* st_backward only: reuse the score band the most recent st_forward left in the
 * same workspace (the reference's r2_backward consumes run.scaled the same way,
 * adjoint.hpp:232).  Honoured only when that forward had the same desc, Q and K
 * pointers (host-side registry); the caller must not have written the workspace
 * or Q/K in between.  Otherwise the band is recomputed. */
#define ST_FLAG_REUSE_BAND 2
/* bf16 problems whose band lines up with 64-column chunks (no dustbin, seq_q == seq_k, half_band a
 * multiple of 64, head_dim 64 or 128 -- BASELINE configs 4 and 5) run band-free by default: the
 * transport output and the R=2 backward recompute their score / cotangent tiles on the tensor cores
 * and st_workspace_bytes() is O(L): no L x W band and (with a driver that provides
 * tensor maps) no packed O(L d) operand plane either.  ST_FLAG_STORED_BAND selects the
 * stored-band kernels (and their O(L W) workspace) instead; mode ST_GENERIC_TAIL and the *_halo
 * entry points need it on such problems and return ST_NOT_SUPPORTED without it. */
#define ST_FLAG_STORED_BAND 4

/* Device bytes of the opaque saved state written by st_forward and read by
 * st_backward: fp32 tail duals u, v at steps T, T+1, T+2 plus the per-head
 * gauge ledger.  O(L) per head -- never the L x W plan. */
size_t st_saved_bytes(const st_desc* desc);

/* Device scratch bytes needed by st_forward / st_backward. */
size_t st_workspace_bytes(const st_desc* desc);

/* Forward = run_surrogate: scores, T base steps, R tail steps, O = P^(T+R,T+R) V.
 * Q, K, V: [B, H, L', d] in desc->dtype.  O: [B, H, L', d] f32.
 * saved: st_saved_bytes(desc) bytes (may be NULL when no backward follows). */
st_status st_forward(const st_desc* desc, const void* Q, const void* K, const void* V,
                     const uint8_t* row_mask, const uint8_t* col_mask, float* O, void* saved,
                     void* workspace, size_t workspace_bytes, void* stream);

/* Backward = r2_backward (modes ST_ONE_REFERENCE / ST_DIRECT_FOUR_PLAN, tail_depth 2) or
 * tail_adjoint_generic (mode ST_GENERIC_TAIL, any tail_depth <= 8): dQ, dK, dV (f32, [B, H, L', d]), d_eps ([B*H] f32,
 * dL/d(epsilon) per head, may be NULL) and eta_v (the base cotangent v-bar^(0),
 * [B, H, L'_k] f32, may be NULL).  dO is the output cotangent G in desc->dtype. */
st_status st_backward(const st_desc* desc, const void* saved, const void* Q, const void* K,
                      const void* V, const void* dO, const uint8_t* row_mask,
                      const uint8_t* col_mask, float* dQ, float* dK, float* dV, float* d_eps,
                      float* eta_v, int32_t mode, void* workspace, size_t workspace_bytes,
                      void* stream);

/* tail_adjoint_generic (adjoint.hpp:132-200) with its full base cotangent: as st_backward in mode
 * ST_GENERIC_TAIL, plus eta_u ([B*H, L'_q] f32, may be NULL) = u-bar^(0), which is nonzero only for
 * tail_depth 0 (then eta = (g_u, g_v), the row / column sums of P^(T,T) (.) dO V^T). */
st_status st_tail_adjoint(const st_desc* desc, const void* saved, const void* Q, const void* K,
                          const void* V, const void* dO, const uint8_t* row_mask, const uint8_t* col_mask,
                          float* dQ, float* dK, float* dV, float* d_eps, float* eta_u, float* eta_v,
                          void* workspace, size_t workspace_bytes, void* stream);

/* base_solve_vjp (certificates.hpp:25-70): pull a base-state cotangent (eta_u [B*H, L'_q] or NULL
 * = 0, eta_v [B*H, L'_k]: the v-bar^(0) that st_backward returns) back through the T stopped base
 * steps to dQ, dK ([B, H, L', d] f32) -- the omitted-gradient certificate c_R of the tail depth
 * (bias_certificate, certificates.hpp:112-140).  Recomputes the base solve keeping every step's
 * duals (T+1 dual pairs in the workspace), then runs the reverse recurrences at each step's stage
 * temperature.  No dustbin; d in {32, 64, 128}.  base_depth = 0 gives zeros. */
size_t st_base_vjp_workspace_bytes(const st_desc* desc);
st_status st_base_solve_vjp(const st_desc* desc, const void* Q, const void* K, const uint8_t* row_mask,
                            const uint8_t* col_mask, const float* eta_u, const float* eta_v, float* dQ,
                            float* dK, void* workspace, size_t workspace_bytes, void* stream);

/* Sequence sharding (config 5): the problem a rank passes is its own rows plus a halo of up to
 * half_band rows on each side.  The library calls `hook` right after it has ENQUEUED (on `stream`)
 * each kernel that produces a vector the next kernel reads across the shard edge -- kind 0: a row
 * vector u / u-bar ([B*H][L'_q] f32), kind 1: a column vector v / v-bar ([B*H][L'_k]).  The hook
 * must enqueue, on `stream`, the replacement of the vector's halo entries by the neighbours' values
 * (e.g. NCCL point-to-point of the w boundary entries); every own row's and own column's reduction
 * lies inside the local window, so the result for the own rows equals the unsharded one.  Outputs
 * of halo rows are unspecified; d_eps sums the rows [own_begin, own_end) only.  Dustbin problems
 * are not supported on this path. */
typedef void (*st_halo_fn)(void* user, int32_t kind, float* vec, int64_t len, void* stream);

st_status st_forward_halo(const st_desc* desc, const void* Q, const void* K, const void* V,
                          const uint8_t* row_mask, const uint8_t* col_mask, float* O, void* saved,
                          void* workspace, size_t workspace_bytes, void* stream, st_halo_fn hook, void* user);

st_status st_backward_halo(const st_desc* desc, const void* saved, const void* Q, const void* K,
                           const void* V, const void* dO, const uint8_t* row_mask,
                           const uint8_t* col_mask, float* dQ, float* dK, float* dV, float* d_eps,
                           float* eta_v, int32_t mode, void* workspace, size_t workspace_bytes,
                           void* stream, st_halo_fn hook, void* user, int64_t own_begin,
                           int64_t own_end);

/* Host-side copy of the saved tail duals in the reference's natural-log units:
 * u[3][B*H][L'_q], v[3][B*H][L'_k] (steps T, T+1, T+2; centered when
 * desc->centered, inactive entries 0) and gauge[3][B*H] (the cumulative ledger
 * value mean_valid(u_raw) at those steps).  Masks are HOST pointers (or NULL).
 * Synchronizes `stream`; returns ST_INFEASIBLE_SUPPORT if the forward hit an
 * empty active reduction.  Any output pointer may be NULL. */
st_status st_saved_duals(const st_desc* desc, const void* saved, const uint8_t* row_mask_host,
                         const uint8_t* col_mask_host, double* u, double* v, double* gauge,
                         void* stream);

/* The device status word of a forward (carried in `saved`): synchronizes `stream`
 * and returns ST_OK, ST_INFEASIBLE_SUPPORT (an active row or column had an empty
 * reduction, the reference's InfeasibleSupport thrown inside row_half_step /
 * col_half_step, sinkhorn.hpp:52-56 / :98-102) or ST_CUDA_ERROR (an internal
 * invariant).  st_forward / st_backward are asynchronous and never block on it;
 * call this (or st_saved_duals) where the reference would have thrown. */
st_status st_check_status(const st_desc* desc, const void* saved, void* stream);

/* Host-side support validation (SupportMask::validate): ST_INFEASIBLE_SUPPORT
 * when an active row or column has no active edge.  Masks are HOST pointers. */
st_status st_validate_support(const st_desc* desc, const uint8_t* row_mask_host,
                              const uint8_t* col_mask_host);

/* Counter RNG (rng.hpp): out[k] = scale * counter_normal(seed, tag, start + k),
 * bit-exact with the reference generator.  Host memory, multi-threaded. */
void st_normal_fill(uint64_t seed, const char* tag, uint64_t start, int64_t n, double scale,
                    double* out);
/* out[k] = counter_uniform(fold_tag(seed, tag) + start + k), in [2^-53, 1). */
void st_uniform_fill(uint64_t seed, const char* tag, uint64_t start, int64_t n, double* out);

/* Message of the last non-OK status on this thread. */
const char* st_last_error(void);

/* Number of this library's kernels launched by the calling thread since the
 * last reset (evidence counter for the bench's gpu_launches). */
int64_t st_launch_count(int32_t reset);

#ifdef __cplusplus
}
#endif

#endif /* SINKATTN_H_ */
