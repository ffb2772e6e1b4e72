// st_kernels.cuh -- host-side launchers of the sm_100a band kernels.
#pragma once

#include <cuda_runtime.h>

#include "st_common.cuh"

namespace st {

struct BwdPtrs {
    const float* S2;
    const float *u1, *u2, *v0, *v1, *v2;
    float *g_u, *g_v, *u2b, *v1b, *u1b, *v0b;
    const void *Q, *K, *V, *dO;
    float *dQ, *dK, *dV, *deps_part;
    const float *Zd = nullptr, *ZdT = nullptr;  // dustbin dots (tile backward)
    float* dpart = nullptr;                     // [BH][8][129] dustbin line partials (null: generic kernels)
};

// extra bands of the tile backward (st_bwd.cu)
struct BwdTPtrs {
    const float *S2T, *Z, *ZT;
    float *Zd, *ZdT;
};

struct FStepPtrs {
    const float* S2;
    const float* u_prev;
    float* u_out;
    const float* v_pp;
    float* v_p_out;
    float* v_p_slot;
    const float* part_in;
    const float* partm_in;
    float* part_out;
    float* partm_out;
    int* err;
};
size_t fstep_smem_bytes(const Geo& g);
cudaError_t launch_fstep(const Geo& g, int t, const FStepPtrs& p, cudaStream_t s);
cudaError_t launch_ffinal(const Geo& g, int t_last, const FStepPtrs& p, cudaStream_t s);

// persistent band-resident solve (st_fsolve.cu)
struct FSolvePtrs {
    const float* S2;
    float* ubuf;
    float* vbuf;
    float* u_slot[9];   // saved u / v at tail steps T .. T+8 (or null)
    float* v_slot[9];
    void* part[2];    // tagged 64-bit partials [BH][NB][128+2w]
    void* partm;
    float* vpriv;     // [BH*NB][128+2w]
    int* flags;
    int* work;
    int* count;
    int* err;
    int nst;            // epsilon stages of the base solve (run-length): steps <= st_end[q] scale by st_scale[q]
    int st_end[8];
    float st_scale[8];
};
size_t fsolve_smem_bytes(const Geo& g);
bool fsolve_supported(const Geo& g);
cudaError_t launch_fsolve(const Geo& g, int T, int R, const FSolvePtrs& p, cudaStream_t s);

long long launch_count(bool reset);
void add_launches(long long n);
size_t bwdT_smem_bytes(const Geo& g);
bool bwdT_supported(const Geo& g);
// host hook after each adjoint sweep that produces a vector the neighbours' sweeps read
// (sequence sharding, st_backward_halo): kind 0 = row vector [BH][Lrq], 1 = column vector [BH][Lrk]
struct BwdHook {
    void (*fn)(void* user, int32_t kind, float* vec, int64_t len, void* stream);
    void* user;
    int64_t nq, nk;  // vector lengths
};
cudaError_t launch_backward_tile(const Geo& g, int dtype, const BwdPtrs& p, const BwdTPtrs& t, bool direct,
                                 cudaStream_t s, long long& launches, const BwdHook* hook = nullptr);
// generic-R tail adjoint (adjoint.hpp:132-200): u[t] / v[t] = raw duals of step T+t (base 2),
// ub[t] / vb[t] = their cotangents (written), t = 0..R
constexpr int kMaxTailSteps = 8;
struct TailPtrs {
    int R;
    const float* u[kMaxTailSteps + 1];
    const float* v[kMaxTailSteps + 1];
    float* ub[kMaxTailSteps + 1];
    float* vb[kMaxTailSteps + 1];
    float* g_u;    // scratch [BH][Lrq]
    float* eta_u;  // R = 0: the base cotangent's u part g_u (may be null)
};
cudaError_t launch_tail_adjoint(const Geo& g, int dtype, const TailPtrs& tp, const float* S2, const float* S2T,
                                float* Z, float* ZT, const void* Q, const void* K, const void* V, const void* dO,
                                float* dQ, float* dK, float* dV, float* deps_part, cudaStream_t s,
                                long long& launches);
// base_solve_vjp (certificates.hpp:25-70): hu / hv = the base duals u_h, v_h of steps h = 0..T
// ([T+1][BH][Lr], base 2); lam[h] = eps / eps_h (host, h = 1..T)
struct BaseVjpPtrs {
    int T;
    const float *hu, *hv;
    const float* lam;
    const void *Q, *K;
    float *S2, *S2T, *A, *AT;  // score band (+T) at the running stage; raw-score cotangent band (+T)
    const float *eta_u, *eta_v;
    float *ab, *vb[2], *zero_u;
    float *dQ, *dK, *deps_part;
};
cudaError_t launch_base_vjp(const Geo& g, int dtype, const BaseVjpPtrs& p, cudaStream_t s, long long& launches);
cudaError_t launch_output_tile(const Geo& g, int dtype, const float* S2, const float* u, const float* v, const void* V,
                               float* O, cudaStream_t s);
// the dustbin row / column of one backward stage through the generic sweeps
cudaError_t launch_backward_dustbin_stage(const Geo& g, int dtype, const BwdPtrs& p, bool direct, int stage,
                                          cudaStream_t s);

cudaError_t launch_scores(const Geo& g, int dtype, const void* Q, const void* K, float* S2, cudaStream_t s);
cudaError_t launch_row_step(const Geo& g, bool first, const float* S2, const float* v, const float* u_prev,
                            float* u_out, int* err, cudaStream_t s);
cudaError_t launch_transpose_band(const Geo& g, const float* S2, float* S2T, cudaStream_t s, float fill);
bool band_dual_supported(const Geo& g);
cudaError_t launch_band_dual(const Geo& g, int dtype, bool z, const void* A, const void* B, float* out, float* outT,
                             cudaStream_t s);
cudaError_t launch_zband(const Geo& g, int dtype, const void* dO, const void* V, float* Z, cudaStream_t s);
size_t stepT_smem_bytes(const Geo& g);
cudaError_t launch_stepT(const Geo& g, bool first, const float* S2, const float* dual_other, const float* off_own,
                         float* out_own, int* err, cudaStream_t s);
cudaError_t launch_col_step(const Geo& g, bool first, const float* S2, const float* u, const float* v_prev,
                            float* v_out, int* err, cudaStream_t s);
cudaError_t launch_output(const Geo& g, int dtype, const float* S2, const float* u, const float* v, const void* V,
                          float* O, cudaStream_t s, int last_only = 0, float* dpart = nullptr);
cudaError_t launch_gauges(const Geo& g, const float* u_slots, int nslots, float* gauge, cudaStream_t s);
cudaError_t launch_backward(const Geo& g, int dtype, const BwdPtrs& p, bool direct, cudaStream_t s);
cudaError_t launch_deps_reduce(const Geo& g, const float* part, float* out, cudaStream_t s, int i_begin = 0,
                               int i_end = -1);
cudaError_t launch_scale(const float* src, float* dst, long n, float sc, cudaStream_t s);

}  // namespace st
