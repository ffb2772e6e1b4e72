// st_bfree.cuh -- host interface of the band-free tcgen05 sweeps (st_bfree.cu): the transport
// output O = P V (apply_transport, sinkhorn.hpp:257-277) and the exact R=2 adjoint
// (r2_backward, adjoint.hpp:232-373) for bf16 inputs WITHOUT any stored L x W band: every sweep
// recomputes its score tile S = Q K^T (and the cotangent tile Z = dO V^T where the stage needs
// it) per 128-row block on the tensor cores, straight from the packed O(L d) operand planes.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace st {

// Geometry of the band-free path (bf16 planes, no dustbin, w a multiple of 64).
struct BfGeo {
    int BH, H;
    int Lq, Lk, Lrq, Lrk;   // rows / columns; strides of the API tensors
    int Lpq, Lpk;           // packed rows / columns (multiples of 128)
    int d, w;
    float c2, inv_qk;
    const uint8_t* row_mask;  // [B, Lq] or null
    const uint8_t* col_mask;  // [B, Lk] or null
};

// O(L) vector workspace of the band-free sweeps: fp32 arrays [BH][Lpq] (row side) and [BH][Lpk]
// (column side); exponent-offset arrays carry -inf on inactive / padding entries.
constexpr int kBfRowVecs = 6;  // U2, U1, ALPHA, U2B, AU1, U1B
constexpr int kBfColVecs = 8;  // V2, V1, V0, BETA, DELTA, GV, BV1, V1B
inline size_t bfree_vec_bytes(int BH, int Lpq, int Lpk) {
    return sizeof(float) * (size_t)BH * ((size_t)kBfRowVecs * Lpq + (size_t)kBfColVecs * Lpk);
}

bool bfree_supported(int d, int w, int dustbin, int esz);
long long bfree_launch_count(bool reset);

// O = P^(T+R,T+R) V.  qp / kp / vp: packed bf16 planes [BH][Lp][d] (launch_pack, shift 0);
// u / v: the final raw duals (base 2) in the API layout; vec: the vector workspace.
// true when the driver exposes cuTensorMapEncodeTiled: the V / dO streams then come straight from the raw
// tensors through tensor maps (cp.async.bulk.tensor, SWIZZLE_128B) and vp / gp may be null
bool bfree_tma_available();
// tensor map of a raw [BH][Lr][d] bf16 tensor: boxes of 64 rows x 64 columns (128 bytes), SWIZZLE_128B, zero fill
bool bfree_make_tmap(CUtensorMap* m, const void* base, int BH, int Lr, int d, int box_rows = 64);
cudaError_t launch_bfree_output(const BfGeo& g, const uint8_t* qp, const uint8_t* kp, const uint8_t* vp, const void* Qraw,
                                const void* Kraw, const void* Vraw, const float* u, const float* v, float* vec, float* O,
                                cudaStream_t s);

struct BfBwd {
    const uint8_t *qp, *kp, *vp, *gp;     // packed Q, K, V, dO
    const float *u1, *u2, *v0, *v1, *v2;  // saved raw tail duals (base 2), API layout
    const void *Q, *K;                    // raw Q, K [BH][Lr][d] bf16 (tensor-map sources)
    const void* V;                        // raw V [BH][Lrk][d] bf16 (g_v = <V_j, dV_j>; tensor-map source)
    const void* dO;                       // raw dO [BH][Lrq][d] bf16 (tensor-map source)
    float* vec;                           // vector workspace (bfree_vec_bytes)
    float *dQ, *dK, *dV;                  // [BH][Lr][d] fp32
    float* deps_part;                     // [BH][Lrq]
    float* eta_v;                         // [BH][Lrk]  (v0_bar)
};
cudaError_t launch_bfree_backward(const BfGeo& g, const BfBwd& p, bool direct, cudaStream_t s);

}  // namespace st
