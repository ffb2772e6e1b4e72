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
};

long long launch_count(bool reset);

cudaError_t launch_scores(const Geo& g, int dtype, const void* Q, const void* K, float* S2, cudaStream_t s);
cudaError_t launch_row_step(const Geo& g, bool first, const float* S2, const float* v, const float* u_prev,
                            float* u_out, int* err, cudaStream_t s);
cudaError_t launch_col_step(const Geo& g, bool first, const float* S2, const float* u, const float* v_prev,
                            float* v_out, int* err, cudaStream_t s);
cudaError_t launch_output(const Geo& g, int dtype, const float* S2, const float* u, const float* v, const void* V,
                          float* O, cudaStream_t s);
cudaError_t launch_gauges(const Geo& g, const float* u_slots, int nslots, float* gauge, cudaStream_t s);
cudaError_t launch_backward(const Geo& g, int dtype, const BwdPtrs& p, bool direct, cudaStream_t s);
cudaError_t launch_deps_reduce(const Geo& g, const float* part, float* out, cudaStream_t s);
cudaError_t launch_scale(const float* src, float* dst, long n, float sc, cudaStream_t s);

}  // namespace st
