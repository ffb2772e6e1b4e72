// st_phase.cuh -- host interface of the tcgen05 half-step kernels (st_phase.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace st {

// One half-step.  "own" = the side whose dual is updated (rows of the MMA
// tile, one TMEM lane each); "other" = the window side (MMA N dimension).
struct alignas(64) PhaseArgs {
    // tensor maps of the raw [BH][L][d] bf16 tensors of the own / other side (tma = 1: the operand tiles are
    // loaded from them as 64-row x 128-byte SWIZZLE_128B boxes and no packed plane is read)
    CUtensorMap tmA, tmB;
    int tma;
    int npl;            // operand planes: 1 (bf16 inputs) or 3 (fp32 inputs split into bf16 hi/mid/lo)
    int CR;             // window chunk rows = MMA N (64 or 128)
    int shift;          // packed row = row + shift: aligns the chunk grid with every band window
    int NA, NSK;        // A buffers (1-2), B chunk ring slots
    int row_bytes;      // d * 2 (one bf16 plane)
    int maxwin;         // floats reserved per window-dual buffer
    int H, NB;          // heads per example, 128-row blocks per head (own side)
    int L_own, L_other, Lr_own, Lr_other, Lp_own, Lp_other;
    int w, dustbin;
    float c2, sd2;
    const uint8_t* mask_own;    // [B, L_own] or null
    const uint8_t* mask_other;  // [B, L_other] or null
    const uint8_t* A_pack[3];   // packed planes of the own side  [BH][Lp_own][d] bf16
    const uint8_t* B_pack[3];   // packed planes of the other side
    const float* dual_other;    // [BH][Lr_other] (read only for the dustbin entry)
    const float* pad_other;     // [BH][pad_ld_other] masked padded duals of the other side (see launch_pad_fill)
    float* pad_own;             // [BH][pad_ld_own] same for the own side: previous duals in, new duals out
    int pad_ld_own, pad_ld_other, pad_off;
    const float* off_own;       // [BH][Lr_own] previous dual of the own side
    float* out_own;             // [BH][Lr_own]
    const int* work;            // active (head, block) list
    const int* nwork;
    int nwork_all;              // work == null: every block 0 .. nwork_all-1 (band write passes)
    float* band_out;            // band write passes: [BH][band_ld][Wf] (null for the half-step)
    int band_ld, Wf;
    int ew_write;               // band write passes: epilogue warps (16, or 8 to fit SMEM)
    int wl_cap;                 // max work items per CTA (SMEM copy of the CTA's work-list slice)
    int* err;
    unsigned long long* trace;  // debug timeline (null in production)
    int dbg;                    // development ablations (ST_PHASE_DBG): 1 = skip epilogue math, 2 = one MMA K-step
};

struct DustArgs {
    int H, L_own, L_other, Lr_own, Lr_other;
    float sd2;
    const uint8_t* mask_other;
    const float* dual_other;
    const float* off_own;
    float* out_own;
    int* err;
};

long long phase_launch_count(bool reset);
size_t phase_smem_bytes(const PhaseArgs& a);
cudaError_t launch_phase(const PhaseArgs& a, bool first, int grid, cudaStream_t s);
cudaError_t launch_dustbin(const DustArgs& a, bool first, int BH, cudaStream_t s);
// the score band (cotangent = false: s2 = q.k c2, -inf off the support) or the cotangent band
// (cotangent = true: dO.v, 0 off the support) of the own side, from packed bf16 planes on tcgen05
cudaError_t launch_phase_band(const PhaseArgs& a, bool cotangent, int grid, cudaStream_t s);
// [BH][Lr][d] (f32 or bf16) -> npl bf16 planes [BH][Lp][d] in the K-major core-matrix
// layout, row r stored at packed row r + shift (other packed rows zero).
cudaError_t launch_pack(int dtype, const void* X, int BH, int L, int Lr, int Lp, int d, int shift, uint8_t* p0,
                        uint8_t* p1, uint8_t* p2, cudaStream_t s);
// pad[bh][pad_off + j] = active(j) ? (src ? src[bh][j] : 0) : -inf; guards -inf
cudaError_t launch_pad_fill(float* pad, const float* src, int BH, int H, int L, int Lr, int pad_ld, int pad_off,
                            const uint8_t* mask, cudaStream_t s);
// Full-step bf16 solve (st_fstep16.cu): one S evaluation per Sinkhorn step.  part: column partials
// [BH][NB][maxwin]; k_vmerge folds them into the padded column duals (and v_out when non-null).
size_t fstep16_smem_bytes(const PhaseArgs& a);
long long fstep16_launch_count(bool reset);
cudaError_t launch_fstep16(const PhaseArgs& a, float* part, bool first, int grid, cudaStream_t s);
cudaError_t launch_vmerge(const float* part, float* pad_v, float* v_out, int BH, int H, int Lq, int Lk, int Lrk, int NB,
                          int maxwin, int w, int CR, int shift, int Lp_other, int pad_ld, int pad_off,
                          const uint8_t* col_mask, int* err, cudaStream_t s);
cudaError_t launch_compact(const int* flags, int n, int* work, int* count, cudaStream_t s);
cudaError_t launch_worklist(const uint8_t* mask, int H, int BH, int L, int NB, int* flags, int* work, int* count,
                            cudaStream_t s);

}  // namespace st
