// gemm_tc.cuh — tcgen05 GEMM arguments (see gemm_tc.cu).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "decode_kernels.cuh"  // PeerAr

namespace sirius {

struct GemmArgs {
  int N, K, M;          // weight rows, reduction length, valid token rows (<= MP)
  int n_tiles, kb;      // ceil(N / 128), ceil(K / 64)
  void* out;            // fp32 [M, ldc] (single) or bf16 [3][out_plane] (dual, SwiGLU: m as three
  size_t out_plane;     //   bf16 terms, split3 — the next GEMM's B operand planes)
  int ldc;
  int nterms;           // B operand terms (1: plain bf16 activations; 3: fp32 activations split3)
  int plane_rows;       // rows between the B operand's term planes in its tensor map
  int row0;             // first B operand row of this launch (row chunks of large M)
  int coarse;           // 1: one TMA op per stage per operand (3-D weight / 4-D activation boxes);
                        // 0: one op per 64-wide weight box and per 16-row activation term box
  float* part;          // stream-K partials [num_sms, 2, NACC, 256, 128]
  unsigned* counters;   // [n_tiles] (self-resetting)
  unsigned long long* trace;  // debug: [8][grid] %globaltimer stamps of thread 0 / the MMA thread, or NULL
  // dual (SwiGLU) epilogue only: CATS mask of the batched sparse decode — m = 0 unless
  // |SiLU(g)| >= *thr (thr NULL: dense); optional per-row active counts and a = SiLU(g) export
  const float* thr;
  int* n_active;           // [M rows] stride n_active_stride, or NULL
  int n_active_stride;
  float* gate_out;         // [M rows] stride gate_stride, or NULL
  long long gate_stride;
  // single (fp32 out, ldc == d) only: fused peer all-reduce of the verify / batched-row forward
  // (SURVEY.md §8(e) phase 2; peer_ar.cuh): every output element is also stored into this rank's slot
  // on every rank over NVLink as the epilogue writes it; the last of par_ctas CTAs (those with work)
  // release-stores the sync point's sequence number into every rank's flag.  The consumer (norm_rows)
  // waits for the flags and sums the slots in rank order.
  PeerAr par;
  int par_ctas;
};

namespace launch {
size_t gemm_workspace_bytes(int num_sms);
// w1 == nullptr: single GEMM (fp32 out); else dual gate/up GEMM with the SwiGLU epilogue.  w0, w1: bf16
// weights [N, K] row-major.  x: the activation operand, g.nterms planes of g.plane_rows rows each
// ([nterms][plane_rows][K] bf16); with 3 terms (split3 of an fp32 tensor) every term is multiplied and
// accumulated: fp32 activations on the bf16 tensor cores, exactly represented.  The tensor maps are
// encoded here for the launch's tile shape (captured by value when the launch is graph-captured).
cudaError_t gemm(const void* w0, const void* w1, const void* x, const GemmArgs& g, int MP, int num_sms,
                 size_t smem_budget, cudaStream_t st);
}  // namespace launch
}  // namespace sirius
