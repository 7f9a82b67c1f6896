// gemm_tc.cuh — tcgen05 GEMM arguments (see gemm_tc.cu).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace sirius {

struct GemmArgs {
  int N, K, M;          // weight rows, reduction length, valid token rows (<= MP)
  int n_tiles, kb;      // ceil(N / 128), ceil(K / 64)
  void* out;            // fp32 [M, ldc] (single) or bf16 hi part [M, ldc] (dual, SwiGLU)
  void* out2;           // dual: bf16 lo part [M, ldc] (m = hi + lo, |m - hi - lo| <= 2^-17 |m|)
  int ldc;
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
};

namespace launch {
constexpr size_t kTmapBytes = 128;  // sizeof(CUtensorMap)
bool make_tmap(void* map, const void* base, uint64_t rows, uint64_t K, uint32_t box_rows);
size_t gemm_workspace_bytes(int num_sms);
// tmA1 == nullptr: single GEMM (fp32 out); else dual gate/up GEMM with SwiGLU bf16 hi/lo epilogue.
// tmBlo != nullptr: the activation operand is the bf16 pair (hi, lo) of an fp32 tensor; both are
// multiplied and accumulated (fp32-grade activations on the bf16 tensor cores).
cudaError_t gemm(const void* tmA0, const void* tmA1, const void* tmB, const void* tmBlo, const GemmArgs& g, int MP,
                 int num_sms, size_t smem_budget, cudaStream_t st);
}  // namespace launch
}  // namespace sirius
