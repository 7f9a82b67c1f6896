// tree.cuh — state of a tree correction kernel (tree.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sirius {

constexpr int kTreeMaxRows = 64;  // flattened rows 1 + (gamma-1) W (64-bit ancestor masks)
constexpr int kTreeMaxW = 8;      // tree width
constexpr int kTreeMaxKB = 8;     // candidates kept per row (max(width, branch))

struct TreeState {                     // device-resident, one per context (batch 1)
  int32_t tok[kTreeMaxRows];           // token of each flattened row
  int32_t parent[kTreeMaxRows];        // parent row (-1 for the root)
  float cum[kTreeMaxRows];             // cumulative sparse log-likelihood of the row's path
  unsigned long long vis[kTreeMaxRows];  // ancestor-or-self mask over the rows
  int32_t row_off[kTreeMaxRows];       // position offset from T (the row's step)
  int32_t path[kTreeMaxRows];          // winning path rows (root first), for the KV commit
  float lse[kTreeMaxRows];             // log-sum-exp of the row's logits (last topk launch over it)
  float q[kTreeMaxRows];               // full-model probability of the row's token given its ancestors
  unsigned long long top[kTreeMaxRows][kTreeMaxKB];  // best (value, lowest index) keys, descending
};

namespace launch {
cudaError_t tree_init(TreeState* ts, const int32_t* pending, cudaStream_t st);
cudaError_t tree_topk(const float* logits, int ldl, int V, int rows, int kb, TreeState* ts, int row_base,
                      cudaStream_t st);
cudaError_t tree_prune(TreeState* ts, int s, int W, int branch, cudaStream_t st);
cudaError_t tree_accept(const float* logits, int ldl, TreeState* ts, int S, int W, float r, int mode, int32_t* n_accept,
                        int32_t* next_token, int32_t* path_tokens, int gamma, cudaStream_t st);
}  // namespace launch
}  // namespace sirius
