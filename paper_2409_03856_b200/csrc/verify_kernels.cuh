// verify_kernels.cuh — argument structs of verify_kernels.cu.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "decode_kernels.cuh"  // PeerAr

namespace sirius {

struct NormRowsArgs {
  const float* base;       // [M, d] residual or NULL (embed mode)
  const float* delta;      // [M, d] or NULL
  const int32_t* tokens;   // embed mode: [M] token ids (else NULL)
  const uint16_t* embed;   // [V, d]
  int vocab, d;
  const uint16_t* norm_w;  // [d]
  float eps;
  float* res_out;          // [M, d] or NULL
  uint16_t* out3;          // [3][plane] bf16: h = t0 + t1 + t2 (split3: fp32 h exactly, as three bf16
  size_t plane;            //          terms for the tensor-core B operand); row m at m * d of each plane
  int par_consume;         // delta = the fused peer all-reduce of the last sync point (GemmArgs.par):
  PeerAr par;              //   wait for every rank's flag, sum the slots of row m in rank order
};

struct RopeStoreArgs {
  const float* qkv;        // [M, (Hr + 2 KVr) * hd]
  const int32_t* start;    // [B] first position of each sequence's rows
  int b_base, rows_per_seq;
  const float* rope_cos;   // [max_seq, hd/2]
  const float* rope_sin;
  int Hr, KVr, hd, max_seq, max_gamma;
  int to_cache;            // 1: K/V -> cache slots pos (prefill); 0: -> staging row stage_base + i (verify)
  int stage_base;          // staging row of the call's row 0 (tree drafting steps); 0 otherwise
  const int32_t* row_off;  // [M] position offset of each row from start (tree rows: their step), or NULL (= i)
  float* q_out;            // [M, Hr * hd] fp32 (post-RoPE)
  uint16_t* k_dst;         // this layer's cache [B, KVr, max_seq, hd] or staging [B, KVr, max_gamma, hd]
  uint16_t* v_dst;
  int* err;
};

struct AttnRowsArgs {
  const float* q;           // [nseq * rows, Hr * hd] fp32 (post-RoPE)
  const int32_t* start;     // [B]  T of each sequence
  int b_base, rows_per_seq, G, Hr, KVr, max_seq;
  const uint16_t* k_cache;  // this layer [B, KVr, max_seq, hd]
  const uint16_t* v_cache;
  const uint16_t* k_fresh;  // staging [B, KVr, fresh_stride, hd] (ignored if fresh_in_cache)
  const uint16_t* v_fresh;
  int fresh_stride, fresh_in_cache;
  int stage_base;                      // staging row of the call's row 0 (tree drafting steps)
  const unsigned long long* tree_vis;  // tree rows: [64] ancestor-or-self bit masks over the staging rows
                                       // (row i sees staging row f iff bit f of tree_vis[stage_base + i]);
                                       // NULL: causal (row i sees staging rows [0, i])
  float* part;              // workspace
  unsigned* counters;       // unused (kept for ABI-internal layout)
  unsigned* group_bar;      // [nseq * KVr * row_blocks][2] barrier (count, generation) of the split groups
  uint16_t* out3;           // [3][plane]: attention output [nseq * rows, Hr * hd] as three bf16 terms
  size_t plane;
  unsigned long long* trace;  // debug: [8][grid CTAs] %globaltimer stamps, or NULL
};

struct RowStat {
  float mx, sum, ld, pad;
  unsigned long long key;
};

struct AcceptStatsArgs {
  const float* logits;     // [M, ldl] (this rank's vocab shard in columns [0, Vr))
  int ldl, Vr, voff, M, gamma, rank;
  const int32_t* tokens;   // [B, gamma] kernel tokens
  RowStat* stats;          // [nranks, M, S]
};

struct AcceptFinalArgs {
  const RowStat* stats;
  int nranks, S, M, gamma, mode;
  float r;
  const int32_t* tokens;
  int32_t* n_accept;
  int32_t* next_token;
  float* q_out;
  int32_t* row_argmax;  // [B, gamma]: the full model's argmax of every verify row (ablation modes)
};

struct KvRewriteArgs {
  const uint16_t* stage_k;  // [L, B, KVr, max_gamma, hd]
  const uint16_t* stage_v;
  uint16_t* k_cache;        // [L, B, KVr, max_seq, hd]
  uint16_t* v_cache;
  const int32_t* start;
  const int32_t* n_rows;
  int B, KVr, hd, max_seq, max_gamma, gamma;
  const int32_t* rows;      // tree commit: staging row of each committed slot [gamma] (batch 1), or NULL
  int* err;
};

namespace launch {
cudaError_t norm_rows(const NormRowsArgs& a, int M, cudaStream_t st);
cudaError_t rope_store(const RopeStoreArgs& a, int M, cudaStream_t st);
cudaError_t attn_rows(const AttnRowsArgs& a, int nseq, int hd, int splits, int row_blocks, cudaStream_t st);
int attn_rows_splits(int nseq, int KVr, int row_blocks, int max_keys, int num_sms);
cudaError_t accept_stats(const AcceptStatsArgs& a, int splits, cudaStream_t st);
cudaError_t accept_finalize(const AcceptFinalArgs& a, int B, cudaStream_t st);
cudaError_t kv_rewrite(const KvRewriteArgs& a, int L, cudaStream_t st);
cudaError_t transpose_bf16(const uint16_t* in, uint16_t* out, int R, int C, cudaStream_t st);
cudaError_t sum_ranks(float* const* bufs_dev, int nranks, size_t rows, size_t width, size_t ld, cudaStream_t st);
}  // namespace launch
}  // namespace sirius
