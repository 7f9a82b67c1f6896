// decode_kernels.cuh — kernel argument structs shared by decode_kernels.cu and runtime.cu.
#pragma once
#include <cstdint>

namespace sirius {

// ---- input prologue modes of the streaming GEMV / fused FFN kernels
enum InMode : int {
  IN_F32 = 0,    // activation already in global (fp32): in_f32 [B, K]
  IN_RESID = 1,  // x = base + delta (delta may be NULL); h = bf16(rmsnorm(x) * norm_w)
  IN_EMBED = 2,  // x = embed[tokens[b]];             h = bf16(rmsnorm(x) * norm_w)
};

// ---- fused peer all-reduce over NVLink peer memory (SURVEY.md §8(e) phase 2; include/sirius.h
// sirius_par_enable).  Every rank owns one comm buffer of the same layout, mapped by its
// peers through CUDA IPC:
//   slots [2][world][slot_n] fp32 | keys [2][world][key_n] u64 | flags [2][world] u64
// indexed (parity of the sync point, SOURCE rank).  The producer kernel's last CTA (the one that
// completes the rank partial) pushes it into slot (par, rank) of every rank, release-stores the sync
// point's sequence number s into flag (par, rank) of every rank, acquire-waits for flags
// (par, 0..world-1) >= s on its own buffer and writes the sum of the slots, in rank order, over the
// partial (the same order on every rank: identical residuals everywhere) — so the next kernel reads
// an all-reduced delta with its usual prologue.  s counts this rank's sync points (device word); all
// ranks make the same sequence of calls, so s agrees.  Two parities suffice: a rank pushes s + 2 only
// after reducing s + 1, which needs every rank's push of s + 1, which each rank makes only after
// reducing s (tests/test_par_protocol.py model-checks this).
struct PeerAr {
  int world;                   // 0: off
  int rank;                    // source index of this rank's pushes
  int fused;                   // 1: the producer's last CTA also waits + reduces (real ranks, loopback);
                               // 0: push only, par_reduce_kernel reduces (single-GPU emulation: the
                               //    emulated ranks' producers run one after another, none may wait)
  int loopback;                // timing proxy (stub comm): every "peer" is this rank's own buffer and
                               // push q lands in source slot q (same stores, no NVLink)
  int slot_n, key_n;           // floats per slot, u64 keys per key slot
  float scale;                 // reduce: sum_r slot_r * scale (1; 1 / world in loopback)
  char* const* peers;          // DEV [world]: every rank's comm buffer as mapped in this process
  char* self;                  // this rank's comm buffer
  unsigned long long* seq;     // this rank's sync-point counter
  unsigned* done;              // producer CTA arrivals (reset by the last CTA)
  int* err;                    // device error word (a peer that never arrives: timeout)
  unsigned long long timeout_ns;  // wait bound (10 s; SIRIUS_PAR_TIMEOUT_MS)
};

struct Prologue {
  int mode;
  const float* in_f32;      // IN_F32
  const float* base;        // IN_RESID [B, K]
  const float* delta;       // IN_RESID [B, K] or NULL
  const int32_t* tokens;    // IN_EMBED [B]
  const uint16_t* embed;    // IN_EMBED [V, K]
  int vocab;
  const uint16_t* norm_w;   // [K]
  float eps;
  float* res_out;           // if non-NULL, CTA 0 stores x [B, K] here (never aliases base)
};

// ---- streaming GEMV: out[b, r] = sum_k W[r, k] * h[b, k]
enum GemvEpi : int { EPI_STORE = 0, EPI_ARGMAX = 1 };

struct GemvArgs {
  Prologue pro;
  const uint16_t* W;  // [rows, K]
  int rows, K;
  int epi;
  float* out;                   // EPI_STORE: [B, ldo]; EPI_ARGMAX: optional logits [B, ldo]
  int ldo;                      // row stride of out
  unsigned long long* amax;     // EPI_ARGMAX: packed (value, lowest index) keys [B]
  uint32_t index_offset;        // EPI_ARGMAX: global vocab offset of row 0 (TP shard)
  int finalize;                 // EPI_ARGMAX: last CTA converts amax -> token_out and resets amax
  unsigned* done_counter;       // EPI_ARGMAX + finalize
  int32_t* token_out;           // EPI_ARGMAX + finalize: [B]
  float* zero_out;              // if non-NULL: the grid zeroes zero_n floats here (the next FFN's accumulator)
  int zero_n;
  PeerAr par;                   // fused all-reduce (world > 0): EPI_STORE: out [B, d] (ldo == d) is
                                // all-reduced in place; EPI_ARGMAX: the packed keys amax [B] are
                                // max-reduced over the ranks (reset to 0) and, fused, -> token_out
};

// ---- fused CATS FFN (gate GEMV + SiLU + threshold + ballot compaction + up/down gathers)
struct FfnArgs {
  Prologue pro;
  const uint16_t *w_gate, *w_up, *w_down;  // [F, d] neuron-major
  int F, d;
  const float* threshold;  // device fp32 (this layer's t_l)
  int dense;               // 1: every neuron active (M_F)
  float* part;             // workspace [grid, B, d] fp32 partial sums
  int* part_cnt;           // workspace [grid, B]
  unsigned long long* barrier;  // grid barrier counter
  float* out;              // [B, d] = sum over active neurons of m_i * W_down[i]
  int32_t* n_active_out;   // [B * n_active_stride] (+layer) or NULL
  int n_active_stride;
  float* gate_out;         // [B * gate_stride] (+layer*F) or NULL: a = SiLU(g)
  long long gate_stride;
  int atomic_out;          // 1: partials added into out (pre-zeroed) with float4 atomics, no grid barrier
  unsigned long long* trace;  // debug: [8][1024] %globaltimer stamps per CTA (phase boundaries), or NULL
  // precomputed-gate mode (top-k FSparse, topk.cu): a = SiLU(g) [B, a_ld] and the selected set as bits
  // [B, m_ld] words come in; no gate rows are read and the threshold is not applied
  const float* a_in;
  const unsigned* mask_in;
  long long a_ld, m_ld;
  PeerAr par;              // fused all-reduce (world > 0): out [B, d] is all-reduced in place
};


// ---- persistent decode step (decode_step.cu): the whole TP-1 decode step in one cooperative launch
struct StepArgs {
  int d, L, Hr, KVr, hd, F, Vr, vocab, max_seq, splits;
  float eps, attn_scale;
  int dense;
  const int32_t* tokens;  // [B]
  const int32_t* pos;     // [B]
  int32_t* token_out;     // [B]
  float* logits_out;      // [B, Vr] or NULL
  int32_t* n_active_out;  // [B, L] or NULL
  float* gate_out;        // [B, L, F] or NULL: a = SiLU(g)
  long long gate_stride;  // = L * F
  const uint16_t *embed, *final_norm, *lm_head;
  const uint16_t* const* attn_norm;  // device arrays [L] of device pointers
  const uint16_t* const* w_qkv;
  const uint16_t* const* w_o;
  const uint16_t* const* ffn_norm;
  const uint16_t* const* w_gate;
  const uint16_t* const* w_up;
  const uint16_t* const* w_down;
  const float* thresholds;  // [L]
  uint16_t *k_cache, *v_cache;  // layer 0; layer stride kv_layer elements
  size_t kv_layer;
  const float *rope_cos, *rope_sin;
  // workspace
  float *x, *x1, *qkv, *o, *attn_part, *ffn_part;
  uint16_t* o3;           // if set: attention output as three bf16 terms (tcgen05 operand planes) instead of o
  size_t o3_plane;
  int* part_cnt;
  unsigned* group_bar;
  unsigned long long* grid_bar;  // dedicated monotone counter (nblocks = grid)
  unsigned long long* amax;
  unsigned* head_cnt;
  int* err;
  int tune;                   // bit 0: evict-first L2 policy on weight loads
  unsigned long long* trace;  // debug: [events][grid] %globaltimer stamps (thread 0 of each CTA), or NULL
};

}  // namespace sirius
