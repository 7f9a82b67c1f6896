/*
 * sirius.h — C ABI of libsirius, the B200 (sm_100a) implementation of the Sirius decode hot path
 * (arXiv 2409.03856, "Sirius: Contextual Sparsity with Correction for Efficient LLMs").
 *
 * The operations and their arguments follow the paper's problem statement, Algorithm 1
 * (PAPER.md:237-271): a prompt, a full model M_F and a sparse model M_S that share weights and a
 * KV cache C ("Require"), a write cursor (here: per-sequence positions), a kernel
 * size n (= gamma here, reading D5) and an acceptance threshold r.
 *
 *   sirius_init         — context: model shape, borrowed weight shards, per-layer CATS thresholds
 *   sirius_prefill      — dense prefill of the prompts (reading D17)
 *   sparse_decode_step  — one decode step of M_S (CATS-sparse FFN, PAPER.md:63/121/182) or of M_F
 *   correct_kernel      — full-model verification of a kernel of gamma positions + likelihood
 *                         accept/reject + interleaved token (Alg. 1 lines 12-18, PAPER.md:258-267;
 *                         §4.2)
 *   kv_rewrite          — commit + rollback: overwrite the committed span with the full model's K/V
 *
 *   sirius_csparse_enable — CSparse draft model: the prompt's fixed neuron set
 *   sirius_tree_kernel  — tree building + tree verification of one kernel
 *   sirius_topk_enable  — top-k FSparse draft model (PAPER.md:121 footnote)
 *   sirius_set_sampling — temperature sampling of drafted / interleaved tokens
 *   sirius_par_export / sirius_par_enable / sirius_par_disable — fused NVLink peer all-reduce (TP > 1)
 *   sirius_destroy / sirius_last_error
 *
 * Conventions (all entry points):
 *  - Return a sirius_status; 0 = OK.  Checks that need only host scalars run synchronously and
 *    return INVALID_ARG / CAPACITY / STATE / UNSUPPORTED without enqueuing anything.  Otherwise the
 *    call enqueues asynchronously on the context's stream and returns OK; the caller synchronises
 *    the stream before reading outputs.
 *  - Device-side checks (positions, n_rows live in device memory so steps can be captured in CUDA
 *    graphs): an offending sequence's writes are suppressed and a sticky device error word is set;
 *    the NEXT call returns SIRIUS_ERR_CAPACITY (and sirius_last_error describes it).
 *  - CUDA / NCCL failures are sticky: the context is unusable afterwards; destroy it.
 *  - Pointers marked DEV are device memory, HOST are host memory.  Every token / position /
 *    output buffer is owned by the caller.  Weights and the stream are borrowed (must outlive the
 *    context).  The context owns the KV cache, the verify staging area and all workspaces.
 *  - A context is single-threaded (one owner at a time).
 *  - Tensor parallelism: every rank makes the same calls with the same scalars
 *    and its own weight shard; token_out / n_accept_out / next_token_out / q_out are identical on
 *    all ranks; logits_out and gate_act_out are rank-local shards.
 */
#ifndef SIRIUS_H_
#define SIRIUS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sirius_ctx sirius_ctx; /* opaque; one per GPU (per rank) */

typedef enum {
  SIRIUS_OK = 0,
  SIRIUS_ERR_INVALID_ARG = -1, /* bad pointer / shape / enum; nothing enqueued                      */
  SIRIUS_ERR_CAPACITY = -2,    /* gamma > max_gamma, rows > capacity, or a sticky device-side
                                  capacity error from a previous call (pos + rows > max_seq,
                                  n_rows outside [1, gamma])                                         */
  SIRIUS_ERR_STATE = -3,       /* call-order violation (kv_rewrite without a preceding
                                  correct_kernel; decode before prefill)                             */
  SIRIUS_ERR_CUDA = -4,        /* sticky                                                             */
  SIRIUS_ERR_NCCL = -5,        /* sticky; includes asynchronous communicator errors, which every
                                  entry point polls (ncclCommGetAsyncError) before enqueuing          */
  SIRIUS_ERR_UNSUPPORTED = -6  /* shape not compiled: head_dim not in {64,128}; d_model % 256;
                                  (n_heads/tp * head_dim) % 64; (ffn_dim/tp) % 8; max_gamma > 64;
                                  batch * max_gamma > 1024; batch not in {1, 2, 4, 8, 16, 32}       */
} sirius_status;

/* Model shape + runtime capacities.  Llama-3 conventions: rotate-half RoPE with base rope_theta,
 * RMSNorm with rms_eps, SiLU-gated MLP, GQA (kv head of q head h = h / (n_heads / n_kv_heads)). */
typedef struct {
  int32_t vocab, d_model, n_layers, n_heads, n_kv_heads, head_dim, ffn_dim;
  float rope_theta, rms_eps;
  int32_t batch;     /* number of sequences (slots 0..batch-1), fixed for the context's life;
                        one of 1, 2, 4, 8, 16, 32 (else SIRIUS_ERR_UNSUPPORTED); batch * max_gamma <= 1024;
                        batch >= 4 decodes through the tensor-core row path        */
  int32_t max_seq;   /* KV capacity per sequence (>= prompt + generated + max_gamma)              */
  int32_t max_gamma; /* max verify rows per sequence per correct_kernel call (<= 64)              */
  int32_t tp_size, tp_rank; /* n_heads, n_kv_heads, ffn_dim, vocab divisible by tp_size (else
                               UNSUPPORTED)                                                      */
} sirius_config;

/* DEVICE pointers to this rank's weight shard: bf16, row-major, a "row" is an output feature or
 * a neuron.  Shard layout per SURVEY.md §8(e): q/k/v heads, W_o columns, neurons and vocab rows
 * split evenly over tp ranks in rank order; embedding and norm weights replicated. */
typedef struct {
  const void* embed;             /* [vocab, d]                                                  */
  const void* final_norm;        /* [d]                                                         */
  const void* lm_head;           /* [vocab/tp, d]  (vocab-parallel)                             */
  const void* const* attn_norm;  /* HOST array [n_layers] of DEV ptrs, each [d]                 */
  const void* const* w_qkv;      /* each [(H + 2 KV)/tp * hd, d]: this rank's q heads, k, v      */
  const void* const* w_o;        /* each [d, H/tp * hd]                                          */
  const void* const* ffn_norm;   /* each [d]                                                     */
  const void* const* w_gate;     /* each [ffn/tp, d]  neuron-major                               */
  const void* const* w_up;       /* each [ffn/tp, d]  neuron-major (= W_up^T)                    */
  const void* const* w_down;     /* each [ffn/tp, d]  neuron-major                               */
} sirius_weights;

/* sparse_decode_step flags */
enum {
  SIRIUS_DENSE = 1u,  /* run M_F (dense FFN) instead of M_S                                            */
  SIRIUS_CSPARSE = 2u, /* run M_S as the CSparse model: the FFN restricted to the last prompt's neuron
                          plan (sirius_csparse_enable), instead of CATS     */
  SIRIUS_TOPK = 4u     /* run M_S as the top-k FSparse model (sirius_topk_enable; PAPER.md:121 footnote
                          "topk on the Gate Layer activations"), instead of the CATS threshold       */
};

/* correct_kernel accept modes */
enum {
  SIRIUS_ACCEPT_THRESHOLD = 0,   /* keep d_{i+1} iff q_i = softmax(l_i)[d_{i+1}] >= r */
  SIRIUS_ACCEPT_EXACT_ARGMAX = 1 /* keep d_{i+1} iff d_{i+1} == argmax l_i (lossless SD greedy)     */
};

/* Create a context.
 *  cfg            HOST, copied.
 *  w              HOST struct of borrowed DEV pointers.  TP emulation on one GPU: if
 *                 cfg->tp_size > 1 and nccl_comm == NULL, `w` points to an array of tp_size
 *                 sirius_weights (rank 0..tp_size-1 shards) and the context runs every rank's
 *                 shard in turn on this GPU, replacing each all-reduce by an in-order sum
 *                 (cfg->tp_rank ignored).  Outputs are then those of the whole TP group (logits_out
 *                 and gate_act_out hold the rank shards concatenated in rank order).
 *  cats_threshold HOST [n_layers] fp32, copied; per-layer CATS threshold t_l >= 0.
 *                 A neuron i of layer l is active iff |SiLU(g_i)| >= t_l (readings D1, D2, D4).
 *  nccl_comm      ncclComm_t (borrowed) when tp_size > 1 with one process per GPU, else NULL.
 *                 (Test/bench only: with the environment variable SIRIUS_DEBUG_STUB_COMM=1 and
 *                 tp_size > 1, a non-NULL comm is never used — every collective is skipped, so one
 *                 GPU runs exactly one rank's share of the work: a compute-only timing proxy of a
 *                 TP rank whose outputs are rank-local partials.)
 *  stream         cudaStream_t (borrowed); every call enqueues on it.
 *  out            receives the context.
 * Errors: INVALID_ARG (NULL / non-positive / inconsistent shape), UNSUPPORTED, CUDA (allocation). */
sirius_status sirius_init(const sirius_config* cfg, const sirius_weights* w, const float* cats_threshold,
                          void* nccl_comm, void* stream, sirius_ctx** out);

/* Dense prefill of every sequence's prompt: writes KV rows [0, prompt_len[b]) of sequence b and
 * returns the dense model's greedy next token (readings D13, D17).
 *  tokens       DEV int32, packed: sequence b's prompt at offset sum_{b'<b} prompt_len[b'].
 *  prompt_len   HOST int32 [batch], each in [1, max_seq - max_gamma].
 *  first_token  DEV int32 [batch]. */
sirius_status sirius_prefill(sirius_ctx* ctx, const int32_t* tokens, const int32_t* prompt_len,
                             int32_t* first_token);

/* One decode step for every sequence: the token token_in[b] at position pos[b] is run through M_S
 * (CATS-sparse FFN: dense gate, |SiLU(g)| >= t_l, only active W_up / W_down rows read) or, with
 * SIRIUS_DENSE, through M_F, or with SIRIUS_CSPARSE through the CSparse model (state error without a
 * plan from sirius_csparse_enable + sirius_prefill; gate_act_out must then be NULL); its K/V are
 * written to cache slot pos[b]; the greedy next token (lowest id on ties) goes to token_out[b].
 * (Alg. 1 "Running sparse model".)
 *  token_in, pos   DEV int32 [batch]; pos[b] in [0, max_seq) (device-checked).
 *  token_out       DEV int32 [batch].
 *  logits_out      DEV fp32 [batch, vocab/tp] or NULL.
 *  n_active_out    DEV int32 [batch, n_layers] or NULL: active neurons per layer (this rank).
 *  gate_act_out    DEV fp32 [batch, n_layers, ffn/tp] or NULL: a = SiLU(g) (debug / parity). */
sirius_status sparse_decode_step(sirius_ctx* ctx, const int32_t* token_in, const int32_t* pos, uint32_t flags,
                                 int32_t* token_out, float* logits_out, int32_t* n_active_out,
                                 float* gate_act_out);

/* Full-model verification of one kernel per sequence (Alg. 1, §4.2):
 * rows [pending, d_1 .. d_{gamma-1}] = kernel_tokens[b, :] at positions start_pos[b] + i are run
 * through M_F in one pass; row i attends to cache[0, start_pos[b]) and to the kernel's own rows
 * [0, i]; the rows' K/V go to the staging area (the cache is NOT modified).  Then
 *   q_i   = softmax(l_i)[d_{i+1}]  (temperature 1, reading D12), i < gamma-1
 *   j     = first i with q_i < r (THRESHOLD) or d_{i+1} != argmax l_i (EXACT_ARGMAX); gamma-1 if none
 *   next  = argmax l_j (interleaved token on rejection, bonus token on accept-all; D10, D11)
 *  kernel_tokens   DEV int32 [batch, gamma].
 *  start_pos       DEV int32 [batch] = T (cache length before the kernel; device-checked
 *                  T + gamma <= max_seq).
 *  gamma           1 .. max_gamma;  accept_threshold r in [0, 1];  accept_mode as above.
 *  n_accept_out    DEV int32 [batch] = j in [0, gamma-1].
 *  next_token_out  DEV int32 [batch].
 *  q_out           DEV fp32 [batch, gamma] or NULL; q[gamma-1] = probability of argmax l_{gamma-1}.
 *  logits_out      DEV fp32 [batch, gamma, vocab/tp] or NULL. */
sirius_status correct_kernel(sirius_ctx* ctx, const int32_t* kernel_tokens, const int32_t* start_pos,
                             int32_t gamma, float accept_threshold, int32_t accept_mode, int32_t* n_accept_out,
                             int32_t* next_token_out, float* q_out, float* logits_out);

/* Commit + rollback after correct_kernel ("Enables Full to directly rewrites KV Cache",
 * :264 "Rollback", :294): staging rows [0, n_rows[b]) of the last correct_kernel overwrite cache
 * slots [start_pos[b], start_pos[b] + n_rows[b]) in every layer.  Normally n_rows = n_accept + 1;
 * rows beyond are dead and are overwritten by the next drafts.
 *  start_pos  DEV int32 [batch] (same values as the preceding correct_kernel).
 *  n_rows     DEV int32 [batch], each in [1, gamma of that call] (device-checked).
 * Errors: STATE if no correct_kernel preceded it. */
sirius_status kv_rewrite(sirius_ctx* ctx, const int32_t* start_pos, const int32_t* n_rows);

/* Tree correction kernel: hardware-friendly tree building and verification (PAPER.md
 * :299-319 §4.3; reading D29).  Batch 1, TP 1.  One call replaces the gamma-1 sparse_decode_step calls
 * and correct_kernel of a kernel: the sparse model drafts a fixed-shape tree of `width` nodes per step
 * (step 1: the pending token's top max(width, branch) tokens; later steps: every node's top `branch`
 * tokens) kept by cumulative log-likelihood (ties to the lower parent rank, then the lower token id);
 * the full model verifies all 1 + (gamma-1)·width rows in one forward with ancestor masks; every leaf's
 * path is scanned as in correct_kernel and the longest accepted path wins (ties to the higher leaf
 * cumulative log-likelihood, then the lower leaf row); the interleaved token is the full model's argmax
 * at the cut.  The following kv_rewrite commits the winning path's full-model K/V.
 *  pending          DEV int32 [1]: the pending token (position T).
 *  start_pos        DEV int32 [1] = T.
 *  gamma            kernel size; 1 + (gamma-1)·width <= min(64, max_gamma) (else CAPACITY).
 *  width, branch    tree width in [1, 8] (width 1: the greedy chain), children per node in [1, 8].
 *  accept_threshold, accept_mode   as correct_kernel.
 *  n_accept_out     DEV int32 [1] = j, accepted nodes on the winning path.
 *  next_token_out   DEV int32 [1] = the full model's argmax at the cut node.
 *  path_tokens_out  DEV int32 [gamma]: the winning path's tokens, pending first; entries > j are -1.
 * Errors: INVALID_ARG, CAPACITY, UNSUPPORTED (batch != 1 or tp_size != 1), CUDA. */
sirius_status sirius_tree_kernel(sirius_ctx* ctx, const int32_t* pending, const int32_t* start_pos, int32_t gamma,
                                 int32_t width, int32_t branch, float accept_threshold, int32_t accept_mode,
                                 int32_t* n_accept_out, int32_t* next_token_out, int32_t* path_tokens_out);

/* Sampled decoding (Alg. 1 "sample" PAPER.md:253 / :267, "the temperature of 0.6
 * works well" PAPER.md:296; reading D31).  temperature > 0: sparse_decode_step samples its token and
 * correct_kernel samples the interleaved / bonus token (instead of argmax), each from softmax(l / T)
 * of the model that produces it, by inverse CDF over the vocabulary in index order with the uniform
 *   u = (splitmix64(seed ^ splitmix64(b * 2^32 + p)) >> 40) / 2^24
 * keyed by the sequence b and the absolute position p of the token being placed (a counter-based
 * generator: the same (seed, b, p) always draws the same u).  The acceptance probability q keeps
 * temperature 1 (reading D12); the prefill's first token stays greedy (reading D17).  temperature 0
 * (default) restores greedy decoding.  The decode of a context with sampling never takes the
 * persistent step kernel.
 * Errors: INVALID_ARG (temperature < 0 or not finite); UNSUPPORTED (tp_size > 1).  Synchronous. */
sirius_status sirius_set_sampling(sirius_ctx* ctx, float temperature, uint64_t seed);

/* Top-k FSparse (PAPER.md:121 footnote: the paper's own FSparse "uses topk on the
 * Gate Layer activations"; reading D30): sparse_decode_step(..., SIRIUS_TOPK) keeps, per layer and
 * sequence, the k = round(keep_fraction * ffn) neurons of largest |SiLU(g)| (exact ties to the lower
 * index) — gate GEMV, exact radix selection, then only the selected W_up / W_down rows.  Unlike the
 * threshold the set depends on the whole layer, so TP > 1 would need a global selection: TP 1 only.
 * keep_fraction 0 disables.
 * Errors: INVALID_ARG (keep_fraction outside [0, 1]); UNSUPPORTED (tp_size > 1, batch > 4, k = 0);
 * CUDA (allocation).  Synchronous. */
sirius_status sirius_topk_enable(sirius_ctx* ctx, float keep_fraction);

/* CSparse / Griffin-style coarse-grained sparsity (§2.1 "within the
 * same input prompt, the sparsity pattern is fixed for all tokens generated", :182 §3.2 the pattern is
 * set after prefilling so the gate is sparse too, :471 the paper's latency numbers use Griffin).
 * After this call every sirius_prefill also accumulates, per layer and neuron of this rank's shard, the
 * statistic s_i = sum over the prompt of |SiLU(g_i)| of the dense model, and then keeps the
 * k = round(keep_fraction * ffn/tp) neurons with the largest s_i (exact ties to the lower index;
 * reading D28), gathering their W_gate / W_up / W_down rows into context-owned compact matrices
 * (3 k d bf16 per layer).  sparse_decode_step(..., SIRIUS_CSPARSE) then runs the FFN as the dense
 * SiLU-gated MLP of the kept neurons.  keep_fraction 0 disables.  TP > 1: each rank keeps the top
 * k of its own shard.
 * Errors: INVALID_ARG (keep_fraction outside [0, 1]); UNSUPPORTED (batch != 1, or k not a positive
 * multiple of 8); CUDA (allocation).  Synchronous. */
sirius_status sirius_csparse_enable(sirius_ctx* ctx, float keep_fraction);

/* Fused peer all-reduce of the tensor-parallel decode step (SURVEY.md §8(e) phase 2: "fuse the
 * all-reduce into the O-proj / down-proj epilogue over NVLink peer memory"; the per-layer all-reduces
 * of S3 and S6 and the LM-head argmax combine of S7 in SURVEY.md §8(a); the paper itself runs on one
 * GPU).  Each rank owns a comm buffer of identical layout
 *   slots [2][tp_size][batch * d_model] fp32 | keys [2][tp_size][8] u64 | flags [2][tp_size] u64
 * that every other rank maps through CUDA IPC.  With the fused path on, sparse_decode_step (per-stage
 * path: batch <= 2, or <= 8 with SIRIUS_DECODE_ROWS=0) launches no collective: the CTA that completes the
 * rank partial of the O-proj GEMV / CATS FFN (or the packed argmax keys of the LM head) stores it into
 * its slot on every rank over NVLink, release-stores the sync point's sequence number into the flags,
 * acquire-waits for every rank's flag and writes the rank-order sum over the partial (the head: the
 * global argmax token), so every rank computes bitwise the same residual and the next kernel reads it
 * as at TP 1.  The verify / batched-row forward (correct_kernel, the tree kernel, batched decode: at
 * most 128 rows and batch * max_gamma rows) does the same from the O-proj / down-proj tcgen05 GEMM
 * epilogues, and the next row-norm kernel waits and sums.  The prefill's all-reduces and
 * correct_kernel's all-gather of per-row softmax statistics stay on NCCL.
 *
 * sirius_par_export: HOST handle_out [SIRIUS_PAR_HANDLE_BYTES] = this rank's cudaIpcMemHandle_t.
 *   Errors: STATE for an emulated / stub / tp_size 1 context; CUDA.
 * sirius_par_enable: peer_handles = HOST [tp_size][SIRIUS_PAR_HANDLE_BYTES], every rank's exported
 *   handle in rank order (the own entry is ignored), or NULL for a single-GPU emulated context (the
 *   ranks' buffers are all in this process; the emulated ranks run one after another, so each one's
 *   wait + reduction runs in a separate kernel once all have pushed) or a SIRIUS_DEBUG_STUB_COMM
 *   context (loopback timing proxy of the fused form: every peer is the rank's own buffer, the
 *   reduction sums tp_size copies scaled by 1 / tp_size).  Every rank
 *   must call it (collectively, after every rank's sirius_init and export) before its next decode.
 *   Errors: INVALID_ARG (handles given / missing for the context kind); UNSUPPORTED (tp_size 1 or
 *   > 8; a peer buffer cannot be mapped); CUDA.  Synchronous.
 * sirius_par_disable: back to the NCCL collectives (the mappings stay until sirius_destroy); all ranks.
 * A rank that does not arrive within 10 s makes the waiting ranks' next call return SIRIUS_ERR_NCCL. */
#define SIRIUS_PAR_HANDLE_BYTES 64
sirius_status sirius_par_export(sirius_ctx* ctx, void* handle_out);
sirius_status sirius_par_enable(sirius_ctx* ctx, const void* peer_handles);
sirius_status sirius_par_disable(sirius_ctx* ctx);

/* The full model's greedy token (argmax, lowest id on ties) of EVERY verify row of the last
 * correct_kernel call — the interleaving candidates of the component ablation without rollback
 * (Table 4: "only letting the LLM correct the token it is evaluating"; reading
 * D27).  out: DEV int32 [batch, gamma of that call]; enqueued on the stream (async copy).
 * Errors: STATE if no correct_kernel preceded it. */
sirius_status sirius_verify_row_argmax(sirius_ctx* ctx, int32_t* out);

sirius_status sirius_destroy(sirius_ctx* ctx);

/* Human-readable description of the last error on ctx (static storage inside ctx; never NULL). */
const char* sirius_last_error(const sirius_ctx* ctx);

/* Library build identification ("sm_100a ..."); never NULL. */
const char* sirius_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SIRIUS_H_ */
