// runtime.cu — libsirius runtime: context, static KV slabs, workspaces, tensor maps, TP all-reduces
// (NCCL over NVLink, or the single-GPU in-order emulation), and the C-ABI entry points declared in
// include/sirius.h.  The Sirius loop itself (Algorithm 1) is driven by the caller through these
// entry points; every arithmetic step runs in the kernels of decode_kernels.cu, gemm_tc.cu and
// verify_kernels.cu.
#include <dlfcn.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/sirius.h"
#include "common.cuh"
#include "decode_kernels.cuh"
#include "gemm_tc.cuh"
#include "verify_kernels.cuh"
#include "tree.cuh"

namespace sirius {
namespace launch {
int gemv_grid(int rows, int num_sms);
cudaError_t gemv(const GemvArgs& a, int B, int grid, cudaStream_t st);

cudaError_t argmax_finalize(unsigned long long* amax, int B, int32_t* token_out, cudaStream_t st);
cudaError_t par_reduce(const PeerAr& p, float* dst, int n, int nk, int32_t* token_out, cudaStream_t st);
int ffn_grid(int F, int num_sms);
cudaError_t ffn(const FfnArgs& a, int B, int grid, cudaStream_t st);
bool decode_step_supported(int d, int H, int KV, int hd, int F, int num_sms);
int decode_step_splits(int B, int KV, int num_sms);
cudaError_t decode_step(const StepArgs& a, int B, int grid, cudaStream_t st);
bool attn_stage_supported(int hd, int G);
extern int g_gemm_kbox;
extern int g_gemm_coarse;
cudaError_t attn_stage(const StepArgs& a, int l, int B, cudaStream_t st);
cudaError_t csparse_colsum(const float* a, int M, int F, long long lda, float* stats, cudaStream_t st);
cudaError_t csparse_select(const float* stats, int L, int F, int k, int32_t* idx, cudaStream_t st);
cudaError_t topk_select(const float* g, long long ldg, int F, int k, float* a_out, long long lda, unsigned* mask,
                        long long ldm, int B, cudaStream_t st);
cudaError_t sample_tokens(const float* logits, int ldl, int V, float temperature, unsigned long long seed,
                          const int32_t* base_pos, const int32_t* jsel, int rows_per_b, int32_t* out, int B,
                          cudaStream_t st);
cudaError_t csparse_gather(const uint16_t* src, const int32_t* idx, int k, int d, uint16_t* dst, int num_sms,
                           cudaStream_t st);
}  // namespace launch
}  // namespace sirius

using namespace sirius;

// ----------------------------------------------------------------------------- NCCL (dlopen'd)
namespace {
typedef int ncclResult_t_;
struct NcclUid {  // ncclUniqueId: passed BY VALUE to ncclCommInitRank (a 128-byte struct, not a pointer)
  char internal[128];
};
struct NcclApi {
  bool loaded = false;
  ncclResult_t_ (*allReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  ncclResult_t_ (*allGather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t_) = nullptr;
  ncclResult_t_ (*getUniqueId)(void*) = nullptr;
  ncclResult_t_ (*commInitRank)(void**, int, NcclUid, int) = nullptr;
  ncclResult_t_ (*commDestroy)(void*) = nullptr;
  ncclResult_t_ (*commGetAsyncError)(void*, ncclResult_t_*) = nullptr;
};
// nccl.h enum values (stable ABI): ncclUint8 = 1... ncclUint64 = 5, ncclFloat32 = 7; ncclSum = 0, ncclMax = 2
constexpr int kNcclUint8 = 1, kNcclUint64 = 5, kNcclFloat32 = 7, kNcclSum = 0, kNcclMax = 2;

NcclApi& nccl() {
  static NcclApi api;
  if (!api.loaded) {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      api.allReduce = (decltype(api.allReduce))dlsym(h, "ncclAllReduce");
      api.allGather = (decltype(api.allGather))dlsym(h, "ncclAllGather");
      api.getErrorString = (decltype(api.getErrorString))dlsym(h, "ncclGetErrorString");
      api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
      api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
      api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
      api.commGetAsyncError = (decltype(api.commGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
      api.loaded = api.allReduce && api.allGather && api.getUniqueId && api.commInitRank;
    }
  }
  return api;
}

int round_up(int x, int m) { return (x + m - 1) / m * m; }
constexpr int kAttnRowUnits = 1024;  // (sequence, kv head, row block, split) partials of attn_rows
}  // namespace

// ----------------------------------------------------------------------------- context
struct RankState {
  int rank = 0;
  // weights (borrowed) + owned transposed W_down copies for the verify GEMM (K-major in ffn)
  const uint16_t *embed = nullptr, *final_norm = nullptr, *lm_head = nullptr;
  std::vector<const uint16_t*> attn_norm, w_qkv, w_o, ffn_norm, w_gate, w_up, w_down;
  std::vector<uint16_t*> w_down_t;
  // KV cache + verify staging
  uint16_t *k_cache = nullptr, *v_cache = nullptr, *stage_k = nullptr, *stage_v = nullptr;
  // activations (MAXM rows)
  float *resA = nullptr, *resB = nullptr, *dA = nullptr, *dF = nullptr, *qkv = nullptr, *logits = nullptr;
  float *qb = nullptr, *ob = nullptr;                      // post-RoPE q (verify), attention out (decode)
  // tensor-core B operands: fp32 activations as three bf16 terms, [3][MAXM][K] (split3, exact)
  uint16_t *xn3 = nullptr, *ob3 = nullptr, *mb3 = nullptr;
  // workspaces
  float *ffn_part = nullptr, *attn_part = nullptr, *gemm_part = nullptr;
  int* ffn_cnt = nullptr;
  unsigned long long* ffn_barrier = nullptr;
  unsigned* attn_bar = nullptr;  // split-group barriers (count, generation) of the attention kernels
  unsigned *attn_cnt = nullptr, *gemm_cnt = nullptr, *head_cnt = nullptr;
  // CSparse (csparse.cu): prompt statistic [L][Fr], the plan [L][k], a-export of a prefill chunk
  // [MAXM][Fr], compact weights [3][L][k][d] (gate, up, down rows of the kept neurons)
  float *cs_stats = nullptr, *cs_scratch = nullptr;
  float *tk_g = nullptr, *tk_a = nullptr;  // top-k FSparse (topk.cu): gate pre-activations, a [B][Fr]
  unsigned* tk_mask = nullptr;             // selected set [B][Fr/32 + 1] bits
  int32_t* cs_idx = nullptr;
  uint16_t* cs_w = nullptr;
  // fused peer all-reduce (TP > 1, peer_ar.cuh): the comm buffer peers map, the device array of every
  // rank's buffer as mapped here, the sync-point counter and the producer arrival counter
  char* par_buf = nullptr;
  char** par_peers = nullptr;
  unsigned long long* par_seq = nullptr;
  unsigned* par_done = nullptr;
};

struct sirius_ctx {
  sirius_config cfg;
  int nranks = 1;  // ranks run by this context (tp_size when emulating, else 1)
  bool emulated = false;
  float cs_keep = 0.f;   // CSparse keep fraction (sirius_csparse_enable); 0 = off
  int topk_k = 0;        // top-k FSparse: neurons kept per layer (sirius_topk_enable); 0 = off
  float samp_temp = 0.f; // sampling temperature of drafted / interleaved tokens (sirius_set_sampling); 0 = greedy
  unsigned long long samp_seed = 0ull;
  int cs_k = 0;          // neurons kept per layer (this rank's shard)
  bool cs_ready = false; // the plan of the last prefill is built
  bool stub_comm = false;  // SIRIUS_DEBUG_STUB_COMM: tp_size > 1 on one GPU with every collective skipped
                           // (one rank's compute, timing proxy only: results are rank-local partials)
  void* comm = nullptr;
  // fused peer all-reduce of the decode step (sirius_par_enable; SURVEY.md §8(e) phase 2)
  bool par_on = false;
  bool par_loopback = false;      // stub comm: every peer is this rank's own buffer (timing proxy)
  bool rows_par = false;          // the last forward_rows fused its all-reduces (its head norm consumes)
  unsigned long long par_timeout_ns = 10000000000ull;  // a peer missing this long -> SIRIUS_ERR_NCCL
  int par_slot_n = 0, par_key_n = 0;
  size_t par_bytes = 0;
  std::vector<void*> par_opened;  // peer buffers opened through CUDA IPC (closed by sirius_destroy)
  cudaStream_t stream = nullptr;
  int Hr = 0, KVr = 0, Fr = 0, Vr = 0, Nqkv = 0, G = 0, MAXM = 0;
  int num_sms = 148;
  size_t smem_optin = 0;
  size_t gemm_smem = 0;
  bool ffn_atomic = true;  // CATS FFN partials via float4 atomics, no grid barrier (SIRIUS_FFN_ATOMIC=0: deterministic)
  int ffn_split = 2;       // atomic-mode FFN CTAs per SM (SIRIUS_FFN_SPLIT; 2 measured best of 1-8)
  bool decode_rows = false;  // batched decode through the tensor-core row path (batch >= 4; SIRIUS_DECODE_ROWS)
  int32_t* dec_nacc = nullptr;
  int attn_stage_splits = 1;
  int accept_splits = 8;
  std::vector<RankState> ranks;
  float *thresholds = nullptr, *rope_cos = nullptr, *rope_sin = nullptr;
  int* err_dev = nullptr;
  int* err_host = nullptr;  // pinned mirror
  unsigned long long* amax = nullptr;
  RowStat *stats = nullptr, *stats_gather = nullptr;
  float** dA_ptrs = nullptr;  // device arrays of per-rank buffer pointers (emulated all-reduce)
  float** dF_ptrs = nullptr;
  int32_t* pre_start = nullptr;  // [batch] chunk start positions (prefill)
  int32_t* pre_start_host = nullptr;
  int32_t* scratch_tok = nullptr;
  int32_t* row_argmax = nullptr;  // [MAXM] full-model argmax of every row of the last verify
  TreeState* tree = nullptr;      // tree correction kernels (tree.cu): the last tree and its winning path
  bool tree_last = false;         // the last correction was a tree kernel (kv_rewrite commits its path)
  int last_gamma = 0;
  bool have_correct = false;
  bool prefilled = false;
  sirius_status sticky = SIRIUS_OK;
  unsigned long long launches = 0;  // kernels this context has launched (bench gpu_launches evidence)
  bool prof_on = false;             // per-kernel CUDA-event timing (bench roofline pass)
  struct ProfEv {
    int id;
    cudaEvent_t a, b;
  };
  std::vector<ProfEv> prof;
  size_t prof_used = 0;
  // profiling with CUDA graphs on: the events are captured into the graph as external event-record
  // nodes around the profiled launches; after each replay the call synchronises and accumulates
  bool capturing = false;
  std::vector<ProfEv> cap_evs;
  double prof_tot[16] = {0};
  int prof_cnt[16] = {0};
  // persistent decode step (decode_step.cu): TP 1 on supported shapes, opt-in (SIRIUS_STEP_KERNEL=1);
  // the default is the one-kernel-per-stage schedule (which TP > 1 needs between its all-reduces)
  bool use_step = false;
  int step_splits = 1;
  const uint16_t** step_w = nullptr;  // device [7][L]: attn_norm, w_qkv, w_o, ffn_norm, w_gate, w_up, w_down
  float *step_x = nullptr, *step_x1 = nullptr, *step_o = nullptr;
  unsigned long long* step_bar = nullptr;
  int trace_layer = -1;
  bool trace_ffn = false;  // debug: the trace buffer records the decode FFN of trace_layer                  // debug: attn_rows trace of this verify layer (sirius_debug_trace_verify)
  int step_tune = 1;                     // SIRIUS_STEP_TUNE (bit 0: evict-first weight loads)
  unsigned long long* trace = nullptr;  // debug: decode-step phase stamps (sirius_debug_trace)
  // CUDA graphs: every ABI call is captured once per distinct argument set and replayed
  bool use_graphs = true;
  cudaStream_t cap_stream = nullptr;
  struct GraphEntry {
    std::vector<uintptr_t> key;
    cudaGraphExec_t exec;
    unsigned long long kernels;
    std::vector<ProfEv> evs;  // profiled graph: (class, start, end) event-record nodes
  };
  std::vector<GraphEntry> graphs;
  std::vector<void*> allocations;
  std::string last_error = "ok";
};

namespace {

sirius_status fail(sirius_ctx* c, sirius_status s, const std::string& msg) {
  if (c) {
    c->last_error = msg;
    if (s == SIRIUS_ERR_CUDA || s == SIRIUS_ERR_NCCL) c->sticky = s;
  }
  return s;
}

#define CU(x)                                                                                        \
  do {                                                                                               \
    cudaError_t _e = (x);                                                                            \
    if (_e != cudaSuccess) return fail(c, SIRIUS_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(_e)); \
  } while (0)

#define LCU(x)     \
  do {             \
    ++c->launches; \
    CU(x);         \
  } while (0)

// ---- optional per-kernel timing: events recorded on the launch stream around selected launches
enum ProfId { P_QKV = 0, P_ATTN = 1, P_OPROJ = 2, P_FFN = 3, P_HEAD = 4, P_VERIFY = 5, P_REWRITE = 6, P_STEP = 7, P_NUM = 8 };
void prof_begin(sirius_ctx* c, int id) {
  if (!c->prof_on) return;
  if (c->capturing) {  // event-record nodes inside the graph being captured
    sirius_ctx::ProfEv e;
    e.id = id;
    cudaEventCreate(&e.a);
    cudaEventCreate(&e.b);
    cudaEventRecordWithFlags(e.a, c->stream, cudaEventRecordExternal);
    c->cap_evs.push_back(e);
    return;
  }
  if (c->prof_used == c->prof.size()) {
    sirius_ctx::ProfEv e;
    e.id = id;
    cudaEventCreate(&e.a);
    cudaEventCreate(&e.b);
    c->prof.push_back(e);
  }
  c->prof[c->prof_used].id = id;
  cudaEventRecord(c->prof[c->prof_used].a, c->stream);
}
void prof_end(sirius_ctx* c) {
  if (!c->prof_on) return;
  if (c->capturing) {
    cudaEventRecordWithFlags(c->cap_evs.back().b, c->stream, cudaEventRecordExternal);
    return;
  }
  cudaEventRecord(c->prof[c->prof_used].b, c->stream);
  ++c->prof_used;
}

template <class T>
sirius_status alloc(sirius_ctx* c, T** p, size_t count, bool zero = true) {
  void* q = nullptr;
  size_t bytes = count * sizeof(T);
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMalloc(&q, bytes);
  if (e != cudaSuccess) return fail(c, SIRIUS_ERR_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  if (zero) cudaMemset(q, 0, bytes);
  c->allocations.push_back(q);
  *p = reinterpret_cast<T*>(q);
  return SIRIUS_OK;
}

#define OK(x)                              \
  do {                                     \
    sirius_status _s = (x);                \
    if (_s != SIRIUS_OK) return _s;        \
  } while (0)

sirius_status check_sticky(sirius_ctx* c) {
  if (c->sticky != SIRIUS_OK) return c->sticky;
  // asynchronous NCCL failures (a peer died, a network/NVLink error) surface through the communicator,
  // not through the enqueueing call: poll it on every entry and make the failure sticky
  if (c->comm && !c->emulated && !c->stub_comm && nccl().commGetAsyncError) {
    ncclResult_t_ ar = 0;
    const ncclResult_t_ q = nccl().commGetAsyncError(c->comm, &ar);
    if (q != 0 || (ar != 0 && ar != 7 /* ncclInProgress */)) {
      const int code = q != 0 ? q : ar;
      return fail(c, SIRIUS_ERR_NCCL, std::string("NCCL asynchronous error: ") +
                                          (nccl().getErrorString ? nccl().getErrorString(code) : std::to_string(code)));
    }
  }
  if (*c->err_host != 0) {
    int e = *c->err_host;
    if (e & 8)
      return fail(c, SIRIUS_ERR_NCCL, "fused peer all-reduce: a rank did not arrive within 10 s");
    return fail(c, SIRIUS_ERR_CAPACITY,
                std::string("device-side capacity error (bits ") + std::to_string(e) +
                    "): 1 = decode pos outside [0, max_seq), 2 = verify/prefill row outside capacity, "
                    "4 = kv_rewrite n_rows/start outside capacity");
  }
  return SIRIUS_OK;
}

typedef std::vector<uintptr_t> GraphKey;

// Capture `enqueue` (which only enqueues work on c->stream) into a CUDA graph the first time a key
// is seen, then replay the instantiated graph: one launch per ABI call instead of ~130 kernels.
// Bypassed while per-kernel profiling is on.
// after a profiled graph's replay: wait for it and add its event pairs to the per-class totals
sirius_status prof_collect(sirius_ctx* c, const std::vector<sirius_ctx::ProfEv>& evs) {
  if (evs.empty()) return SIRIUS_OK;
  CU(cudaStreamSynchronize(c->stream));
  for (const auto& e : evs) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, e.a, e.b) == cudaSuccess) {
      c->prof_tot[e.id] += ms;
      c->prof_cnt[e.id] += 1;
    }
  }
  return SIRIUS_OK;
}

template <class F>
sirius_status run_graphed(sirius_ctx* c, const GraphKey& key0, F enqueue) {
  if (!c->use_graphs) return enqueue();
  GraphKey key = key0;
  key.push_back(c->prof_on ? 1u : 0u);  // profiled graphs carry event-record nodes
  key.push_back(c->par_on ? 1u : 0u);   // the decode step with the fused peer all-reduce
  for (auto& g : c->graphs)
    if (g.key == key) {
      c->launches += g.kernels;
      CU(cudaGraphLaunch(g.exec, c->stream));
      return prof_collect(c, g.evs);
    }
  // capture on a private stream (the caller's stream may be the legacy default stream, which cannot
  // be captured); the instantiated graph is then launched on the caller's stream
  if (!c->cap_stream) CU(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
  const unsigned long long before = c->launches;
  cudaStream_t user = c->stream;
  CU(cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeRelaxed));
  c->stream = c->cap_stream;
  c->capturing = true;
  c->cap_evs.clear();
  sirius_status s = enqueue();
  c->capturing = false;
  c->stream = user;
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamEndCapture(c->cap_stream, &graph);
  cudaGraphExec_t exec = nullptr;
  if (s == SIRIUS_OK && e == cudaSuccess) e = cudaGraphInstantiate(&exec, graph, 0);
  if (graph) cudaGraphDestroy(graph);
  if (s != SIRIUS_OK || e != cudaSuccess || !exec) {
    // not capturable on this driver / configuration: fall back to direct launches for good
    cudaGetLastError();
    c->use_graphs = false;
    c->sticky = SIRIUS_OK;
    c->launches = before;
    for (auto& e : c->cap_evs) {
      cudaEventDestroy(e.a);
      cudaEventDestroy(e.b);
    }
    c->cap_evs.clear();
    return enqueue();
  }
  if (c->graphs.size() >= 256) {
    cudaGraphExecDestroy(c->graphs.front().exec);
    for (auto& e : c->graphs.front().evs) {
      cudaEventDestroy(e.a);
      cudaEventDestroy(e.b);
    }
    c->graphs.erase(c->graphs.begin());
  }
  c->graphs.push_back({key, exec, c->launches - before, c->cap_evs});
  c->cap_evs.clear();
  CU(cudaGraphLaunch(exec, c->stream));
  return prof_collect(c, c->graphs.back().evs);
}

// enqueue a copy of the device error word into the pinned host mirror (read by the next call)
void mirror_err(sirius_ctx* c) { cudaMemcpyAsync(c->err_host, c->err_dev, sizeof(int), cudaMemcpyDeviceToHost, c->stream); }

sirius_status allreduce(sirius_ctx* c, float* RankState::*buf, float** ptrs_dev, size_t rows) {
  const size_t n = rows * c->cfg.d_model;
  if (c->nranks > 1) {
    LCU(launch::sum_ranks(ptrs_dev, c->nranks, rows, c->cfg.d_model, c->cfg.d_model, c->stream));
  } else if (c->cfg.tp_size > 1 && !c->stub_comm) {
    NcclApi& api = nccl();
    float* p = c->ranks[0].*buf;
    int r = api.allReduce(p, p, n, kNcclFloat32, kNcclSum, c->comm, c->stream);
    if (r != 0) return fail(c, SIRIUS_ERR_NCCL, std::string("ncclAllReduce: ") + api.getErrorString(r));
  }
  return SIRIUS_OK;
}

sirius_status run_gemv(sirius_ctx* c, const GemvArgs& a, int B);

// the rank's fused peer all-reduce descriptor (sirius_par_enable)
PeerAr par_of(const sirius_ctx* c, const RankState& R) {
  PeerAr p = {};
  p.world = c->cfg.tp_size;
  p.rank = R.rank;
  p.fused = c->emulated ? 0 : 1;  // emulated ranks run one after another: none may wait (par_reduce)
  p.loopback = c->par_loopback ? 1 : 0;
  p.slot_n = c->par_slot_n;
  p.key_n = c->par_key_n;
  p.scale = c->par_loopback ? 1.0f / (float)c->cfg.tp_size : 1.0f;
  p.peers = R.par_peers;
  p.self = R.par_buf;
  p.seq = R.par_seq;
  p.done = R.par_done;
  p.err = c->err_dev;
  p.timeout_ns = c->par_timeout_ns;
  return p;
}
// a norm_rows consumer of the last fused sync point (forward_rows with GemmArgs.par producers)
void par_consume_rows(const sirius_ctx* c, const RankState& R, NormRowsArgs& na) {
  na.delta = nullptr;
  na.par_consume = 1;
  na.par = par_of(c, R);
}

// the all-reduce of the partials buf [B, d] of every rank of this context: fused into the producer
// (nothing to launch), the emulated reduction (every emulated rank has pushed), or NCCL / in-order sums
sirius_status par_or_allreduce(sirius_ctx* c, float* RankState::*buf, float** ptrs_dev, int B, bool par) {
  if (!par) return allreduce(c, buf, ptrs_dev, B);
  if (c->emulated)
    for (auto& R : c->ranks) LCU(launch::par_reduce(par_of(c, R), R.*buf, B * c->cfg.d_model, 0, nullptr, c->stream));
  return SIRIUS_OK;
}

// ---- the decode CATS FFN of layer l (S4-S6) on residual rows base (+ delta): out = the FFN's
// contribution to the residual (accumulated into out, which the O-proj GEMV zeroed, in atomic mode)
sirius_status launch_decode_ffn(sirius_ctx* c, RankState& R, int l, const float* base, const float* delta,
                                float* res_out, float* out, bool dense, int32_t* n_active_out, int n_active_stride,
                                float* gate_out, long long gate_stride, bool csparse = false, bool topk = false,
                                bool par_decode = false) {
  const sirius_config& cf = c->cfg;
  FfnArgs f = {};
  if (topk) {  // gate GEMV -> exact top-k selection (topk.cu) -> the FFN kernel in precomputed-gate mode
    GemvArgs gv = {};
    gv.pro.mode = IN_RESID;
    gv.pro.base = base;
    gv.pro.delta = delta;
    gv.pro.norm_w = R.ffn_norm[l];
    gv.pro.eps = cf.rms_eps;
    gv.W = R.w_gate[l];
    gv.rows = c->Fr;
    gv.K = cf.d_model;
    gv.epi = EPI_STORE;
    gv.out = R.tk_g;
    gv.ldo = c->Fr;
    OK(run_gemv(c, gv, cf.batch));
    const long long mw = c->Fr / 32 + 1;
    LCU(launch::topk_select(R.tk_g, c->Fr, c->Fr, c->topk_k, R.tk_a, c->Fr, R.tk_mask, mw, cf.batch, c->stream));
    f.a_in = R.tk_a;
    f.mask_in = R.tk_mask;
    f.a_ld = c->Fr;
    f.m_ld = mw;
  }
  f.pro.mode = IN_RESID;
  f.pro.base = base;
  f.pro.delta = delta;
  f.pro.norm_w = R.ffn_norm[l];
  f.pro.eps = cf.rms_eps;
  f.pro.res_out = res_out;
  f.w_gate = R.w_gate[l];
  f.w_up = R.w_up[l];
  f.w_down = R.w_down[l];
  f.F = c->Fr;
  if (csparse) {  // the prompt's fixed neuron set: the dense FFN over the compact [k, d] matrices
    const size_t per = (size_t)c->cs_k * cf.d_model, L = cf.n_layers;
    f.w_gate = R.cs_w + (0 * L + l) * per;
    f.w_up = R.cs_w + (1 * L + l) * per;
    f.w_down = R.cs_w + (2 * L + l) * per;
    f.F = c->cs_k;
    dense = true;
  }
  f.d = cf.d_model;
  f.threshold = c->thresholds + l;
  f.dense = dense ? 1 : 0;
  f.part = R.ffn_part;
  f.part_cnt = R.ffn_cnt;
  f.barrier = R.ffn_barrier;
  f.out = out;
  f.n_active_out = n_active_out;
  f.n_active_stride = n_active_stride;
  f.atomic_out = c->ffn_atomic ? 1 : 0;
  if (c->par_on && par_decode) f.par = par_of(c, R);  // fused peer all-reduce of the FFN partial
  f.trace = (c->trace && l == c->trace_layer && c->trace_ffn) ? c->trace : nullptr;
  f.gate_out = gate_out;
  f.gate_stride = gate_stride;
  const int grid = c->ffn_atomic ? std::min((f.F + 7) / 8, c->ffn_split * c->num_sms) : launch::ffn_grid(f.F, c->num_sms);
  if (grid < 1) return fail(c, SIRIUS_ERR_UNSUPPORTED, "FFN width not supported by the decode FFN kernel");
  LCU(launch::ffn(f, cf.batch, grid, c->stream));
  return SIRIUS_OK;
}

// ---- one GEMV (decode) launch
sirius_status run_gemv(sirius_ctx* c, const GemvArgs& a, int B) {
  LCU(launch::gemv(a, B, launch::gemv_grid(a.rows, c->num_sms), c->stream));
  return SIRIUS_OK;
}

struct GemmMask {  // CATS mask of the dual (SwiGLU) GEMM in the batched sparse decode
  const float* thr = nullptr;
  int* n_active = nullptr;
  int n_active_stride = 0;
  float* gate_out = nullptr;
  long long gate_stride = 0;
};

// out: fp32 [M, ldc] (single) or, dual (wb != NULL), the SwiGLU product's three bf16 term planes
// (plane stride MAXM * ldc).  x: the activation's three term planes ([3 * MAXM, K] map).

sirius_status run_gemm(sirius_ctx* c, RankState& R, const void* wa, const void* wb, const void* x, int N, int K,
                       int M, void* out, int ldc, unsigned long long* trace = nullptr, const GemmMask* mask = nullptr,
                       bool par = false) {
  GemmArgs g = {};
  g.trace = trace;
  if (par) {  // fused peer all-reduce of the fp32 output (forward_rows: one launch, M <= 128, ldc == d)
    g.par = par_of(c, R);
  }
  if (mask) {
    g.thr = mask->thr;
    g.n_active = mask->n_active;
    g.n_active_stride = mask->n_active_stride;
    g.gate_out = mask->gate_out;
    g.gate_stride = mask->gate_stride;
  }
  g.N = N;
  g.K = K;
  g.n_tiles = (N + 127) / 128;
  g.kb = (K + 63) / 64;
  g.out_plane = (size_t)c->MAXM * ldc;
  g.ldc = ldc;
  g.nterms = 3;
  g.plane_rows = c->MAXM;
  g.part = R.gemm_part;
  g.counters = R.gemm_cnt;
  // more than 128 token rows (prefill chunks, batched verify): launches of <= 128 rows, so that the
  // three activation terms of >= 2 pipeline stages fit in shared memory next to the weight boxes
  const int chunk = M > 128 ? 128 : M;
  for (int r0 = 0; r0 < M; r0 += chunk) {
    const int Mc = M - r0 < chunk ? M - r0 : chunk;
    GemmArgs gc = g;
    gc.M = Mc;
    gc.row0 = r0;
    gc.out = wb ? (void*)((uint16_t*)out + (size_t)r0 * ldc) : (void*)((float*)out + (size_t)r0 * ldc);
    if (gc.n_active) gc.n_active += (size_t)r0 * gc.n_active_stride;
    if (gc.gate_out) gc.gate_out += (size_t)r0 * gc.gate_stride;
    if (r0) gc.trace = nullptr;
    const int MP = round_up(Mc, 16);
    LCU(launch::gemm(wa, wb, x, gc, MP, c->num_sms,
                     MP <= 64 ? c->gemm_smem : c->smem_optin, c->stream));
  }
  return SIRIUS_OK;
}

// ---- the dense / verify / prefill forward over M token rows (chunk).  Rows are ordered
// (sequence, i); rows_per_seq rows per sequence, sequences b_base .. b_base + nseq - 1.
//   ROWS_PREFILL: K/V -> cache at start[b] + i, attention reads the cache only (one sequence per call);
//   ROWS_VERIFY : K/V -> staging rows i, attention reads cache [0, start[b]) + staging [0, i];
//   ROWS_DECODE : batched decode, one row per sequence of the whole batch (b_base 0, nseq = batch),
//                 K/V -> cache at start[b] through the decode-attention item kernel.
// sparse: CATS mask on the FFN (batched sparse decode, rows_per_seq = 1); n_active_out [rows, L] and
// gate_act_out [rows, L, ffn] (emulated TP: rank shards concatenated) optional.
enum RowsMode { ROWS_PREFILL = 0, ROWS_VERIFY = 1, ROWS_DECODE = 2 };
// Tree rows (tree.cu, batch 1, ROWS_VERIFY): stage_base = staging row of the call's row 0, row_off [rows] =
// each row's position offset from start, tree_vis = the ancestor masks (attn_rows).
sirius_status forward_rows(sirius_ctx* c, const int32_t* tokens, const int32_t* start, int b_base, int nseq,
                           int rows_per_seq, RowsMode mode, bool sparse = false, int32_t* n_active_out = nullptr,
                           float* gate_act_out = nullptr, int stage_base = 0, const int32_t* row_off = nullptr,
                           const unsigned long long* tree_vis = nullptr) {
  const bool to_cache = mode != ROWS_VERIFY;
  const sirius_config& cf = c->cfg;
  const int M = nseq * rows_per_seq, d = cf.d_model, hd = cf.head_dim, L = cf.n_layers;
  // TP > 1 with sirius_par_enable: the O-proj / down-proj GEMMs push their outputs to every rank in the
  // epilogue and the next norm_rows sums them (no collective launch) — verify and batched-row forwards
  // (one GEMM launch of <= 128 rows); the prefill keeps the NCCL all-reduce
  const bool par = c->par_on && cf.tp_size > 1 && mode != ROWS_PREFILL && M <= 128 &&
                   (size_t)M * d <= (size_t)c->par_slot_n;
  c->rows_par = par;
  for (int l = 0; l < L; ++l) {
    for (auto& R : c->ranks) {
      NormRowsArgs na = {};
      if (l == 0) {
        na.tokens = tokens;
        na.embed = R.embed;
      } else {
        na.base = R.resB;
        na.delta = R.dF;
        if (par) par_consume_rows(c, R, na);
      }
      na.vocab = cf.vocab;
      na.d = d;
      na.norm_w = R.attn_norm[l];
      na.eps = cf.rms_eps;
      na.res_out = R.resA;
      na.out3 = R.xn3;
      na.plane = (size_t)c->MAXM * d;
      LCU(launch::norm_rows(na, M, c->stream));
      unsigned long long* gtr = (!to_cache && l == c->trace_layer && c->trace) ? c->trace + 8 * 1024 : nullptr;
      OK(run_gemm(c, R, R.w_qkv[l], nullptr, R.xn3, c->Nqkv, d, M, R.qkv, c->Nqkv, gtr));
      const size_t kv_layer = (size_t)cf.batch * c->KVr * cf.max_seq * hd;
      const size_t st_layer = (size_t)cf.batch * c->KVr * cf.max_gamma * hd;
      if (mode == ROWS_DECODE) {
        // one query row per sequence (batched decode): the decode-attention item kernel does RoPE,
        // the K/V append at pos and split-K attention, writing the O-proj operand as a hi/lo pair
        StepArgs sa = {};
        sa.d = d;
        sa.Hr = c->Hr;
        sa.KVr = c->KVr;
        sa.hd = hd;
        sa.max_seq = cf.max_seq;
        sa.splits = c->attn_stage_splits;
        sa.attn_scale = 1.0f / sqrtf((float)hd);
        sa.pos = start;
        sa.qkv = R.qkv;
        sa.o3 = R.ob3;
        sa.o3_plane = (size_t)c->MAXM * c->Hr * hd;
        sa.k_cache = R.k_cache;
        sa.v_cache = R.v_cache;
        sa.kv_layer = kv_layer;
        sa.rope_cos = c->rope_cos;
        sa.rope_sin = c->rope_sin;
        sa.attn_part = R.attn_part;
        sa.group_bar = R.attn_bar;
        sa.err = c->err_dev;
        LCU(launch::attn_stage(sa, l, cf.batch, c->stream));
        OK(run_gemm(c, R, R.w_o[l], nullptr, R.ob3, d, c->Hr * hd, M, R.dA, d, nullptr, nullptr, par));
        continue;
      }
      RopeStoreArgs ra = {};
      ra.qkv = R.qkv;
      ra.start = start;
      ra.b_base = b_base;
      ra.rows_per_seq = rows_per_seq;
      ra.rope_cos = c->rope_cos;
      ra.rope_sin = c->rope_sin;
      ra.Hr = c->Hr;
      ra.KVr = c->KVr;
      ra.hd = hd;
      ra.max_seq = cf.max_seq;
      ra.max_gamma = cf.max_gamma;
      ra.to_cache = to_cache ? 1 : 0;
      ra.stage_base = stage_base;
      ra.row_off = row_off;
      ra.q_out = R.qb;
      ra.k_dst = to_cache ? R.k_cache + l * kv_layer : R.stage_k + l * st_layer;
      ra.v_dst = to_cache ? R.v_cache + l * kv_layer : R.stage_v + l * st_layer;
      ra.err = c->err_dev;
      LCU(launch::rope_store(ra, M, c->stream));
      AttnRowsArgs aa = {};
      aa.q = R.qb;
      aa.start = start;
      aa.b_base = b_base;
      aa.rows_per_seq = rows_per_seq;
      aa.G = c->G;
      aa.Hr = c->Hr;
      aa.KVr = c->KVr;
      aa.max_seq = cf.max_seq;
      aa.k_cache = R.k_cache + l * kv_layer;
      aa.v_cache = R.v_cache + l * kv_layer;
      aa.k_fresh = R.stage_k + l * st_layer;
      aa.v_fresh = R.stage_v + l * st_layer;
      aa.fresh_stride = cf.max_gamma;
      aa.fresh_in_cache = to_cache ? 1 : 0;
      aa.stage_base = stage_base;
      aa.tree_vis = tree_vis;
      aa.part = R.attn_part;
      aa.counters = R.attn_cnt;
      aa.group_bar = R.attn_bar;
      aa.out3 = R.ob3;
      aa.plane = (size_t)c->MAXM * c->Hr * hd;
      aa.trace = (!to_cache && l == c->trace_layer) ? c->trace : nullptr;
      const int row_blocks = (rows_per_seq * c->G + 63) / 64;
      int splits = launch::attn_rows_splits(nseq, c->KVr, row_blocks, cf.max_seq, c->num_sms);
      while (splits > 1 && nseq * c->KVr * row_blocks * splits > kAttnRowUnits) --splits;  // workspace bound
      LCU(launch::attn_rows(aa, nseq, hd, splits, row_blocks, c->stream));
      OK(run_gemm(c, R, R.w_o[l], nullptr, R.ob3, d, c->Hr * hd, M, R.dA, d, gtr ? gtr + 8 * 1024 : nullptr, nullptr,
                  par));
    }
    if (!par) OK(allreduce(c, &RankState::dA, c->dA_ptrs, M));
    for (auto& R : c->ranks) {
      NormRowsArgs na = {};
      na.base = R.resA;
      na.delta = R.dA;
      if (par) par_consume_rows(c, R, na);
      na.vocab = cf.vocab;
      na.d = d;
      na.norm_w = R.ffn_norm[l];
      na.eps = cf.rms_eps;
      na.res_out = R.resB;
      na.out3 = R.xn3;
      na.plane = (size_t)c->MAXM * d;
      LCU(launch::norm_rows(na, M, c->stream));
      unsigned long long* gtr2 = (!to_cache && l == c->trace_layer && c->trace) ? c->trace + 3 * 8 * 1024 : nullptr;
      GemmMask mk;
      if (sparse) mk.thr = c->thresholds + l;
      if (n_active_out) {
        mk.n_active = n_active_out + l;
        mk.n_active_stride = L;
      }
      if (gate_act_out) {
        const int Ff = c->emulated ? cf.ffn_dim : c->Fr;
        mk.gate_out = gate_act_out + (size_t)l * Ff + (c->emulated ? (size_t)R.rank * c->Fr : 0);
        mk.gate_stride = (long long)L * Ff;
      }
      const bool cs_stats = mode == ROWS_PREFILL && c->cs_keep > 0.f;  // CSparse statistic of the prompt
      if (cs_stats) {
        mk.gate_out = R.cs_scratch;
        mk.gate_stride = c->Fr;
      }
      OK(run_gemm(c, R, R.w_gate[l], R.w_up[l], R.xn3, c->Fr, d, M, R.mb3, c->Fr, gtr2, &mk));
      if (cs_stats) LCU(launch::csparse_colsum(R.cs_scratch, M, c->Fr, c->Fr, R.cs_stats + (size_t)l * c->Fr, c->stream));
      OK(run_gemm(c, R, R.w_down_t[l], nullptr, R.mb3, d, c->Fr, M, R.dF, d, gtr2 ? gtr2 + 8 * 1024 : nullptr,
                  nullptr, par));
    }
    if (!par) OK(allreduce(c, &RankState::dF, c->dF_ptrs, M));
  }
  return SIRIUS_OK;
}

}  // namespace

// ============================================================================= C ABI
extern "C" {

const char* sirius_version(void) { return "libsirius sm_100a (tcgen05 verify GEMM, bulk-copy GEMV, CATS FFN)"; }

const char* sirius_last_error(const sirius_ctx* c) { return c ? c->last_error.c_str() : "null context"; }

sirius_status sirius_init(const sirius_config* cfgp, const sirius_weights* w, const float* cats_threshold,
                          void* nccl_comm, void* stream, sirius_ctx** out) {
  if (!cfgp || !w || !cats_threshold || !out) return SIRIUS_ERR_INVALID_ARG;
  *out = nullptr;
  const sirius_config cf = *cfgp;
  if (cf.vocab <= 0 || cf.d_model <= 0 || cf.n_layers <= 0 || cf.n_heads <= 0 || cf.n_kv_heads <= 0 ||
      cf.head_dim <= 0 || cf.ffn_dim <= 0 || cf.batch <= 0 || cf.max_seq <= 0 || cf.max_gamma <= 0 ||
      cf.tp_size <= 0 || cf.n_heads % cf.n_kv_heads || cf.rms_eps <= 0.f || cf.rope_theta <= 0.f)
    return SIRIUS_ERR_INVALID_ARG;
  if (cf.tp_rank < 0 || cf.tp_rank >= cf.tp_size) return SIRIUS_ERR_INVALID_ARG;
  if (cf.n_heads % cf.tp_size || cf.n_kv_heads % cf.tp_size || cf.ffn_dim % cf.tp_size || cf.vocab % cf.tp_size)
    return SIRIUS_ERR_UNSUPPORTED;
  if (cf.head_dim != 64 && cf.head_dim != 128) return SIRIUS_ERR_UNSUPPORTED;
  if (cf.d_model % 256 || ((cf.n_heads / cf.tp_size) * cf.head_dim) % 64 || (cf.ffn_dim / cf.tp_size) % 8)
    return SIRIUS_ERR_UNSUPPORTED;
  if (cf.max_gamma > 64 || (long)cf.batch * cf.max_gamma > 1024) return SIRIUS_ERR_UNSUPPORTED;
  if (cf.batch != 1 && cf.batch != 2 && cf.batch != 4 && cf.batch != 8 && cf.batch != 16 && cf.batch != 32)
    return SIRIUS_ERR_UNSUPPORTED;
  for (int l = 0; l < cf.n_layers; ++l)
    if (!(cats_threshold[l] >= 0.f)) return SIRIUS_ERR_INVALID_ARG;
  const bool emulate = cf.tp_size > 1 && nccl_comm == nullptr;
  if (cf.tp_size > 1 && !emulate && !nccl().loaded) return SIRIUS_ERR_NCCL;

  sirius_ctx* c = new sirius_ctx();
  c->cfg = cf;
  c->stream = (cudaStream_t)stream;
  c->comm = nccl_comm;
  c->emulated = emulate;
  if (const char* e = getenv("SIRIUS_DEBUG_STUB_COMM")) c->stub_comm = !emulate && cf.tp_size > 1 && atoi(e) != 0;
  c->nranks = emulate ? cf.tp_size : 1;
  c->Hr = cf.n_heads / cf.tp_size;
  c->KVr = cf.n_kv_heads / cf.tp_size;
  c->Fr = cf.ffn_dim / cf.tp_size;
  c->Vr = cf.vocab / cf.tp_size;
  c->G = cf.n_heads / cf.n_kv_heads;
  c->Nqkv = (c->Hr + 2 * c->KVr) * cf.head_dim;
  // activation rows: a verify of batch x gamma rows (GEMM launches chunk them by 128), at least 256
  c->MAXM = std::max(256, round_up(cf.batch * cf.max_gamma, 16));
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, dev);
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  c->smem_optin = (size_t)optin - 1024;  // keep room for static shared memory
  c->gemm_smem = c->smem_optin;            // verify GEMM pipeline budget (SIRIUS_GEMM_SMEM_KB caps it)
  if (const char* e = getenv("SIRIUS_GEMM_SMEM_KB")) c->gemm_smem = std::min(c->smem_optin, (size_t)atoi(e) * 1024);
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (major != 10) {
    sirius_status s = fail(c, SIRIUS_ERR_UNSUPPORTED, "libsirius is built for sm_100a (B200) only");
    delete c;
    return s;
  }
  if (!launch::attn_stage_supported(cf.head_dim, c->G)) {  // decode attention instantiations (decode_step.cu)
    sirius_status s = fail(c, SIRIUS_ERR_UNSUPPORTED, "decode attention: (head_dim, GQA group) not compiled");
    delete c;
    return s;
  }
  if (const char* e = getenv("SIRIUS_FFN_ATOMIC")) c->ffn_atomic = atoi(e) != 0;
  // measured (profiles/batch_r02): batch 4 dense 5.81 ms per step on the per-stage CUDA-core kernels vs
  // 4.30 on the row path; batch 2 3.62 vs 4.10 — the row path from batch 4 on
  c->decode_rows = cf.batch >= 4;
  if (const char* e = getenv("SIRIUS_DECODE_ROWS")) c->decode_rows = atoi(e) != 0;
  if (cf.batch > 8) c->decode_rows = true;  // the per-stage decode kernels are instantiated up to batch 8
  if (const char* e = getenv("SIRIUS_FFN_SPLIT")) c->ffn_split = std::max(1, atoi(e));
  c->attn_stage_splits = launch::decode_step_splits(cf.batch, c->KVr, c->num_sms);
  if (const char* e = getenv("SIRIUS_ATTN_SPLITS")) c->attn_stage_splits = std::max(1, std::min(64, atoi(e)));
  // verify / prefill chain with programmatic dependent launch (SIRIUS_VERIFY_PDL=0 disables)
  if (const char* e = getenv("SIRIUS_VERIFY_PDL")) launch::g_chain_pdl = atoi(e) != 0;
  if (const char* e = getenv("SIRIUS_DECODE_PDL")) launch::g_decode_pdl = atoi(e) != 0;
  if (const char* e = getenv("SIRIUS_PAR_TIMEOUT_MS")) c->par_timeout_ns = (unsigned long long)std::max(1, atoi(e)) * 1000000ull;
  if (const char* e = getenv("SIRIUS_GEMM_KBOX")) launch::g_gemm_kbox = atoi(e);
  if (const char* e = getenv("SIRIUS_GEMM_COARSE")) launch::g_gemm_coarse = atoi(e);
  auto cleanup_fail = [&](sirius_status s) {
    sirius_destroy(c);
    return s;
  };
  const int L = cf.n_layers, d = cf.d_model, hd = cf.head_dim, B = cf.batch;
  // shared buffers
  if (alloc(c, &c->thresholds, L) || alloc(c, &c->rope_cos, (size_t)cf.max_seq * hd / 2) ||
      alloc(c, &c->rope_sin, (size_t)cf.max_seq * hd / 2) || alloc(c, &c->err_dev, 4) || alloc(c, &c->amax, 64) ||
      alloc(c, &c->stats, (size_t)c->nranks * c->MAXM * c->accept_splits) ||
      alloc(c, &c->stats_gather, (size_t)cf.tp_size * c->MAXM * c->accept_splits) ||
      alloc(c, &c->dA_ptrs, 64) || alloc(c, &c->dF_ptrs, 64) || alloc(c, &c->pre_start, B) ||
      alloc(c, &c->dec_nacc, B) || alloc(c, &c->row_argmax, c->MAXM) ||
      alloc(c, &c->scratch_tok, 64) || alloc(c, &c->tree, 1))
    return cleanup_fail(SIRIUS_ERR_CUDA);
  if (cudaHostAlloc(&c->err_host, 64, cudaHostAllocDefault) != cudaSuccess ||
      cudaHostAlloc(&c->pre_start_host, sizeof(int32_t) * B, cudaHostAllocDefault) != cudaSuccess)
    return cleanup_fail(SIRIUS_ERR_CUDA);
  *c->err_host = 0;
  cudaMemcpy(c->thresholds, cats_threshold, sizeof(float) * L, cudaMemcpyHostToDevice);
  {  // RoPE table: fp64 then rounded to fp32 (reading D16); rotate-half pairs (i, i + hd/2)
    std::vector<float> cs((size_t)cf.max_seq * hd / 2), sn((size_t)cf.max_seq * hd / 2);
    for (int p = 0; p < cf.max_seq; ++p)
      for (int i = 0; i < hd / 2; ++i) {
        const double inv = std::pow((double)cf.rope_theta, -2.0 * i / hd);
        const double ang = (double)p * inv;
        cs[(size_t)p * hd / 2 + i] = (float)std::cos(ang);
        sn[(size_t)p * hd / 2 + i] = (float)std::sin(ang);
      }
    cudaMemcpy(c->rope_cos, cs.data(), sizeof(float) * cs.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(c->rope_sin, sn.data(), sizeof(float) * sn.size(), cudaMemcpyHostToDevice);
  }
  c->ranks.resize(c->nranks);
  std::vector<float*> dA_h, dF_h;
  const int ffn_grid = launch::ffn_grid(c->Fr, c->num_sms);
  if (ffn_grid < 0) return cleanup_fail(SIRIUS_ERR_UNSUPPORTED);
  for (int r = 0; r < c->nranks; ++r) {
    RankState& R = c->ranks[r];
    const sirius_weights& W = w[emulate ? r : 0];
    R.rank = emulate ? r : cf.tp_rank;
    if (!W.embed || !W.final_norm || !W.lm_head || !W.attn_norm || !W.w_qkv || !W.w_o || !W.ffn_norm || !W.w_gate ||
        !W.w_up || !W.w_down)
      return cleanup_fail(SIRIUS_ERR_INVALID_ARG);
    R.embed = (const uint16_t*)W.embed;
    R.final_norm = (const uint16_t*)W.final_norm;
    R.lm_head = (const uint16_t*)W.lm_head;
    for (int l = 0; l < L; ++l) {
      const void* ptrs[7] = {W.attn_norm[l], W.w_qkv[l], W.w_o[l], W.ffn_norm[l], W.w_gate[l], W.w_up[l], W.w_down[l]};
      for (const void* p : ptrs)
        if (!p || ((uintptr_t)p & 15)) return cleanup_fail(SIRIUS_ERR_INVALID_ARG);
      R.attn_norm.push_back((const uint16_t*)W.attn_norm[l]);
      R.w_qkv.push_back((const uint16_t*)W.w_qkv[l]);
      R.w_o.push_back((const uint16_t*)W.w_o[l]);
      R.ffn_norm.push_back((const uint16_t*)W.ffn_norm[l]);
      R.w_gate.push_back((const uint16_t*)W.w_gate[l]);
      R.w_up.push_back((const uint16_t*)W.w_up[l]);
      R.w_down.push_back((const uint16_t*)W.w_down[l]);
    }
    const size_t kv = (size_t)L * B * c->KVr * cf.max_seq * hd;
    const size_t stg = (size_t)L * B * c->KVr * cf.max_gamma * hd;
    const int M = c->MAXM;
    const int row_blocks_max = (cf.max_gamma * c->G + 63) / 64 + (M * c->G + 63) / 64;
    if (alloc(c, &R.k_cache, kv) || alloc(c, &R.v_cache, kv) || alloc(c, &R.stage_k, stg) ||
        alloc(c, &R.stage_v, stg) || alloc(c, &R.resA, (size_t)M * d) || alloc(c, &R.resB, (size_t)M * d) ||
        alloc(c, &R.dA, (size_t)M * d) || alloc(c, &R.dF, (size_t)M * d) || alloc(c, &R.qkv, (size_t)M * c->Nqkv) ||
        alloc(c, &R.logits, (size_t)M * c->Vr) || alloc(c, &R.xn3, (size_t)3 * M * d) ||
        alloc(c, &R.qb, (size_t)M * c->Hr * hd) || alloc(c, &R.ob, (size_t)M * c->Hr * hd) ||
        alloc(c, &R.ob3, (size_t)3 * M * c->Hr * hd) || alloc(c, &R.mb3, (size_t)3 * M * c->Fr) || alloc(c, &R.ffn_part, (size_t)c->num_sms * std::max(4, B) * d) ||
        alloc(c, &R.ffn_cnt, (size_t)c->num_sms * std::max(4, B)) || alloc(c, &R.ffn_barrier, 8) ||
        alloc(c, &R.attn_part, (size_t)kAttnRowUnits * 64 * (hd + 2) + (size_t)B * c->KVr * 64 * 8 * (hd + 2)) ||
        alloc(c, &R.attn_cnt, (size_t)(B + 1) * c->KVr * (row_blocks_max + 1) * 4 + 4096) || alloc(c, &R.attn_bar, 8192) ||
        alloc(c, &R.gemm_part, launch::gemm_workspace_bytes(c->num_sms) / sizeof(float)) ||
        alloc(c, &R.gemm_cnt, (size_t)(c->Vr / 128 + 1024)) || alloc(c, &R.head_cnt, 16))
      return cleanup_fail(SIRIUS_ERR_CUDA);
    dA_h.push_back(R.dA);
    dF_h.push_back(R.dF);
    if (cf.tp_size > 1) {  // fused peer all-reduce buffers (zeroed: flags 0 < every sequence number)
      c->par_slot_n = round_up(std::max(B, std::min(B * cf.max_gamma, 128)) * d, 4);  // decode / verify rows
      c->par_key_n = 8;
      c->par_bytes = (size_t)2 * cf.tp_size * ((size_t)c->par_slot_n * 4 + (size_t)c->par_key_n * 8 + 8);
      if (alloc(c, &R.par_buf, c->par_bytes) || alloc(c, &R.par_peers, 8) || alloc(c, &R.par_seq, 1) ||
          alloc(c, &R.par_done, 1))
        return cleanup_fail(SIRIUS_ERR_CUDA);
    }
    // transposed W_down ([d, F/tp], K-major in the neuron dim) for the verify down-projection GEMM
    R.w_down_t.resize(L);
    for (int l = 0; l < L; ++l) {
      if (alloc(c, &R.w_down_t[l], (size_t)d * c->Fr, false)) return cleanup_fail(SIRIUS_ERR_CUDA);
      if (launch::transpose_bf16(R.w_down[l], R.w_down_t[l], c->Fr, d, c->stream) != cudaSuccess)
        return cleanup_fail(SIRIUS_ERR_CUDA);
    }
  }
  cudaMemcpy(c->dA_ptrs, dA_h.data(), sizeof(float*) * dA_h.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(c->dF_ptrs, dF_h.data(), sizeof(float*) * dF_h.size(), cudaMemcpyHostToDevice);
  // persistent decode step (TP 1)
  if (!emulate && cf.tp_size == 1 && cf.batch <= 4 &&
      launch::decode_step_supported(d, cf.n_heads, cf.n_kv_heads, hd, cf.ffn_dim, c->num_sms)) {
    // opt-in: measured at parity / slightly slower than the per-stage kernels on the 8B step
    // (2.90-2.93 vs 2.86-2.89 ms), so the per-stage schedule stays the default
    const char* e = getenv("SIRIUS_STEP_KERNEL");
    c->use_step = e && atoi(e) != 0;
    if (const char* t = getenv("SIRIUS_STEP_TUNE")) c->step_tune = atoi(t);
  }
  if (c->use_step) {
    RankState& R = c->ranks[0];
    if (alloc(c, &c->step_w, (size_t)7 * L) || alloc(c, &c->step_x, (size_t)B * d) ||
        alloc(c, &c->step_x1, (size_t)B * d) || alloc(c, &c->step_o, (size_t)B * c->Hr * hd) ||
        alloc(c, &c->step_bar, 1))
      return cleanup_fail(SIRIUS_ERR_CUDA);
    std::vector<const uint16_t*> wp;
    for (auto* v : {&R.attn_norm, &R.w_qkv, &R.w_o, &R.ffn_norm, &R.w_gate, &R.w_up, &R.w_down})
      wp.insert(wp.end(), v->begin(), v->end());
    cudaMemcpy(c->step_w, wp.data(), sizeof(const uint16_t*) * wp.size(), cudaMemcpyHostToDevice);
    c->step_splits = launch::decode_step_splits(B, c->KVr, c->num_sms);
  }
  if (cudaStreamSynchronize(c->stream) != cudaSuccess || cudaGetLastError() != cudaSuccess)
    return cleanup_fail(SIRIUS_ERR_CUDA);
  *out = c;
  return SIRIUS_OK;
}

sirius_status sirius_destroy(sirius_ctx* c) {
  if (!c) return SIRIUS_ERR_INVALID_ARG;
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto& e : c->prof) {
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  for (auto& g : c->graphs) {
    cudaGraphExecDestroy(g.exec);
    for (auto& e : g.evs) {
      cudaEventDestroy(e.a);
      cudaEventDestroy(e.b);
    }
  }
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  for (void* p : c->par_opened) cudaIpcCloseMemHandle(p);
  for (void* p : c->allocations) cudaFree(p);
  if (c->err_host) cudaFreeHost(c->err_host);
  if (c->pre_start_host) cudaFreeHost(c->pre_start_host);
  delete c;
  return SIRIUS_OK;
}

sirius_status sirius_prefill(sirius_ctx* c, const int32_t* tokens, const int32_t* prompt_len, int32_t* first_token) {
  if (!c || !tokens || !prompt_len || !first_token) return SIRIUS_ERR_INVALID_ARG;
  OK(check_sticky(c));
  const sirius_config& cf = c->cfg;
  long off = 0;
  for (int b = 0; b < cf.batch; ++b) {
    if (prompt_len[b] < 1) return fail(c, SIRIUS_ERR_INVALID_ARG, "prompt_len must be >= 1");
    if (prompt_len[b] > cf.max_seq - cf.max_gamma) return fail(c, SIRIUS_ERR_CAPACITY, "prompt longer than max_seq - max_gamma");
  }
  const int d = cf.d_model;
  c->cs_ready = false;
  if (c->cs_keep > 0.f)
    for (auto& R : c->ranks) CU(cudaMemsetAsync(R.cs_stats, 0, sizeof(float) * cf.n_layers * c->Fr, c->stream));
  for (int b = 0; b < cf.batch; ++b) {
    const int P = prompt_len[b];
    for (int s = 0; s < P; s += c->MAXM) {
      const int rows = P - s < c->MAXM ? P - s : c->MAXM;
      c->pre_start_host[b] = s;
      CU(cudaMemcpyAsync(c->pre_start + b, c->pre_start_host + b, sizeof(int32_t), cudaMemcpyHostToDevice, c->stream));
      OK(forward_rows(c, tokens + off + s, c->pre_start, b, 1, rows, ROWS_PREFILL));
      CU(cudaStreamSynchronize(c->stream));  // pre_start_host reuse
      if (s + rows == P) {  // dense greedy next token from the last prompt row (reading D17)
        for (auto& R : c->ranks) {
          GemvArgs a = {};
          a.pro.mode = IN_RESID;
          a.pro.base = R.resB + (size_t)(rows - 1) * d;
          a.pro.delta = R.dF + (size_t)(rows - 1) * d;
          a.pro.norm_w = R.final_norm;
          a.pro.eps = cf.rms_eps;
          a.W = R.lm_head;
          a.rows = c->Vr;
          a.K = d;
          a.epi = EPI_ARGMAX;
          a.ldo = c->Vr;
          a.amax = c->amax;
          a.index_offset = (uint32_t)R.rank * c->Vr;
          a.finalize = (cf.tp_size == 1);
          a.done_counter = R.head_cnt;
          a.token_out = first_token + b;
          OK(run_gemv(c, a, 1));
        }
        if (cf.tp_size > 1) {
          if (!c->emulated && !c->stub_comm) {
            NcclApi& api = nccl();
            int r = api.allReduce(c->amax, c->amax, 1, kNcclUint64, kNcclMax, c->comm, c->stream);
            if (r != 0) return fail(c, SIRIUS_ERR_NCCL, "ncclAllReduce(max)");
          }
          LCU(launch::argmax_finalize(c->amax, 1, first_token + b, c->stream));
        }
      }
    }
    off += P;
  }
  if (c->cs_keep > 0.f) {  // CSparse plan of this prompt (reading D28) + compact weights
    const int L = cf.n_layers, k = c->cs_k;
    const size_t per = (size_t)k * d;
    for (auto& R : c->ranks) {
      LCU(launch::csparse_select(R.cs_stats, L, c->Fr, k, R.cs_idx, c->stream));
      for (int l = 0; l < L; ++l) {
        const int32_t* idx = R.cs_idx + (size_t)l * k;
        LCU(launch::csparse_gather(R.w_gate[l], idx, k, d, R.cs_w + (0 * (size_t)L + l) * per, c->num_sms, c->stream));
        LCU(launch::csparse_gather(R.w_up[l], idx, k, d, R.cs_w + (1 * (size_t)L + l) * per, c->num_sms, c->stream));
        LCU(launch::csparse_gather(R.w_down[l], idx, k, d, R.cs_w + (2 * (size_t)L + l) * per, c->num_sms, c->stream));
      }
    }
    c->cs_ready = true;
  }
  mirror_err(c);
  CU(cudaGetLastError());
  c->prefilled = true;
  c->have_correct = false;
  return SIRIUS_OK;
}

// Sampled decoding (reading D31): temperature > 0 makes
// sparse_decode_step sample its token and correct_kernel sample the interleaved / bonus token.
sirius_status sirius_set_sampling(sirius_ctx* c, float temperature, uint64_t seed) {
  if (!c || !(temperature >= 0.f) || !std::isfinite(temperature)) return SIRIUS_ERR_INVALID_ARG;
  OK(check_sticky(c));
  if (temperature > 0.f && c->cfg.tp_size != 1) return fail(c, SIRIUS_ERR_UNSUPPORTED, "sampling: TP 1 only");
  c->samp_temp = temperature;
  c->samp_seed = seed;
  return SIRIUS_OK;
}

// Top-k FSparse (PAPER.md:121 footnote): SIRIUS_TOPK decode steps keep, per layer
// and sequence, the k = round(keep_fraction * ffn) neurons of largest |SiLU(g)| (reading D30).
sirius_status sirius_topk_enable(sirius_ctx* c, float keep_fraction) {
  if (!c || !(keep_fraction >= 0.f && keep_fraction <= 1.f)) return SIRIUS_ERR_INVALID_ARG;
  OK(check_sticky(c));
  const sirius_config& cf = c->cfg;
  if (keep_fraction == 0.f) {
    c->topk_k = 0;
    return SIRIUS_OK;
  }
  if (cf.tp_size != 1 || cf.batch > 4)
    return fail(c, SIRIUS_ERR_UNSUPPORTED, "top-k FSparse: TP 1 and the per-stage decode path (batch <= 4)");
  const int k = (int)std::floor((double)keep_fraction * c->Fr + 0.5);
  if (k < 1) return fail(c, SIRIUS_ERR_UNSUPPORTED, "top-k FSparse: keep_fraction * ffn rounds to 0");
  if (c->Fr > 32768) return fail(c, SIRIUS_ERR_UNSUPPORTED, "top-k FSparse: at most 32768 neurons per layer");
  for (auto& R : c->ranks) {
    if (R.tk_g) continue;
    if (alloc(c, &R.tk_g, (size_t)cf.batch * c->Fr) || alloc(c, &R.tk_a, (size_t)cf.batch * c->Fr) ||
        alloc(c, &R.tk_mask, (size_t)cf.batch * (c->Fr / 32 + 1)))
      return SIRIUS_ERR_CUDA;
  }
  c->topk_k = k;
  return SIRIUS_OK;
}

// ---- fused peer all-reduce (SURVEY.md §8(e) phase 2; peer_ar.cuh, include/sirius.h)
sirius_status sirius_par_export(sirius_ctx* c, void* handle_out) {
  if (!c || !handle_out) return SIRIUS_ERR_INVALID_ARG;
  OK(check_sticky(c));
  if (c->cfg.tp_size == 1 || c->emulated || c->stub_comm)
    return fail(c, SIRIUS_ERR_STATE, "sirius_par_export: only a real tensor-parallel rank (tp_size > 1, NCCL) exports");
  CU(cudaDeviceSynchronize());  // the buffer's zeroing (flags 0) is complete before any peer can map it
  cudaIpcMemHandle_t h;
  CU(cudaIpcGetMemHandle(&h, c->ranks[0].par_buf));
  memcpy(handle_out, &h, sizeof(h));
  return SIRIUS_OK;
}

sirius_status sirius_par_enable(sirius_ctx* c, const void* peer_handles) {
  if (!c) return SIRIUS_ERR_INVALID_ARG;
  OK(check_sticky(c));
  const sirius_config& cf = c->cfg;
  if (cf.tp_size == 1) return fail(c, SIRIUS_ERR_UNSUPPORTED, "sirius_par_enable: tp_size 1 has no all-reduce");
  if (cf.tp_size > 8) return fail(c, SIRIUS_ERR_UNSUPPORTED, "sirius_par_enable: at most 8 ranks");
  if (c->par_on) return SIRIUS_OK;
  const bool real = !c->emulated && !c->stub_comm;
  if (real != (peer_handles != nullptr))
    return fail(c, SIRIUS_ERR_INVALID_ARG, real ? "sirius_par_enable: a real rank needs the peers' handles"
                                                : "sirius_par_enable: emulated / stub contexts take no handles");
  std::vector<char*> peers(cf.tp_size);
  if (c->emulated) {  // every emulated rank's buffer is in this process
    for (int r = 0; r < cf.tp_size; ++r) peers[r] = c->ranks[r].par_buf;
  } else if (c->stub_comm) {
    for (int r = 0; r < cf.tp_size; ++r) peers[r] = c->ranks[0].par_buf;
  } else {
    const cudaIpcMemHandle_t* hs = static_cast<const cudaIpcMemHandle_t*>(peer_handles);
    for (int r = 0; r < cf.tp_size; ++r) {
      if (r == cf.tp_rank) {
        peers[r] = c->ranks[0].par_buf;
        continue;
      }
      void* p = nullptr;
      if (cudaIpcOpenMemHandle(&p, hs[r], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        for (void* q : c->par_opened) cudaIpcCloseMemHandle(q);
        c->par_opened.clear();
        return fail(c, SIRIUS_ERR_UNSUPPORTED, "sirius_par_enable: cudaIpcOpenMemHandle failed (no peer access?)");
      }
      c->par_opened.push_back(p);
      peers[r] = static_cast<char*>(p);
    }
  }
  for (auto& R : c->ranks) CU(cudaMemcpy(R.par_peers, peers.data(), sizeof(char*) * peers.size(), cudaMemcpyHostToDevice));
  c->par_loopback = c->stub_comm;
  c->par_on = true;
  return SIRIUS_OK;
}

sirius_status sirius_par_disable(sirius_ctx* c) {
  if (!c) return SIRIUS_ERR_INVALID_ARG;
  c->par_on = false;  // the peers stay mapped (sirius_destroy unmaps); the sequence numbers keep counting
  return SIRIUS_OK;
}

// CSparse: allocate the plan and the compact weights; every later sirius_prefill
// gathers the statistic and builds the plan (reading D28); SIRIUS_CSPARSE decode steps use it.
sirius_status sirius_csparse_enable(sirius_ctx* c, float keep_fraction) {
  if (!c || !(keep_fraction >= 0.f && keep_fraction <= 1.f)) return SIRIUS_ERR_INVALID_ARG;
  OK(check_sticky(c));
  const sirius_config& cf = c->cfg;
  if (keep_fraction == 0.f) {
    c->cs_keep = 0.f;
    c->cs_ready = false;
    return SIRIUS_OK;
  }
  if (cf.batch != 1) return fail(c, SIRIUS_ERR_UNSUPPORTED, "CSparse: batch 1 only (one prompt, one neuron set)");
  const int k = (int)std::floor((double)keep_fraction * c->Fr + 0.5);
  if (k < 8 || k % 8) return fail(c, SIRIUS_ERR_UNSUPPORTED, "CSparse: kept neurons per rank must be a multiple of 8");
  const int L = cf.n_layers;
  for (auto& R : c->ranks) {
    if (R.cs_stats) continue;  // allocated by an earlier call for the full width
    if (alloc(c, &R.cs_stats, (size_t)L * c->Fr) || alloc(c, &R.cs_scratch, (size_t)c->MAXM * c->Fr) ||
        alloc(c, &R.cs_idx, (size_t)L * c->Fr) || alloc(c, &R.cs_w, (size_t)3 * L * c->Fr * cf.d_model, false))
      return SIRIUS_ERR_CUDA;
  }
  c->cs_keep = keep_fraction;
  c->cs_k = k;
  c->cs_ready = false;
  return SIRIUS_OK;
}

// test/debug: the last prefill's statistic [n_layers, ffn/tp] (DEV fp32) and plan [n_layers, k] (DEV
// int32, ascending neuron indices within the shard); either may be NULL.  Synchronous.
int sirius_debug_csparse_plan(sirius_ctx* c, float* stats_out, int32_t* idx_out, int32_t* k_out) {
  if (!c || !c->cs_ready) return SIRIUS_ERR_STATE;
  RankState& R = c->ranks[0];
  const int L = c->cfg.n_layers;
  if (k_out) *k_out = c->cs_k;
  cudaStreamSynchronize(c->stream);
  if (stats_out) cudaMemcpy(stats_out, R.cs_stats, sizeof(float) * L * c->Fr, cudaMemcpyDeviceToDevice);
  if (idx_out) cudaMemcpy(idx_out, R.cs_idx, sizeof(int32_t) * L * c->cs_k, cudaMemcpyDeviceToDevice);
  return (int)cudaGetLastError();
}

static sirius_status enqueue_head_argmax(sirius_ctx* c, const int32_t* tokens, int gamma, int M, float* logits_out,
                                         int32_t* n_accept_out, int32_t* next_token_out, float* q_out,
                                         float accept_threshold, int32_t accept_mode);

// Batched decode (batch >= 4) through the tensor-core row path: one row per sequence at pos[b] (K/V
// straight into the cache), CATS mask in the SwiGLU epilogue (sparse) — at these batch sizes the
// union of the per-sequence active sets covers ~all neurons (SURVEY.md §7 hard part 7), so every
// W_up / W_down row is read anyway and inactive (b, n) pairs contribute exact zeros (reading D19) —
// then final norm + head GEMM + argmax (accept machinery with gamma = 1: next = argmax row 0).
static sirius_status enqueue_decode_rows(sirius_ctx* c, const int32_t* token_in, const int32_t* pos, bool dense,
                                         int32_t* token_out, float* logits_out, int32_t* n_active_out,
                                         float* gate_act_out) {
  const int B = c->cfg.batch;
  if (n_active_out) CU(cudaMemsetAsync(n_active_out, 0, sizeof(int32_t) * B * c->cfg.n_layers, c->stream));
  prof_begin(c, P_STEP);
  OK(forward_rows(c, token_in, pos, 0, B, 1, ROWS_DECODE, !dense, n_active_out, gate_act_out));
  OK(enqueue_head_argmax(c, token_in, 1, B, logits_out, c->dec_nacc, token_out, nullptr, 0.f, 0));
  if (c->samp_temp > 0.f) {
    const float* lo = logits_out ? logits_out : c->ranks[0].logits;
    LCU(launch::sample_tokens(lo, c->Vr, c->Vr, c->samp_temp, c->samp_seed, pos, nullptr, 1, token_out, B, c->stream));
  }
  prof_end(c);
  CU(cudaGetLastError());
  return SIRIUS_OK;
}

static sirius_status enqueue_decode(sirius_ctx* c, const int32_t* token_in, const int32_t* pos, uint32_t flags,
                                    int32_t* token_out, float* logits_out, int32_t* n_active_out,
                                    float* gate_act_out) {
  const sirius_config& cf = c->cfg;
  const int B = cf.batch, d = cf.d_model, hd = cf.head_dim, L = cf.n_layers;
  const bool dense = flags & SIRIUS_DENSE;
  const bool csparse = flags & SIRIUS_CSPARSE;
  const bool topk = flags & SIRIUS_TOPK;
  // top-k / CSparse steps run the per-stage kernels (batch <= 4) even where dense / CATS steps take the rows
  if (c->decode_rows && !topk && !csparse)
    return enqueue_decode_rows(c, token_in, pos, dense, token_out, logits_out, n_active_out,
                                                 gate_act_out);
  if (n_active_out) CU(cudaMemsetAsync(n_active_out, 0, sizeof(int32_t) * B * L, c->stream));
  if (c->use_step && !csparse && !topk && c->samp_temp == 0.f) {  // the whole step in one persistent launch
    RankState& R = c->ranks[0];
    StepArgs s = {};
    s.d = d;
    s.L = L;
    s.Hr = c->Hr;
    s.KVr = c->KVr;
    s.hd = hd;
    s.F = c->Fr;
    s.Vr = c->Vr;
    s.vocab = cf.vocab;
    s.max_seq = cf.max_seq;
    s.splits = c->step_splits;
    s.eps = cf.rms_eps;
    s.attn_scale = 1.0f / sqrtf((float)hd);
    s.dense = dense ? 1 : 0;
    s.tokens = token_in;
    s.pos = pos;
    s.token_out = token_out;
    s.logits_out = logits_out;
    s.n_active_out = n_active_out;
    s.gate_out = gate_act_out;
    s.gate_stride = (long long)L * c->Fr;
    s.embed = R.embed;
    s.final_norm = R.final_norm;
    s.lm_head = R.lm_head;
    s.attn_norm = c->step_w + 0 * L;
    s.w_qkv = c->step_w + 1 * L;
    s.w_o = c->step_w + 2 * L;
    s.ffn_norm = c->step_w + 3 * L;
    s.w_gate = c->step_w + 4 * L;
    s.w_up = c->step_w + 5 * L;
    s.w_down = c->step_w + 6 * L;
    s.thresholds = c->thresholds;
    s.k_cache = R.k_cache;
    s.v_cache = R.v_cache;
    s.kv_layer = (size_t)B * c->KVr * cf.max_seq * hd;
    s.rope_cos = c->rope_cos;
    s.rope_sin = c->rope_sin;
    s.x = c->step_x;
    s.x1 = c->step_x1;
    s.qkv = R.qkv;
    s.o = c->step_o;
    s.attn_part = R.attn_part;
    s.ffn_part = R.ffn_part;
    s.part_cnt = R.ffn_cnt;
    s.group_bar = R.attn_bar;
    s.grid_bar = c->step_bar;
    s.amax = c->amax;
    s.head_cnt = R.head_cnt;
    s.err = c->err_dev;
    s.trace = c->trace;
    s.tune = c->step_tune;
    prof_begin(c, P_STEP);
    LCU(launch::decode_step(s, B, c->num_sms, c->stream));
    prof_end(c);
    CU(cudaGetLastError());
    return SIRIUS_OK;
  }
  // TP > 1 with sirius_par_enable: the all-reduces are fused into the producing kernels' epilogues and
  // the consuming kernels' prologues (peer_ar.cuh) instead of NCCL launches between them
  const bool par = c->par_on && cf.tp_size > 1;
  for (int l = 0; l < L; ++l) {
    for (auto& R : c->ranks) {
      GemvArgs a = {};
      if (l == 0) {
        a.pro.mode = IN_EMBED;
        a.pro.tokens = token_in;
        a.pro.embed = R.embed;
        a.pro.vocab = cf.vocab;
      } else {
        a.pro.mode = IN_RESID;
        a.pro.base = R.resB;
        a.pro.delta = R.dF;
      }
      a.pro.norm_w = R.attn_norm[l];
      a.pro.eps = cf.rms_eps;
      a.pro.res_out = R.resA;
      a.W = R.w_qkv[l];
      a.rows = c->Nqkv;
      a.K = d;
      a.epi = EPI_STORE;
      a.out = R.qkv;
      a.ldo = c->Nqkv;
      prof_begin(c, P_QKV);
      OK(run_gemv(c, a, B));
      prof_end(c);
      const size_t kv_layer = (size_t)B * c->KVr * cf.max_seq * hd;
      prof_begin(c, P_ATTN);
      {  // one (sequence, kv head, split) item per 512-thread CTA, last-split combine (decode_step.cu)
        StepArgs sa = {};
        sa.d = d;
        sa.Hr = c->Hr;
        sa.KVr = c->KVr;
        sa.hd = hd;
        sa.max_seq = cf.max_seq;
        sa.splits = c->attn_stage_splits;
        sa.attn_scale = 1.0f / sqrtf((float)hd);
        sa.pos = pos;
        sa.qkv = R.qkv;
        sa.o = R.ob;
        sa.k_cache = R.k_cache;
        sa.v_cache = R.v_cache;
        sa.kv_layer = kv_layer;
        sa.rope_cos = c->rope_cos;
        sa.rope_sin = c->rope_sin;
        sa.attn_part = R.attn_part;
        sa.group_bar = R.attn_bar;
        sa.err = c->err_dev;
        LCU(launch::attn_stage(sa, l, B, c->stream));
      }
      prof_end(c);
      GemvArgs o = {};
      o.pro.mode = IN_F32;
      o.pro.in_f32 = R.ob;
      o.W = R.w_o[l];
      o.rows = d;
      o.K = c->Hr * hd;
      o.epi = EPI_STORE;
      o.out = R.dA;
      o.ldo = d;
      if (c->ffn_atomic) {  // zero the FFN accumulator dF (the QKV prologue above consumed it)
        o.zero_out = R.dF;
        o.zero_n = B * d;
      }
      if (par) o.par = par_of(c, R);  // fused peer all-reduce of the O-proj partial
      prof_begin(c, P_OPROJ);
      OK(run_gemv(c, o, B));
      prof_end(c);
    }
    OK(par_or_allreduce(c, &RankState::dA, c->dA_ptrs, B, par));
    for (auto& R : c->ranks) {
      float* g_out = nullptr;
      long long g_stride = 0;
      if (gate_act_out) {  // [B, L, F] (emulated group: rank shards concatenated) or [B, L, F/tp]
        const int F = c->emulated ? cf.ffn_dim : c->Fr;
        g_out = gate_act_out + (size_t)l * F + (c->emulated ? (size_t)R.rank * c->Fr : 0);
        g_stride = (long long)L * F;
      }
      prof_begin(c, P_FFN);
      OK(launch_decode_ffn(c, R, l, R.resA, R.dA, R.resB, R.dF, dense, n_active_out ? n_active_out + l : nullptr, L,
                           g_out, g_stride, csparse, topk, par));
      prof_end(c);
    }
    OK(par_or_allreduce(c, &RankState::dF, c->dF_ptrs, B, par));
  }
  for (auto& R : c->ranks) {
    GemvArgs a = {};
    a.pro.mode = IN_RESID;
    a.pro.base = R.resB;
    a.pro.delta = R.dF;
    a.pro.norm_w = R.final_norm;
    a.pro.eps = cf.rms_eps;
    a.W = R.lm_head;
    a.rows = c->Vr;
    a.K = d;
    a.epi = EPI_ARGMAX;
    a.out = logits_out ? logits_out + (c->emulated ? (size_t)R.rank * c->Vr : 0)
                       : (c->samp_temp > 0.f ? R.logits : nullptr);  // sampling needs the logits
    a.ldo = logits_out ? (c->emulated ? cf.vocab : c->Vr) : c->Vr;
    a.amax = c->amax;
    a.index_offset = (uint32_t)R.rank * c->Vr;
    a.finalize = (cf.tp_size == 1);
    a.done_counter = R.head_cnt;
    a.token_out = token_out;
    if (par) a.par = par_of(c, R);  // the packed argmax keys max-reduced over the ranks -> token
    prof_begin(c, P_HEAD);
    OK(run_gemv(c, a, B));
    prof_end(c);
  }
  if (par) {
    if (c->emulated)
      for (auto& R : c->ranks) LCU(launch::par_reduce(par_of(c, R), nullptr, 0, B, token_out, c->stream));
  } else if (cf.tp_size > 1) {
    if (!c->emulated && !c->stub_comm) {
      NcclApi& api = nccl();
      int r = api.allReduce(c->amax, c->amax, B, kNcclUint64, kNcclMax, c->comm, c->stream);
      if (r != 0) return fail(c, SIRIUS_ERR_NCCL, "ncclAllReduce(max)");
    }
    LCU(launch::argmax_finalize(c->amax, B, token_out, c->stream));
  }
  if (c->samp_temp > 0.f) {  // sampled draft (reading D31): the token at position pos + 1
    const float* lo = logits_out ? logits_out : c->ranks[0].logits;
    LCU(launch::sample_tokens(lo, c->Vr, c->Vr, c->samp_temp, c->samp_seed, pos, nullptr, 1, token_out, B, c->stream));
  }
  CU(cudaGetLastError());
  return SIRIUS_OK;
}

sirius_status sparse_decode_step(sirius_ctx* c, const int32_t* token_in, const int32_t* pos, uint32_t flags,
                                 int32_t* token_out, float* logits_out, int32_t* n_active_out, float* gate_act_out) {
  if (!c || !token_in || !pos || !token_out) return SIRIUS_ERR_INVALID_ARG;
  if (flags & ~(uint32_t)(SIRIUS_DENSE | SIRIUS_CSPARSE | SIRIUS_TOPK)) return fail(c, SIRIUS_ERR_INVALID_ARG, "unknown flag");
  if (__builtin_popcount(flags & (SIRIUS_DENSE | SIRIUS_CSPARSE | SIRIUS_TOPK)) > 1)
    return fail(c, SIRIUS_ERR_INVALID_ARG, "DENSE, CSPARSE and TOPK are exclusive");
  if ((flags & SIRIUS_TOPK) && !c->topk_k)
    return fail(c, SIRIUS_ERR_STATE, "TOPK decode without sirius_topk_enable");
  if ((flags & SIRIUS_CSPARSE) && gate_act_out) return fail(c, SIRIUS_ERR_INVALID_ARG, "CSPARSE exports no gate");
  OK(check_sticky(c));
  if ((flags & SIRIUS_CSPARSE) && !c->cs_ready)
    return fail(c, SIRIUS_ERR_STATE, "CSPARSE decode without a plan (sirius_csparse_enable + sirius_prefill)");
  uint32_t tbits;
  memcpy(&tbits, &c->samp_temp, 4);
  GraphKey key = {0xDEC0u, flags, (uintptr_t)token_in, (uintptr_t)pos, (uintptr_t)token_out, (uintptr_t)logits_out,
                  (uintptr_t)n_active_out, (uintptr_t)gate_act_out, (uintptr_t)tbits, (uintptr_t)c->samp_seed};
  return run_graphed(c, key, [&] {
    OK(enqueue_decode(c, token_in, pos, flags, token_out, logits_out, n_active_out, gate_act_out));
    mirror_err(c);  // a position outside [0, max_seq) is reported by the NEXT call (include/sirius.h)
    return SIRIUS_OK;
  });
}

static sirius_status enqueue_correct(sirius_ctx* c, const int32_t* kernel_tokens, const int32_t* start_pos,
                                     int32_t gamma, float accept_threshold, int32_t accept_mode,
                                     int32_t* n_accept_out, int32_t* next_token_out, float* q_out,
                                     float* logits_out) {
  const sirius_config& cf = c->cfg;
  const int B = cf.batch, d = cf.d_model, M = B * gamma;
  prof_begin(c, P_VERIFY);
  OK(forward_rows(c, kernel_tokens, start_pos, 0, B, gamma, ROWS_VERIFY));
  OK(enqueue_head_argmax(c, kernel_tokens, gamma, M, logits_out, n_accept_out, next_token_out, q_out,
                         accept_threshold, accept_mode));
  if (c->samp_temp > 0.f) {  // interleaved / bonus token sampled from the full model's row j (reading D31)
    const float* lo = logits_out ? logits_out : c->ranks[0].logits;
    LCU(launch::sample_tokens(lo, c->Vr, c->Vr, c->samp_temp, c->samp_seed, start_pos, n_accept_out, gamma,
                              next_token_out, B, c->stream));
  }
  prof_end(c);
  mirror_err(c);
  CU(cudaGetLastError());
  return SIRIUS_OK;
}

// final RMSNorm of the M rows + head GEMM + per-row softmax statistics (+ TP all-gather) + the accept
// scan / interleave (gamma = 1: next = argmax of the row)
static sirius_status enqueue_head_argmax(sirius_ctx* c, const int32_t* kernel_tokens, int gamma, int M,
                                         float* logits_out, int32_t* n_accept_out, int32_t* next_token_out,
                                         float* q_out, float accept_threshold, int32_t accept_mode) {
  const sirius_config& cf = c->cfg;
  const int B = cf.batch, d = cf.d_model;
  for (auto& R : c->ranks) {
    NormRowsArgs na = {};
    na.base = R.resB;
    na.delta = R.dF;
    if (c->rows_par) par_consume_rows(c, R, na);  // the last forward_rows fused its all-reduces
    na.vocab = cf.vocab;
    na.d = d;
    na.norm_w = R.final_norm;
    na.eps = cf.rms_eps;
    na.out3 = R.xn3;
    na.plane = (size_t)c->MAXM * d;
    LCU(launch::norm_rows(na, M, c->stream));
    float* lo = logits_out ? logits_out + (c->emulated ? (size_t)R.rank * c->Vr : 0) : R.logits;
    const int ldl = logits_out ? (c->emulated ? cf.vocab : c->Vr) : c->Vr;
    OK(run_gemm(c, R, R.lm_head, nullptr, R.xn3, c->Vr, d, M, lo, ldl));
    AcceptStatsArgs as = {};
    as.logits = lo;
    as.ldl = ldl;
    as.Vr = c->Vr;
    as.voff = R.rank * c->Vr;
    as.M = M;
    as.gamma = gamma;
    as.rank = c->emulated ? R.rank : 0;
    as.tokens = kernel_tokens;
    as.stats = c->stats;
    LCU(launch::accept_stats(as, c->accept_splits, c->stream));
  }
  const RowStat* stats = c->stats;
  int nranks = c->nranks;
  if (cf.tp_size > 1 && !c->emulated && !c->stub_comm) {
    NcclApi& api = nccl();
    int r = api.allGather(c->stats, c->stats_gather, (size_t)M * c->accept_splits * sizeof(RowStat), kNcclUint8,
                          c->comm, c->stream);
    if (r != 0) return fail(c, SIRIUS_ERR_NCCL, "ncclAllGather(stats)");
    stats = c->stats_gather;
    nranks = cf.tp_size;
  }
  AcceptFinalArgs fa = {};
  fa.stats = stats;
  fa.nranks = nranks;
  fa.S = c->accept_splits;
  fa.M = M;
  fa.gamma = gamma;
  fa.mode = accept_mode;
  fa.r = accept_threshold;
  fa.tokens = kernel_tokens;
  fa.n_accept = n_accept_out;
  fa.next_token = next_token_out;
  fa.q_out = q_out;
  fa.row_argmax = n_accept_out == c->dec_nacc ? nullptr : c->row_argmax;  // verify rows only
  LCU(launch::accept_finalize(fa, B, c->stream));
  return SIRIUS_OK;
}

sirius_status correct_kernel(sirius_ctx* c, const int32_t* kernel_tokens, const int32_t* start_pos, int32_t gamma,
                             float accept_threshold, int32_t accept_mode, int32_t* n_accept_out,
                             int32_t* next_token_out, float* q_out, float* logits_out) {
  if (!c || !kernel_tokens || !start_pos || !n_accept_out || !next_token_out) return SIRIUS_ERR_INVALID_ARG;
  if (accept_mode != SIRIUS_ACCEPT_THRESHOLD && accept_mode != SIRIUS_ACCEPT_EXACT_ARGMAX)
    return fail(c, SIRIUS_ERR_INVALID_ARG, "accept_mode");
  if (!(accept_threshold >= 0.f && accept_threshold <= 1.f)) return fail(c, SIRIUS_ERR_INVALID_ARG, "r outside [0,1]");
  if (gamma < 1) return fail(c, SIRIUS_ERR_INVALID_ARG, "gamma < 1");
  if (gamma > c->cfg.max_gamma) return fail(c, SIRIUS_ERR_CAPACITY, "gamma > max_gamma");
  OK(check_sticky(c));
  uint32_t rbits;
  memcpy(&rbits, &accept_threshold, 4);
  uint32_t tbits;
  memcpy(&tbits, &c->samp_temp, 4);
  GraphKey key = {0xC0EEu, (uintptr_t)gamma, (uintptr_t)rbits, (uintptr_t)accept_mode, (uintptr_t)kernel_tokens,
                  (uintptr_t)start_pos, (uintptr_t)n_accept_out, (uintptr_t)next_token_out, (uintptr_t)q_out,
                  (uintptr_t)logits_out, (uintptr_t)tbits, (uintptr_t)c->samp_seed};
  OK(run_graphed(c, key, [&] {
    return enqueue_correct(c, kernel_tokens, start_pos, gamma, accept_threshold, accept_mode, n_accept_out,
                           next_token_out, q_out, logits_out);
  }));
  c->last_gamma = gamma;
  c->have_correct = true;
  c->tree_last = false;
  return SIRIUS_OK;
}

// ---- tree correction kernel (tree.cu, reading D29), batch 1, TP 1:
// drafting steps s = 1 .. gamma-1 through the verify row machinery with the CATS FFN and ancestor-masked
// attention (the step-(s-1) nodes' sparse K/V land in their staging rows), head GEMM, top-k + prune; then
// one dense forward over every tree row, head GEMM, per-row LSE / argmax, accept on every leaf's path.
static sirius_status head_rows(sirius_ctx* c, RankState& R, int M) {  // final RMSNorm + LM head -> R.logits
  const sirius_config& cf = c->cfg;
  NormRowsArgs na = {};
  na.base = R.resB;
  na.delta = R.dF;
  if (c->rows_par) par_consume_rows(c, R, na);  // the last forward_rows fused its all-reduces
  na.vocab = cf.vocab;
  na.d = cf.d_model;
  na.norm_w = R.final_norm;
  na.eps = cf.rms_eps;
  na.out3 = R.xn3;
  na.plane = (size_t)c->MAXM * cf.d_model;
  LCU(launch::norm_rows(na, M, c->stream));
  OK(run_gemm(c, R, R.lm_head, nullptr, R.xn3, c->Vr, cf.d_model, M, R.logits, c->Vr));
  return SIRIUS_OK;
}

static sirius_status enqueue_tree(sirius_ctx* c, const int32_t* pending, const int32_t* start_pos, int gamma,
                                  int width, int branch, float r, int mode, int32_t* n_accept_out,
                                  int32_t* next_token_out, int32_t* path_tokens_out) {
  RankState& R = c->ranks[0];
  TreeState* ts = c->tree;
  const int S = gamma - 1, W = width, n_rows = 1 + S * W;
  const int kb = W > branch ? W : branch;
  prof_begin(c, P_VERIFY);
  LCU(launch::tree_init(ts, pending, c->stream));
  for (int s = 1; s <= S; ++s) {  // sparse drafting (Alg. 1 lines 6-11 with a tree)
    const int np = s == 1 ? 1 : W, f0 = s == 1 ? 0 : 1 + (s - 2) * W;
    OK(forward_rows(c, ts->tok + f0, start_pos, 0, 1, np, ROWS_VERIFY, true, nullptr, nullptr, f0, ts->row_off + f0,
                    ts->vis));
    OK(head_rows(c, R, np));
    LCU(launch::tree_topk(R.logits, c->Vr, c->Vr, np, kb, ts, f0, c->stream));
    LCU(launch::tree_prune(ts, s, W, branch, c->stream));
  }
  // full-model verification of every tree row (staging rows [0, n_rows) rewritten with the full K/V)
  OK(forward_rows(c, ts->tok, start_pos, 0, 1, n_rows, ROWS_VERIFY, false, nullptr, nullptr, 0, ts->row_off, ts->vis));
  OK(head_rows(c, R, n_rows));
  LCU(launch::tree_topk(R.logits, c->Vr, c->Vr, n_rows, 1, ts, 0, c->stream));
  LCU(launch::tree_accept(R.logits, c->Vr, ts, S, W, r, mode, n_accept_out, next_token_out, path_tokens_out, gamma,
                          c->stream));
  prof_end(c);
  mirror_err(c);
  CU(cudaGetLastError());
  return SIRIUS_OK;
}

sirius_status sirius_tree_kernel(sirius_ctx* c, const int32_t* pending, const int32_t* start_pos, int32_t gamma,
                                 int32_t width, int32_t branch, float accept_threshold, int32_t accept_mode,
                                 int32_t* n_accept_out, int32_t* next_token_out, int32_t* path_tokens_out) {
  if (!c || !pending || !start_pos || !n_accept_out || !next_token_out || !path_tokens_out)
    return SIRIUS_ERR_INVALID_ARG;
  if (accept_mode != SIRIUS_ACCEPT_THRESHOLD && accept_mode != SIRIUS_ACCEPT_EXACT_ARGMAX)
    return fail(c, SIRIUS_ERR_INVALID_ARG, "accept_mode");
  if (!(accept_threshold >= 0.f && accept_threshold <= 1.f)) return fail(c, SIRIUS_ERR_INVALID_ARG, "r outside [0,1]");
  if (gamma < 1 || width < 1 || width > kTreeMaxW || branch < 1 || branch > kTreeMaxKB)
    return fail(c, SIRIUS_ERR_INVALID_ARG, "gamma / width / branch");
  const int n_rows = 1 + (gamma - 1) * width;
  if (n_rows > kTreeMaxRows || n_rows > c->cfg.max_gamma) return fail(c, SIRIUS_ERR_CAPACITY, "tree rows > max_gamma / 64");
  if (c->cfg.batch != 1 || c->cfg.tp_size != 1) return fail(c, SIRIUS_ERR_UNSUPPORTED, "tree kernels: batch 1, TP 1");
  OK(check_sticky(c));
  uint32_t rbits;
  memcpy(&rbits, &accept_threshold, 4);
  GraphKey key = {0x7EEEu, (uintptr_t)gamma, (uintptr_t)width, (uintptr_t)branch, (uintptr_t)rbits,
                  (uintptr_t)accept_mode, (uintptr_t)pending, (uintptr_t)start_pos, (uintptr_t)n_accept_out,
                  (uintptr_t)next_token_out, (uintptr_t)path_tokens_out};
  OK(run_graphed(c, key, [&] {
    return enqueue_tree(c, pending, start_pos, gamma, width, branch, accept_threshold, accept_mode, n_accept_out,
                        next_token_out, path_tokens_out);
  }));
  c->last_gamma = gamma;
  c->have_correct = true;
  c->tree_last = true;
  return SIRIUS_OK;
}

static sirius_status enqueue_rewrite(sirius_ctx* c, const int32_t* start_pos, const int32_t* n_rows) {
  const sirius_config& cf = c->cfg;
  for (auto& R : c->ranks) {
    KvRewriteArgs a = {};
    a.stage_k = R.stage_k;
    a.stage_v = R.stage_v;
    a.k_cache = R.k_cache;
    a.v_cache = R.v_cache;
    a.start = start_pos;
    a.n_rows = n_rows;
    a.B = cf.batch;
    a.KVr = c->KVr;
    a.hd = cf.head_dim;
    a.max_seq = cf.max_seq;
    a.max_gamma = cf.max_gamma;
    a.gamma = c->last_gamma;
    a.rows = c->tree_last ? c->tree->path : nullptr;  // tree kernel: the winning path's staging rows
    a.err = c->err_dev;
    prof_begin(c, P_REWRITE);
    LCU(launch::kv_rewrite(a, cf.n_layers, c->stream));
    prof_end(c);
  }
  mirror_err(c);
  CU(cudaGetLastError());
  return SIRIUS_OK;
}

sirius_status kv_rewrite(sirius_ctx* c, const int32_t* start_pos, const int32_t* n_rows) {
  if (!c || !start_pos || !n_rows) return SIRIUS_ERR_INVALID_ARG;
  if (!c->have_correct) return fail(c, SIRIUS_ERR_STATE, "kv_rewrite without a preceding correct_kernel");
  OK(check_sticky(c));
  GraphKey key = {0xE11Eu, (uintptr_t)start_pos, (uintptr_t)n_rows, (uintptr_t)c->last_gamma, (uintptr_t)c->tree_last};
  OK(run_graphed(c, key, [&] { return enqueue_rewrite(c, start_pos, n_rows); }));
  c->have_correct = false;
  return SIRIUS_OK;
}

sirius_status sirius_verify_row_argmax(sirius_ctx* c, int32_t* out) {
  if (!c || !out) return SIRIUS_ERR_INVALID_ARG;
  if (c->last_gamma < 1) return fail(c, SIRIUS_ERR_STATE, "no correct_kernel call yet");
  OK(check_sticky(c));
  CU(cudaMemcpyAsync(out, c->row_argmax, sizeof(int32_t) * c->cfg.batch * c->last_gamma, cudaMemcpyDeviceToDevice,
                     c->stream));
  return SIRIUS_OK;
}

// ---------------------------------------------------------------- NCCL bootstrap helpers (X4)
int sirius_nccl_available(void) { return nccl().loaded ? 1 : 0; }
int sirius_nccl_unique_id(void* out128) {
  NcclApi& api = nccl();
  if (!api.loaded) return -1;
  return api.getUniqueId(out128);
}
int sirius_nccl_comm_init(int nranks, const void* id128, int rank, void** comm_out) {
  NcclApi& api = nccl();
  if (!api.loaded) return -1;
  NcclUid id;
  memcpy(id.internal, id128, 128);
  return api.commInitRank(comm_out, nranks, id, rank);
}
int sirius_nccl_comm_destroy(void* comm) {
  NcclApi& api = nccl();
  if (!api.loaded || !api.commDestroy) return -1;
  return api.commDestroy(comm);
}

// ---------------------------------------------------------------- bench / test instrumentation
unsigned long long sirius_debug_launches(const sirius_ctx* c) { return c ? c->launches : 0ull; }
// CUDA-graph replay of the ABI calls on (default) / off (every kernel launched from the host).
// on = -1: query only.  Returns the (new) state: 1 = graphs in use.
// Debug: per-phase %globaltimer stamps of the persistent decode step into buf (DEV, u64
// [events][num_sms], events = 10 L + 3), or buf = NULL to stop.  Returns 1 if the step kernel is used.
int sirius_debug_trace(sirius_ctx* c, void* buf) {
  if (!c) return -1;
  c->trace = static_cast<unsigned long long*>(buf);
  return c->use_step ? 1 : 0;
}

// Debug: %globaltimer phase stamps of the verify attention of `layer` into buf (DEV u64 [8][CTAs]);
// layer < 0 stops.  Graphs should be off (the pointer is captured into graphs).
int sirius_debug_trace_verify(sirius_ctx* c, void* buf, int layer) {
  if (!c) return -1;
  c->trace = static_cast<unsigned long long*>(buf);
  c->trace_layer = layer;
  c->trace_ffn = false;
  return 0;
}

// Debug: %globaltimer phase stamps of the decode CATS FFN of `layer` (DEV u64 [8][1024]); graphs off.
int sirius_debug_trace_ffn(sirius_ctx* c, void* buf, int layer) {
  if (!c) return -1;
  c->trace = static_cast<unsigned long long*>(buf);
  c->trace_layer = layer;
  c->trace_ffn = buf != nullptr;
  return 0;
}

int sirius_debug_graphs(sirius_ctx* c, int on) {
  if (!c) return -1;
  if (on >= 0) c->use_graphs = on != 0;
  return c->use_graphs ? 1 : 0;
}
// enable/disable per-kernel event timing (resets the accumulated records)
int sirius_debug_profile(sirius_ctx* c, int on) {
  if (!c) return -1;
  c->prof_on = on != 0;
  c->prof_used = 0;
  for (int i = 0; i < 16; ++i) {
    c->prof_tot[i] = 0.0;
    c->prof_cnt[i] = 0;
  }
  return 0;
}
// totals_ms[P_NUM], counts[P_NUM]: summed device time per kernel class since enabling (synchronises).
// ids: 0 QKV GEMV, 1 decode attention, 2 O-proj GEMV, 3 CATS FFN, 4 LM head, 5 correct_kernel, 6 kv_rewrite
int sirius_debug_profile_read(sirius_ctx* c, float* totals_ms, int* counts) {
  if (!c) return -1;
  cudaStreamSynchronize(c->stream);
  for (int i = 0; i < P_NUM; ++i) {
    totals_ms[i] = (float)c->prof_tot[i];
    counts[i] = c->prof_cnt[i];
  }
  for (size_t i = 0; i < c->prof_used; ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->prof[i].a, c->prof[i].b);
    totals_ms[c->prof[i].id] += ms;
    counts[c->prof[i].id] += 1;
  }
  return 0;
}

// ---------------------------------------------------------------- test-only: copy an internal buffer
// which: 0 resA, 1 resB, 2 dA, 3 dF, 4 qkv, 5 ob (fp32), 6 xn3 (bf16 term planes), 7 k_cache, 8 v_cache,
// 9 stage_k, 10 stage_v, 11 mb3 (bf16 term planes), 12 qb (fp32).  Synchronous D2D copy of `bytes` bytes into dst.
int sirius_debug_buffer(sirius_ctx* c, int rank, int which, void* dst, size_t bytes) {
  if (!c || rank < 0 || rank >= c->nranks) return -1;
  RankState& R = c->ranks[rank];
  const void* src[13] = {R.resA, R.resB, R.dA, R.dF, R.qkv, R.ob, R.xn3, R.k_cache, R.v_cache,
                         R.stage_k, R.stage_v, R.mb3, R.qb};
  if (which < 0 || which > 12) return -1;
  cudaStreamSynchronize(c->stream);
  return (int)cudaMemcpy(dst, src[which], bytes, cudaMemcpyDeviceToDevice);
}

// ---------------------------------------------------------------- test-only entry: the decode CATS FFN
// Runs layer `layer`'s decode FFN kernel (exactly the launch sparse_decode_step makes; rank 0's shard)
// on the residual rows x (DEV fp32 [batch, d]): h2 = RMSNorm(x), a = SiLU(h2 W_gate^T), CATS mask,
// out (DEV fp32 [batch, d]) = sum over active neurons of a_i (h2 . W_up[i]) W_down[i]; gate_out (DEV
// fp32 [batch, ffn/tp] or NULL) = a; n_active (DEV int32 [batch] or NULL).  Synchronous; returns a
// sirius_status.
int sirius_debug_ffn(sirius_ctx* c, int layer, const float* x, int dense, float* out, float* gate_out,
                     int32_t* n_active) {
  if (!c || !x || !out || layer < 0 || layer >= c->cfg.n_layers) return SIRIUS_ERR_INVALID_ARG;
  const int B = c->cfg.batch, d = c->cfg.d_model;
  CU(cudaMemsetAsync(out, 0, sizeof(float) * B * d, c->stream));
  if (n_active) CU(cudaMemsetAsync(n_active, 0, sizeof(int32_t) * B, c->stream));
  OK(launch_decode_ffn(c, c->ranks[0], layer, x, nullptr, nullptr, out, dense != 0, n_active, 1, gate_out, c->Fr));
  CU(cudaStreamSynchronize(c->stream));
  return SIRIUS_OK;
}

// ---------------------------------------------------------------- test-only entry: peer all-reduce skew
// adds delta to rank `rank`'s sync-point counter of the fused peer all-reduce (emulated / stub contexts):
// its next wait then expects a sequence number no peer will publish — the timeout path.  Synchronous.
int sirius_debug_par_skew(sirius_ctx* c, int rank, int delta) {
  if (!c || rank < 0 || rank >= (int)c->ranks.size() || !c->ranks[rank].par_seq) return -1;
  cudaStreamSynchronize(c->stream);
  unsigned long long v = 0;
  if (cudaMemcpy(&v, c->ranks[rank].par_seq, 8, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  v += (unsigned long long)(long long)delta;
  return cudaMemcpy(c->ranks[rank].par_seq, &v, 8, cudaMemcpyHostToDevice) == cudaSuccess ? 0 : -1;
}

// ---------------------------------------------------------------- test-only entry: top-k selection
// the exact top-k FSparse selection kernel (topk.cu) on B given gate pre-activation rows g [B, F]:
// a_out [B, F] = SiLU(g), mask [B, F / 32 + 1] = the k largest |a| (ties to the lower index).
// Synchronous.  Returns cudaError_t.
int sirius_debug_topk(const float* g, int F, int k, int B, float* a_out, unsigned* mask) {
  cudaError_t e = launch::topk_select(g, F, F, k, a_out, F, mask, F / 32 + 1, B, 0);
  if (e != cudaSuccess) return (int)e;
  return (int)cudaDeviceSynchronize();
}

// ---------------------------------------------------------------- test-only entry: the decode GEMV
// out[b, r] = sum_k W[r, k] h[b, k] through the decode GEMV kernel (the launch run_gemv makes); h = x (fp32 [B, K]), or with norm_w h = RMSNorm(x + delta) * norm_w
// (res_out = x + delta), or with embed h = RMSNorm(embed[tokens]) * norm_w (eps 1e-5); argmax (optional,
// DEV int32 [B]) = lowest-index argmax.
// Synchronous.  Returns cudaError_t.
int sirius_debug_gemv(const void* W, int rows, int K, const float* x, int B, float* out, int32_t* argmax,
                      const float* delta, const void* norm_w, float* res_out, const int32_t* tokens,
                      const void* embed, int vocab) {
  static unsigned long long* amax = nullptr;
  static unsigned* cnt = nullptr;
  if (!amax) {
    if (cudaMalloc(&amax, 64 * sizeof(unsigned long long)) || cudaMalloc(&cnt, 16 * sizeof(unsigned))) return -1;
    cudaMemset(amax, 0, 64 * sizeof(unsigned long long));
    cudaMemset(cnt, 0, 16 * sizeof(unsigned));
  }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  GemvArgs a = {};
  a.pro.mode = embed ? IN_EMBED : (norm_w ? IN_RESID : IN_F32);
  a.pro.in_f32 = x;
  a.pro.base = x;
  a.pro.delta = delta;
  a.pro.norm_w = static_cast<const uint16_t*>(norm_w);
  a.pro.eps = 1e-5f;
  a.pro.res_out = res_out;
  a.pro.tokens = tokens;
  a.pro.embed = static_cast<const uint16_t*>(embed);
  a.pro.vocab = vocab;
  a.W = static_cast<const uint16_t*>(W);
  a.rows = rows;
  a.K = K;
  a.epi = argmax ? EPI_ARGMAX : EPI_STORE;
  a.out = out;
  a.ldo = rows;
  a.amax = amax;
  a.finalize = 1;
  a.done_counter = cnt;
  a.token_out = argmax;
  cudaError_t e = launch::gemv(a, B, launch::gemv_grid(rows, sms), 0);
  if (e != cudaSuccess) return (int)e;
  return (int)cudaDeviceSynchronize();
}

// ---------------------------------------------------------------- test-only entry: the tcgen05 GEMM
// out[m, n] = sum_k sum_p X[p][m, k] W[n, k] (fp32), or (W2 != NULL) m = SiLU(x W^T) * (x W2^T) as three
// bf16 term planes out[3][M][N] (x = sum of the terms).  X: DEV bf16 [nterms][x_rows >= M][K] (term
// planes); W, W2: DEV bf16 [N, K].  Synchronous.  Returns cudaError_t.
int sirius_debug_gemm(const void* X, int nterms, int x_rows, const void* Wt, const void* W2, void* out, int M, int N,
                      int K) {
  static float* part = nullptr;
  static unsigned* cnt = nullptr;
  int dev = 0, sms = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (!part) {
    if (cudaMalloc(&part, launch::gemm_workspace_bytes(sms))) return -1;
    if (cudaMalloc(&cnt, 65536 * sizeof(unsigned))) return -1;
    cudaMemset(cnt, 0, 65536 * sizeof(unsigned));
  }
  if (const char* e = getenv("SIRIUS_GEMM_KBOX")) launch::g_gemm_kbox = atoi(e);
  if (const char* e = getenv("SIRIUS_GEMM_COARSE")) launch::g_gemm_coarse = atoi(e);
  GemmArgs g = {};
  g.N = N;
  g.K = K;
  g.M = M;
  g.n_tiles = (N + 127) / 128;
  g.kb = (K + 63) / 64;
  g.out = out;
  g.out_plane = (size_t)M * N;
  g.ldc = N;
  g.nterms = nterms;
  g.plane_rows = x_rows;
  g.part = part;
  g.counters = cnt;
  cudaError_t e = launch::gemm(Wt, W2, X, g, round_up(M, 16), sms, (size_t)optin - 1024, 0);
  if (e != cudaSuccess) return (int)e;
  return (int)cudaDeviceSynchronize();
}

}  // extern "C"
