// tree.cu — hardware-friendly tree building and verification (PAPER.md:299-319
// §4.3; reading D29).  Batch 1.  The tree of a kernel of size gamma and width W is a fixed shape of
// 1 + (gamma-1) W flattened rows: row 0 = the pending token at position T, node w of step s = row
// 1 + (s-1) W + w at position T + s.  The sparse / full forwards run through the verify row machinery
// (tcgen05 GEMMs, attn_rows with ancestor masks); these kernels hold the tree's bookkeeping:
//
//   tree_init_kernel     row 0 <- the pending token
//   tree_topk_kernel     per logits row: log-sum-exp and the KB best (value, lowest index) entries
//   tree_prune_kernel    step s: expand each step-(s-1) node with its top-`branch` tokens (step 1: the
//                        root's top max(W, branch)), keep the W of largest cumulative log-likelihood,
//                        ties to the lower parent rank, then the lower token id ("a fixed number of
//                        leaves ... through tree pruning based on ranking the cumulative
//                        log-likelihood of the path")
//   tree_accept_kernel   q_n = softmax(full logits of the parent row)[token n] per node; per leaf the
//                        accepted prefix of its path (q >= r, or greedy match); the longest wins
//                        ("select the one that reaches the longest advance length"), ties to the higher
//                        leaf cumulative log-likelihood, then the lower leaf row; the interleaved token
//                        is the full model's argmax at the cut node; the winning path's rows are kept
//                        for the KV commit (kv_rewrite with a row list).
#include "common.cuh"
#include "tree.cuh"

namespace sirius {
namespace {

constexpr int kTopThreads = 1024;

__global__ void tree_init_kernel(TreeState* ts, const int32_t* pending) {
  if (threadIdx.x == 0) {
    ts->tok[0] = pending[0];
    ts->parent[0] = -1;
    ts->cum[0] = 0.f;
    ts->vis[0] = 1ull;
    ts->row_off[0] = 0;
  }
}

// one CTA per row: LSE and the KB largest entries as packed (value, lowest index) keys, descending
template <int KB>
__global__ void __launch_bounds__(kTopThreads) tree_topk_kernel(const float* __restrict__ logits, int ldl, int V,
                                                               TreeState* ts, int row_base) {
  __shared__ float red_s[32];
  __shared__ unsigned long long key_s[32];
  __shared__ unsigned long long win_s;
  const float* l = logits + (size_t)blockIdx.x * ldl;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // thread-local top KB (sorted descending) and max
  unsigned long long loc[KB];
#pragma unroll
  for (int k = 0; k < KB; ++k) loc[k] = 0ull;
  float mx = -INFINITY;
  for (int v = tid; v < V; v += kTopThreads) {
    const float x = l[v];
    mx = fmaxf(mx, x);
    unsigned long long key = argmax_key(x, (uint32_t)v);
#pragma unroll
    for (int k = 0; k < KB; ++k) {  // insertion into the sorted list
      if (key > loc[k]) {
        const unsigned long long t = loc[k];
        loc[k] = key;
        key = t;
      }
    }
  }
  mx = warp_max(mx);
  if (lane == 0) red_s[warp] = mx;
  __syncthreads();
  float m = -INFINITY;
  for (int w = 0; w < kTopThreads / 32; ++w) m = fmaxf(m, red_s[w]);
  __syncthreads();
  float se = 0.f;
  for (int v = tid; v < V; v += kTopThreads) se += expf(l[v] - m);
  se = warp_sum(se);
  if (lane == 0) red_s[warp] = se;
  __syncthreads();
  if (tid == 0) {
    float tot = 0.f;
    for (int w = 0; w < kTopThreads / 32; ++w) tot += red_s[w];
    ts->lse[row_base + blockIdx.x] = m + logf(tot);
  }
  // KB rounds of a block-wide max over the threads' current heads
  int head = 0;
  for (int k = 0; k < KB; ++k) {
    const unsigned long long mine = head < KB ? loc[head] : 0ull;
    const unsigned long long wm = warp_max_u64(mine);
    if (lane == 0) key_s[warp] = wm;
    __syncthreads();
    if (tid == 0) {
      unsigned long long best = 0ull;
      for (int w = 0; w < kTopThreads / 32; ++w) best = key_s[w] > best ? key_s[w] : best;
      win_s = best;
      ts->top[row_base + blockIdx.x][k] = best;
    }
    __syncthreads();
    if (head < KB && loc[head] == win_s && win_s != 0ull) ++head;  // keys are unique (index in the low bits)
    __syncthreads();
  }
}

SIRIUS_DEV float key_value(unsigned long long k) { return ordered_float((uint32_t)(k >> 32)); }

__global__ void tree_prune_kernel(TreeState* ts, int s, int W, int branch) {
  if (threadIdx.x != 0) return;
  const int np = s == 1 ? 1 : W;
  const int f0 = s == 1 ? 0 : 1 + (s - 2) * W;
  const int nb = s == 1 ? (W > branch ? W : branch) : branch;
  float cc[kTreeMaxW * kTreeMaxKB];
  int cp[kTreeMaxW * kTreeMaxKB], ct[kTreeMaxW * kTreeMaxKB];
  int n = 0;
  for (int pr = 0; pr < np; ++pr) {
    const int f = f0 + pr;
    for (int k = 0; k < nb; ++k) {
      const unsigned long long key = ts->top[f][k];
      cc[n] = ts->cum[f] + (key_value(key) - ts->lse[f]);
      cp[n] = pr;
      ct[n] = (int)argmax_key_index(key);
      ++n;
    }
  }
  unsigned taken[(kTreeMaxW * kTreeMaxKB + 31) / 32] = {};
  for (int w = 0; w < W; ++w) {  // W selections of the best remaining (cum desc, parent rank asc, token asc)
    int best = -1;
    for (int i = 0; i < n; ++i) {
      if ((taken[i / 32] >> (i % 32)) & 1u) continue;
      if (best < 0 || cc[i] > cc[best] || (cc[i] == cc[best] && (cp[i] < cp[best] || (cp[i] == cp[best] && ct[i] < ct[best]))))
        best = i;
    }
    taken[best / 32] |= 1u << (best % 32);
    const int row = 1 + (s - 1) * W + w, f = f0 + cp[best];
    ts->tok[row] = ct[best];
    ts->parent[row] = f;
    ts->cum[row] = cc[best];
    ts->vis[row] = ts->vis[f] | (1ull << row);
    ts->row_off[row] = s;
  }
}

__global__ void tree_accept_kernel(const float* __restrict__ logits, int ldl, TreeState* ts, int S, int W, float r,
                                   int mode, int32_t* n_accept, int32_t* next_token, int32_t* path_tokens, int gamma) {
  __shared__ unsigned char ok_s[kTreeMaxRows];
  const int n_rows = 1 + S * W;
  for (int n = 1 + threadIdx.x; n < n_rows; n += blockDim.x) {
    const int p = ts->parent[n], t = ts->tok[n];
    bool ok;
    if (mode == 0) {
      const float q = expf(logits[(size_t)p * ldl + t] - ts->lse[p]);
      ts->q[n] = q;
      ok = q >= r;
    } else {
      ok = t == (int)argmax_key_index(ts->top[p][0]);
    }
    ok_s[n] = ok ? 1 : 0;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  int best_leaf = -1, best_acc = -1;
  float best_cum = 0.f;
  int chain[kTreeMaxRows];
  for (int w = 0; w < W; ++w) {
    const int leaf = S > 0 ? 1 + (S - 1) * W + w : 0;
    int len = 0;
    for (int x = leaf; x > 0; x = ts->parent[x]) chain[len++] = x;  // leaf .. step-1 node
    int acc = 0;
    for (int i = len - 1; i >= 0 && ok_s[chain[i]]; --i) ++acc;
    if (best_leaf < 0 || acc > best_acc || (acc == best_acc && ts->cum[leaf] > best_cum)) {
      best_leaf = leaf;
      best_acc = acc;
      best_cum = ts->cum[leaf];
    }
    if (S == 0) break;
  }
  int len = 0;
  for (int x = best_leaf; x > 0; x = ts->parent[x]) chain[len++] = x;
  ts->path[0] = 0;
  for (int i = 0; i < best_acc; ++i) ts->path[1 + i] = chain[len - 1 - i];
  for (int i = 0; i < gamma; ++i) path_tokens[i] = i <= best_acc ? ts->tok[ts->path[i]] : -1;
  n_accept[0] = best_acc;
  next_token[0] = (int32_t)argmax_key_index(ts->top[ts->path[best_acc]][0]);
}

}  // namespace

namespace launch {

cudaError_t tree_init(TreeState* ts, const int32_t* pending, cudaStream_t st) {
  tree_init_kernel<<<1, 32, 0, st>>>(ts, pending);
  return cudaGetLastError();
}

cudaError_t tree_topk(const float* logits, int ldl, int V, int rows, int kb, TreeState* ts, int row_base,
                      cudaStream_t st) {
  if (kb <= 1) tree_topk_kernel<1><<<rows, kTopThreads, 0, st>>>(logits, ldl, V, ts, row_base);
  else if (kb <= 4) tree_topk_kernel<4><<<rows, kTopThreads, 0, st>>>(logits, ldl, V, ts, row_base);
  else tree_topk_kernel<8><<<rows, kTopThreads, 0, st>>>(logits, ldl, V, ts, row_base);
  return cudaGetLastError();
}

cudaError_t tree_prune(TreeState* ts, int s, int W, int branch, cudaStream_t st) {
  tree_prune_kernel<<<1, 32, 0, st>>>(ts, s, W, branch);
  return cudaGetLastError();
}

cudaError_t tree_accept(const float* logits, int ldl, TreeState* ts, int S, int W, float r, int mode, int32_t* n_accept,
                        int32_t* next_token, int32_t* path_tokens, int gamma, cudaStream_t st) {
  tree_accept_kernel<<<1, 64, 0, st>>>(logits, ldl, ts, S, W, r, mode, n_accept, next_token, path_tokens, gamma);
  return cudaGetLastError();
}

}  // namespace launch
}  // namespace sirius
