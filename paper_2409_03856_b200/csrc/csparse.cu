// csparse.cu — coarse-grained contextual sparsity (CSparse, Griffin-style):
// PAPER.md:62 (§2.1) "within the same input prompt, the sparsity pattern is fixed for all tokens
// generated", PAPER.md:182 (§3.2) the pattern is predetermined after prefilling, so the gate is
// sparsified too; PAPER.md:471 (Griffin is the sparse model of every latency number in the paper).
// Reading D28: statistic = sum over the prompt of |SiLU(g)| per neuron, keep
// k = round(keep * ffn) neurons per layer, exact ties to the lower neuron index.
//
//   colsum_abs_kernel    stats[n] += sum_m |a[m, n]|        (a = SiLU(g) of one prefill chunk, exported
//                        by the dual gate/up GEMM's epilogue; rows in order -> deterministic)
//   select_kernel        per layer: the k largest stats (exact k-th value by a bitwise search over the
//                        non-negative float bit patterns, ties to the lower index), ascending indices
//   gather_kernel        compact [k, d] copies of W_gate / W_up / W_down rows (the decode then runs
//                        the dense CATS FFN kernel on the compact matrices: HBM bytes = 3 k d)
#include "common.cuh"

namespace sirius {
namespace {

constexpr int kSelThreads = 1024;

__global__ void colsum_abs_kernel(const float* __restrict__ a, int M, int F, long long lda, float* __restrict__ stats) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= F) return;
  float s = stats[n];
  for (int m = 0; m < M; ++m) s += fabsf(a[(size_t)m * lda + n]);
  stats[n] = s;
}

// block-wide exclusive scan of one int per thread (1024 threads), returns the exclusive prefix;
// *total receives the sum
SIRIUS_DEV int block_exscan(int v, int* warp_s, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_s[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = warp_s[lane];
    int z = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, z, o);
      if (lane >= o) z += y;
    }
    warp_s[lane] = z - w;  // exclusive prefix of the warp totals
    if (lane == 31) warp_s[32] = z;
  }
  __syncthreads();
  const int r = warp_s[warp] + x - v;
  *total = warp_s[32];
  __syncthreads();
  return r;
}

// one CTA per layer: stats [L][F] (>= 0), idx [L][k] (ascending neuron indices of the kept set)
__global__ void __launch_bounds__(kSelThreads) select_kernel(const float* __restrict__ stats, int F, int k,
                                                             int32_t* __restrict__ idx) {
  __shared__ int warp_s[33];
  __shared__ unsigned cnt_s;
  const float* s = stats + (size_t)blockIdx.x * F;
  int32_t* out = idx + (size_t)blockIdx.x * k;
  const int tid = threadIdx.x;
  // the k-th largest value T (as bits; non-negative floats order like their bit patterns):
  // the largest T with count(s >= T) >= k, built bit by bit from the top
  unsigned T = 0u;
  for (int b = 30; b >= 0; --b) {  // bit 31 (sign) is 0 for every statistic
    const unsigned cand = T | (1u << b);
    if (tid == 0) cnt_s = 0u;
    __syncthreads();
    unsigned c = 0u;
    for (int i = tid; i < F; i += kSelThreads) c += __float_as_uint(s[i]) >= cand ? 1u : 0u;
    c = __reduce_add_sync(0xffffffffu, c);
    if ((tid & 31) == 0) atomicAdd(&cnt_s, c);
    __syncthreads();
    if (cnt_s >= (unsigned)k) T = cand;
    __syncthreads();
  }
  // kept: every s > T, and the lowest-index (k - count(s > T)) of the s == T
  const int chunk = (F + kSelThreads - 1) / kSelThreads;
  const int i0 = min(F, tid * chunk), i1 = min(F, i0 + chunk);
  int n_gt = 0, n_eq = 0;
  for (int i = i0; i < i1; ++i) {
    const unsigned u = __float_as_uint(s[i]);
    n_gt += u > T;
    n_eq += u == T;
  }
  int tot_gt, tot_eq, tot_kept;
  block_exscan(n_gt, warp_s, &tot_gt);
  const int eq_before = block_exscan(n_eq, warp_s, &tot_eq);
  const int need_eq = k - tot_gt;
  const int kept = n_gt + max(0, min(n_eq, need_eq - eq_before));
  int pos = block_exscan(kept, warp_s, &tot_kept);
  int eq_seen = eq_before;
  for (int i = i0; i < i1; ++i) {
    const unsigned u = __float_as_uint(s[i]);
    bool keep = u > T;
    if (u == T) keep = eq_seen++ < need_eq;
    if (keep) out[pos++] = i;
  }
}

// dst[j, :] = src[idx[j], :] for j < k (rows of d bf16), 16-byte copies
__global__ void gather_kernel(const uint16_t* __restrict__ src, const int32_t* __restrict__ idx, int k, int d,
                              uint16_t* __restrict__ dst) {
  const int cpr = d / 8;  // uint4 per row
  const size_t n = (size_t)k * cpr;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (size_t)gridDim.x * blockDim.x) {
    const size_t j = t / cpr, c = t % cpr;
    reinterpret_cast<uint4*>(dst)[t] = reinterpret_cast<const uint4*>(src + (size_t)idx[j] * d)[c];
  }
}

}  // namespace

namespace launch {

cudaError_t csparse_colsum(const float* a, int M, int F, long long lda, float* stats, cudaStream_t st) {
  colsum_abs_kernel<<<(F + 255) / 256, 256, 0, st>>>(a, M, F, lda, stats);
  return cudaGetLastError();
}

cudaError_t csparse_select(const float* stats, int L, int F, int k, int32_t* idx, cudaStream_t st) {
  select_kernel<<<L, kSelThreads, 0, st>>>(stats, F, k, idx);
  return cudaGetLastError();
}

cudaError_t csparse_gather(const uint16_t* src, const int32_t* idx, int k, int d, uint16_t* dst, int num_sms,
                           cudaStream_t st) {
  gather_kernel<<<2 * num_sms, 256, 0, st>>>(src, idx, k, d, dst);
  return cudaGetLastError();
}

}  // namespace launch
}  // namespace sirius
