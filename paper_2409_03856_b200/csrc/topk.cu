// topk.cu — top-k FSparse selection (PAPER.md:121 footnote "our implementation
// uses topk on the Gate Layer activations"; reading D30): per sequence, a = SiLU(g) of every neuron of
// the layer and the exact k = round(keep * ffn) largest |a| (ties to the lower neuron index).
// The gate pre-activations g come from the decode GEMV; the selected set goes to the CATS FFN kernel
// in its precomputed-gate mode (ffn_kernel with a_in / mask_in), which reads only the selected
// W_up / W_down rows.  Unlike the threshold rule the set depends on the whole layer, so it is
// computed here, between the gate GEMV and the up/down gathers.
#include "common.cuh"

namespace sirius {
namespace {

constexpr int kSelT = 1024;
constexpr int kMaxPer = 32;  // F <= kSelT * kMaxPer neurons per sequence (the rank's shard)

// one CTA per sequence: exact k-th largest |a| by a 4-pass 8-bit radix select over the non-negative
// float bit patterns, then the mask (all |a| > T, and the lowest-index ones == T up to k).
// The |a| bit patterns stay in registers (strided: element tid + kSelT j); the histogram is
// warp-aggregated (__match_any_sync: the top digits of |SiLU(g)| fall into a handful of bins, so
// per-element shared atomics would serialise), and the digit is found by one warp's suffix scan.
__global__ void __launch_bounds__(kSelT) topk_select_kernel(const float* __restrict__ g, long long ldg, int F, int k,
                                                           float* __restrict__ a_out, long long lda,
                                                           unsigned* __restrict__ mask, long long ldm) {
  __shared__ unsigned hist[256];
  __shared__ unsigned sel_s[2];  // selected digit, remaining rank
  __shared__ int warp_s[33];
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const float* gb = g + (size_t)b * ldg;
  float* ab = a_out + (size_t)b * lda;
  unsigned* mb = mask + (size_t)b * ldm;
  const int nper = (F + kSelT - 1) / kSelT;  // uniform over the block
  unsigned u[kMaxPer];
#pragma unroll
  for (int j = 0; j < kMaxPer; ++j) {
    const int i = tid + kSelT * j;
    u[j] = 0u;
    if (j < nper && i < F) {
      const float x = __ldg(gb + i);
      const float av = x / (1.0f + expf(-x));  // the CATS FFN kernel's SiLU
      ab[i] = av;
      u[j] = __float_as_uint(fabsf(av));
    }
  }
  for (int w = tid; w < (F + 31) / 32; w += kSelT) mb[w] = 0u;
  unsigned prefix = 0u, pmask = 0u;
  unsigned krem = (unsigned)k;
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    if (tid < 256) hist[tid] = 0u;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kMaxPer; ++j) {
      if (j < nper) {
        const int i = tid + kSelT * j;
        const bool ok = i < F && (u[j] & pmask) == prefix;
        const unsigned dg = ok ? (u[j] >> shift) & 255u : 256u;
        const unsigned peers = __match_any_sync(0xffffffffu, dg);
        if (ok && lane == __ffs(peers) - 1) atomicAdd(&hist[dg], (unsigned)__popc(peers));
      }
    }
    __syncthreads();
    if (warp == 0) {  // digit of the krem-th largest among the matching elements (from the top)
      unsigned c[8], tot = 0u;  // lane l: digits 255 - 8 l .. 248 - 8 l, descending
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        c[q] = hist[255 - 8 * lane - q];
        tot += c[q];
      }
      unsigned incl = tot;  // inclusive scan from the top digit down
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const unsigned excl = incl - tot;
      const unsigned hit = __ballot_sync(0xffffffffu, excl < krem && incl >= krem);
      if (lane == __ffs(hit) - 1) {
        unsigned acc = excl;
        int dsel = 255 - 8 * lane - 7;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (acc + c[q] >= krem) {
            dsel = 255 - 8 * lane - q;
            break;
          }
          acc += c[q];
        }
        sel_s[0] = (unsigned)dsel;
        sel_s[1] = krem - acc;
      }
    }
    __syncthreads();
    prefix |= sel_s[0] << shift;
    pmask |= 255u << shift;
    krem = sel_s[1];
  }
  const unsigned T = prefix;  // the k-th largest |a| (bits); krem = how many of the == T to keep
  // common case: exactly krem elements equal T -> keep every |a| >= T; the mask words come straight
  // from ballots (lanes of a warp hold 32 consecutive neurons of column j: word 32 j + warp)
  int n_eq = 0;
#pragma unroll
  for (int j = 0; j < kMaxPer; ++j)
    if (j < nper && tid + kSelT * j < F) n_eq += u[j] == T;
  n_eq = __reduce_add_sync(0xffffffffu, n_eq);
  if (lane == 0) warp_s[warp] = n_eq;
  __syncthreads();
  int tot_eq = 0;
  for (int w = 0; w < kSelT / 32; ++w) tot_eq += warp_s[w];
  if ((unsigned)tot_eq == krem) {
    const int nw = (F + 31) / 32;
#pragma unroll
    for (int j = 0; j < kMaxPer; ++j) {
      if (j < nper) {
        const int i = tid + kSelT * j;
        const unsigned word = __ballot_sync(0xffffffffu, i < F && u[j] >= T);
        if (lane == 0 && 32 * j + warp < nw) mb[32 * j + warp] = word;
      }
    }
    return;
  }
  __syncthreads();  // warp_s reuse
  // ties across the k boundary (rare): the lowest-index krem of the == T, by a scan in index order
  // (contiguous chunks per thread; ab was written by this block and is visible after the barriers)
  const int chunk = (F + kSelT - 1) / kSelT;
  const int i0 = min(F, tid * chunk), i1 = min(F, i0 + chunk);
  int c_eq = 0;
  for (int i = i0; i < i1; ++i) c_eq += __float_as_uint(fabsf(ab[i])) == T;
  int x = c_eq;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_s[warp] = x;
  __syncthreads();
  if (tid == 0) {
    int s = 0;
    for (int w = 0; w < kSelT / 32; ++w) {
      const int t = warp_s[w];
      warp_s[w] = s;
      s += t;
    }
  }
  __syncthreads();
  int eq_seen = warp_s[warp] + x - c_eq;
  for (int i = i0; i < i1; ++i) {
    const unsigned uu = __float_as_uint(fabsf(ab[i]));
    bool keep = uu > T;
    if (uu == T) keep = (unsigned)eq_seen++ < krem;
    if (keep) atomicOr(&mb[i >> 5], 1u << (i & 31));
  }
}

}  // namespace

namespace launch {
cudaError_t topk_select(const float* g, long long ldg, int F, int k, float* a_out, long long lda, unsigned* mask,
                        long long ldm, int B, cudaStream_t st) {
  if (F > kSelT * kMaxPer) return cudaErrorInvalidValue;
  topk_select_kernel<<<B, kSelT, 0, st>>>(g, ldg, F, k, a_out, lda, mask, ldm);
  return cudaGetLastError();
}
}  // namespace launch
}  // namespace sirius
