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

// one CTA per sequence: exact k-th largest |a| by a 4-pass 8-bit radix select over the non-negative
// float bit patterns, then the mask (all |a| > T, and the lowest-index ones == T up to k)
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
  for (int i = tid; i < F; i += kSelT) {
    const float x = gb[i];
    ab[i] = x / (1.0f + expf(-x));  // the CATS FFN kernel's SiLU
  }
  for (int w = tid; w < (F + 31) / 32; w += kSelT) mb[w] = 0u;
  __syncthreads();
  unsigned prefix = 0u, pmask = 0u;
  unsigned krem = (unsigned)k;
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    for (int i = tid; i < 256; i += kSelT) hist[i] = 0u;
    __syncthreads();
    for (int i = tid; i < F; i += kSelT) {
      const unsigned u = __float_as_uint(fabsf(ab[i]));
      if ((u & pmask) == prefix) atomicAdd(&hist[(u >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid == 0) {  // digit of the krem-th largest among the matching elements (from the top)
      unsigned acc = 0u;
      int dsel = 0;
      for (int dgt = 255; dgt >= 0; --dgt) {
        if (acc + hist[dgt] >= krem) {
          dsel = dgt;
          break;
        }
        acc += hist[dgt];
      }
      sel_s[0] = (unsigned)dsel;
      sel_s[1] = krem - acc;
    }
    __syncthreads();
    prefix |= sel_s[0] << shift;
    pmask |= 255u << shift;
    krem = sel_s[1];
    __syncthreads();
  }
  const unsigned T = prefix;  // the k-th largest |a| (bits); krem = how many of the == T to keep
  // keep |a| > T, and the first krem (lowest index) == T: contiguous chunks per thread, scan of eq counts
  const int chunk = (F + kSelT - 1) / kSelT;
  const int i0 = min(F, tid * chunk), i1 = min(F, i0 + chunk);
  int n_eq = 0;
  for (int i = i0; i < i1; ++i) n_eq += __float_as_uint(fabsf(ab[i])) == T;
  int x = n_eq;
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
  int eq_seen = warp_s[warp] + x - n_eq;
  for (int i = i0; i < i1; ++i) {
    const unsigned u = __float_as_uint(fabsf(ab[i]));
    bool keep = u > T;
    if (u == T) keep = (unsigned)eq_seen++ < krem;
    if (keep) atomicOr(&mb[i >> 5], 1u << (i & 31));
  }
}

}  // namespace

namespace launch {
cudaError_t topk_select(const float* g, long long ldg, int F, int k, float* a_out, long long lda, unsigned* mask,
                        long long ldm, int B, cudaStream_t st) {
  topk_select_kernel<<<B, kSelT, 0, st>>>(g, ldg, F, k, a_out, lda, mask, ldm);
  return cudaGetLastError();
}
}  // namespace launch
}  // namespace sirius
