// sample.cu — temperature sampling of the drafted and the interleaved tokens (
// PAPER.md:253 / :267 "sample", :296 "the threshold of 0.1 and the temperature of 0.6 works well";
// reading D31).  The token placed at absolute position p of sequence b is drawn with the uniform
//   u = (splitmix64(seed ^ splitmix64(b * 2^32 + p)) >> 40) / 2^24        (24 bits, exact in fp32)
// by inverse CDF over the vocabulary in index order: the smallest v with sum_{w <= v} e_w > u Z,
// e_w = exp((l_w - max l) / temperature), Z = sum of all e_w.  The oracle implements the same
// counter-based generator and rule independently (oracle/sirius_oracle.py).
#include "common.cuh"

namespace sirius {
namespace {

constexpr int kST = 1024;

SIRIUS_DEV uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// one CTA per sequence b: row = b * rows_per_b + (jsel ? jsel[b] : 0), position p = base_pos[b] +
// (jsel ? jsel[b] : 0) + 1
__global__ void __launch_bounds__(kST) sample_kernel(const float* __restrict__ logits, int ldl, int V, float inv_temp,
                                                    unsigned long long seed, const int32_t* base_pos,
                                                    const int32_t* jsel, int rows_per_b, int32_t* out) {
  __shared__ float red_s[32];
  __shared__ float pre_s[kST];
  __shared__ int tok_s;
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int j = jsel ? jsel[b] : 0;
  const float* l = logits + (size_t)(b * rows_per_b + j) * ldl;
  const long long p = (long long)base_pos[b] + j + 1;
  float m = -INFINITY;
  for (int v = tid; v < V; v += kST) m = fmaxf(m, l[v]);
  m = warp_max(m);
  if (lane == 0) red_s[warp] = m;
  if (tid == 0) tok_s = -1;
  __syncthreads();
  float mx = -INFINITY;
  for (int w = 0; w < kST / 32; ++w) mx = fmaxf(mx, red_s[w]);
  const int chunk = (V + kST - 1) / kST;
  const int v0 = min(V, tid * chunk), v1 = min(V, v0 + chunk);
  float s = 0.f;
  for (int v = v0; v < v1; ++v) s += expf((l[v] - mx) * inv_temp);
  pre_s[tid] = s;
  __syncthreads();
  if (tid == 0) {  // exclusive prefix of the chunk sums, in order
    float acc = 0.f;
    for (int t = 0; t < kST; ++t) {
      const float x = pre_s[t];
      pre_s[t] = acc;
      acc += x;
    }
    red_s[0] = acc;
  }
  __syncthreads();
  const float Z = red_s[0];
  const uint64_t key = ((uint64_t)(uint32_t)b << 32) + (uint64_t)p;
  const float u = (float)(splitmix64(seed ^ splitmix64(key)) >> 40) * (1.0f / 16777216.0f);
  const float target = u * Z;
  float acc = pre_s[tid];
  if (acc <= target && acc + s > target) {
    for (int v = v0; v < v1; ++v) {
      acc += expf((l[v] - mx) * inv_temp);
      if (acc > target) {
        tok_s = v;
        break;
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    int t = tok_s;
    if (t < 0) {  // rounding put the target at the very end: the last token of nonzero weight
      t = V - 1;
      while (t > 0 && expf((l[t] - mx) * inv_temp) == 0.f) --t;
    }
    out[b] = t;
  }
}

}  // namespace

namespace launch {
cudaError_t sample_tokens(const float* logits, int ldl, int V, float temperature, unsigned long long seed,
                          const int32_t* base_pos, const int32_t* jsel, int rows_per_b, int32_t* out, int B,
                          cudaStream_t st) {
  sample_kernel<<<B, kST, 0, st>>>(logits, ldl, V, 1.0f / temperature, seed, base_pos, jsel, rows_per_b, out);
  return cudaGetLastError();
}
}  // namespace launch
}  // namespace sirius
