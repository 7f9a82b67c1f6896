// synth_gpu.cu — seeded synthetic-input generator (device side).
//
// Independent CUDA implementation of the recipe in synth/synth_cpu.c (same counter-based
// SplitMix64 / Irwin–Hall(4) / per-row gain / bf16-RNE steps, written again here, no shared code).
// Inputs only: no Sirius arithmetic lives in this file.  Used by the GPU tests and bench.py to
// materialise Llama-3-8B/70B-shaped weights directly in HBM (16–141 GB would be too slow to
// generate on the host).
#include <cstdint>
#include <cuda_runtime.h>

namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

struct GainTable {
  float g[49];
};

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ int32_t ih4(uint64_t r) {
  return (int32_t)(r & 0xFFFF) + (int32_t)((r >> 16) & 0xFFFF) + (int32_t)((r >> 32) & 0xFFFF) +
         (int32_t)((r >> 48) & 0xFFFF) - 131070;
}

__device__ __forceinline__ uint16_t bf16_rne_bits(float f) {
  uint32_t u = __float_as_uint(f);
  if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu)) return (uint16_t)((u >> 16) | 0x40u);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

__global__ void fill_bf16_kernel(uint64_t key, uint64_t ld, uint64_t row0, uint64_t col0, uint64_t ncols,
                                 uint64_t n, float scale, float offset, uint64_t gain_key, int32_t step,
                                 GainTable table, uint16_t* __restrict__ out) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t o = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; o < n; o += stride) {
    const uint64_t row = row0 + o / ncols;
    const uint64_t i = row * ld + col0 + o % ncols;  // index in the full tensor
    float s = scale;
    if (gain_key) {
      const int32_t z = ih4(mix64(gain_key + (row + 1) * kGolden)) + step / 2;
      int32_t k = z >= 0 ? z / step : -((-z + step - 1) / step);  // floor division
      k = k < -24 ? -24 : (k > 24 ? 24 : k);
      s = __fmul_rn(scale, table.g[k + 24]);
    }
    float prod = __fmul_rn((float)ih4(mix64(key + (i + 1) * kGolden)), s);  // never contracted into an FMA
    out[o] = bf16_rne_bits(__fadd_rn(prod, offset));
  }
}

__global__ void fill_tokens_kernel(uint64_t key, uint64_t n, int32_t vocab, int32_t* __restrict__ out) {
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = (int32_t)(mix64(key + (i + 1) * kGolden) % (uint64_t)vocab);
}

}  // namespace

extern "C" {

// Fill device buffer out ([nrows, ncols] row-major) with the sub-block rows [row0, row0+nrows) x
// cols [col0, col0+ncols) of the full tensor (seed, tensor_id) of row length ld.  gain_id != 0:
// per-row gain from the 49-entry fp32 table (host pointer).  Async on `stream`.
int synth_gpu_fill_bf16(uint64_t seed, uint64_t tensor_id, uint64_t ld, uint64_t row0, uint64_t nrows,
                        uint64_t col0, uint64_t ncols, float scale, float offset, uint64_t gain_id, int32_t step,
                        const float* table, void* out, void* stream) {
  uint64_t key = mix64(seed ^ mix64(tensor_id));
  uint64_t gain_key = gain_id ? mix64(seed ^ mix64(gain_id)) : 0;
  GainTable t = {};
  if (gain_id)
    for (int j = 0; j < 49; ++j) t.g[j] = table[j];
  uint64_t n = nrows * ncols;
  if (n == 0) return 0;
  int blocks = 148 * 8;
  fill_bf16_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(key, ld, row0, col0, ncols, n, scale, offset, gain_key,
                                                              step, t, (uint16_t*)out);
  return (int)cudaGetLastError();
}

int synth_gpu_fill_tokens(uint64_t seed, uint64_t stream_id, uint64_t n, int32_t vocab, int32_t* out,
                          void* stream) {
  uint64_t key = mix64(seed ^ mix64(0x70726F6D7074ULL ^ stream_id));
  if (n == 0) return 0;
  fill_tokens_kernel<<<64, 256, 0, (cudaStream_t)stream>>>(key, n, vocab, out);
  return (int)cudaGetLastError();
}

}  // extern "C"
