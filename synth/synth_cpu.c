/*
 * synth_cpu.c — seeded synthetic-input generator (host side).
 *
 * This module generates INPUTS only (weights, prompt tokens); it holds none of
 * the Sirius method's arithmetic.  It is the one piece of code that serves both
 * the CPU oracle (oracle/) and the GPU tests/bench: the GPU twin is
 * synth/synth_gpu.cu, an independent implementation of the same counter-based
 * recipe, and tests/test_synth.py checks the two agree bit for bit.
 *
 * Recipe (DESIGN.md §"Input recipe", SURVEY.md §8(d) "Weight generator"):
 *   key      = mix64(seed ^ mix64(tensor_id))
 *   r_i      = mix64(key + (i + 1) * GOLDEN)                 (SplitMix64 stream)
 *   z_i      = lane0 + lane1 + lane2 + lane3 - 131070         (Irwin–Hall(4) of u16 lanes, exact int)
 *   w_i      = bf16_rne( (float)z_i * scale + offset )       (fp32 multiply-add, then bf16 RNE)
 * `scale` and `offset` are fp32 constants supplied by the caller (fan-in scaled gain; see
 * synth/__init__.py).  No transcendental function is used, so every platform
 * produces the same bits.
 */
#include <stdint.h>
#include <string.h>
#include <pthread.h>

#define GOLDEN 0x9E3779B97F4A7C15ULL

static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static inline uint16_t f32_to_bf16_rne(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu)) return (uint16_t)((u >> 16) | 0x40u); /* NaN */
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

static inline int32_t irwin_hall4(uint64_t r) {
  return (int32_t)(r & 0xFFFF) + (int32_t)((r >> 16) & 0xFFFF) + (int32_t)((r >> 32) & 0xFFFF) +
         (int32_t)((r >> 48) & 0xFFFF) - 131070;
}

uint64_t synth_key(uint64_t seed, uint64_t tensor_id) { return mix64(seed ^ mix64(tensor_id)); }

/* Integer sample i of tensor (seed, tensor_id): exposed for tests. */
int32_t synth_irwin_hall(uint64_t seed, uint64_t tensor_id, uint64_t i) {
  return irwin_hall4(mix64(synth_key(seed, tensor_id) + (i + 1) * GOLDEN));
}

typedef struct {
  uint64_t key, ld, row0, col0, ncols, rbegin, rend;
  float scale, offset;
  uint16_t* out;
} fill_job;

static void* fill_worker(void* p) {
  fill_job* j = (fill_job*)p;
  for (uint64_t r = j->rbegin; r < j->rend; ++r)
    for (uint64_t c = 0; c < j->ncols; ++c) {
      uint64_t i = (j->row0 + r) * j->ld + j->col0 + c; /* index in the FULL (unsharded) tensor */
      int32_t z = irwin_hall4(mix64(j->key + (i + 1) * GOLDEN));
      volatile float prod = (float)z * j->scale; /* no contraction: one rounding, then the add */
      j->out[r * j->ncols + c] = f32_to_bf16_rne(prod + j->offset);
    }
  return 0;
}

/* Fill the sub-block rows [row0,row0+nrows) x cols [col0,col0+ncols) of the full tensor
 * (seed, tensor_id) whose row length is ld, into out (row-major [nrows, ncols], bf16 bits).
 * A 1-D tensor is ld = n, nrows = 1.  Threads: 1..64 (host cores). */
void synth_fill_bf16(uint64_t seed, uint64_t tensor_id, uint64_t ld, uint64_t row0, uint64_t nrows,
                     uint64_t col0, uint64_t ncols, float scale, float offset, uint16_t* out, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 64) threads = 64;
  if (nrows * ncols < (1u << 16) || nrows < (uint64_t)threads) threads = 1;
  pthread_t th[64];
  fill_job jobs[64];
  uint64_t key = synth_key(seed, tensor_id);
  for (int t = 0; t < threads; ++t) {
    jobs[t].key = key;
    jobs[t].ld = ld;
    jobs[t].row0 = row0;
    jobs[t].col0 = col0;
    jobs[t].ncols = ncols;
    jobs[t].rbegin = nrows * (uint64_t)t / (uint64_t)threads;
    jobs[t].rend = nrows * (uint64_t)(t + 1) / (uint64_t)threads;
    jobs[t].scale = scale;
    jobs[t].offset = offset;
    jobs[t].out = out;
  }
  if (threads == 1) { fill_worker(&jobs[0]); return; }
  for (int t = 0; t < threads; ++t) pthread_create(&th[t], 0, fill_worker, &jobs[t]);
  for (int t = 0; t < threads; ++t) pthread_join(th[t], 0);
}

/* Prompt tokens: tok[i] = mix64(key(seed, stream) + (i+1)*GOLDEN) mod vocab. */
void synth_fill_tokens(uint64_t seed, uint64_t stream, uint64_t n, int32_t vocab, int32_t* out) {
  uint64_t key = synth_key(seed, 0x70726F6D7074ULL ^ stream); /* "prompt" ^ stream */
  for (uint64_t i = 0; i < n; ++i) out[i] = (int32_t)(mix64(key + (i + 1) * GOLDEN) % (uint64_t)vocab);
}
