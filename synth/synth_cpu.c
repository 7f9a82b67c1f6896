/*
 * synth_cpu.c — seeded synthetic-input generator (host side).
 *
 * This module generates INPUTS only (weights, prompt tokens); it holds none of
 * the Sirius method's arithmetic.  It is the one piece of code that serves both
 * the CPU oracle (oracle/) and the GPU tests/bench: the GPU twin is
 * synth/synth_gpu.cu, an independent implementation of the same counter-based
 * recipe, and tests/test_synth.py checks the two agree bit for bit.
 *
 * Recipe (DESIGN.md §3 "Input recipe"):
 *   key(t)   = mix64(seed ^ mix64(t))
 *   IH(t, i) = sum of the four u16 lanes of mix64(key(t) + (i + 1) * GOLDEN) - 131070
 *              (Irwin–Hall(4), an exact integer, std 65536/sqrt(3))
 *   row gain (optional, W_gate / W_up): k_r = clamp(floor_div(IH(gain_id, r) + step/2, step), -24, 24),
 *              scale_r = fp32(scale * gain_table[k_r + 24])       (gain_table[j] = fp32(2^((j-24)/4)))
 *   w[r][c]  = bf16_rne( fp32(IH(tensor_id, r*ld + c) * scale_r) + offset )
 * Only integer ops and fp32 multiply/add (no contraction, no transcendental), so every platform
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

static inline int32_t floor_div(int32_t a, int32_t b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

/* Gain index k in [-24, 24] of row r (quarter octaves): exposed for tests and threshold recipes. */
int32_t synth_row_gain_k(uint64_t seed, uint64_t gain_id, uint64_t r, int32_t step) {
  int32_t k = floor_div(synth_irwin_hall(seed, gain_id, r) + step / 2, step);
  return k < -24 ? -24 : (k > 24 ? 24 : k);
}

void synth_row_gain_ks(uint64_t seed, uint64_t gain_id, uint64_t n, int32_t step, int8_t* out) {
  for (uint64_t r = 0; r < n; ++r) out[r] = (int8_t)synth_row_gain_k(seed, gain_id, r, step);
}

typedef struct {
  uint64_t key, ld, row0, col0, ncols, rbegin, rend, seed, gain_id;
  float scale, offset;
  int32_t step;
  const float* table;
  uint16_t* out;
} fill_job;

static void* fill_worker(void* p) {
  fill_job* j = (fill_job*)p;
  for (uint64_t r = j->rbegin; r < j->rend; ++r) {
    volatile float sc = j->scale;
    if (j->gain_id) {
      int32_t k = synth_row_gain_k(j->seed, j->gain_id, j->row0 + r, j->step);
      sc = j->scale * j->table[k + 24];
    }
    const float s = sc;
    for (uint64_t c = 0; c < j->ncols; ++c) {
      uint64_t i = (j->row0 + r) * j->ld + j->col0 + c; /* index in the FULL (unsharded) tensor */
      int32_t z = irwin_hall4(mix64(j->key + (i + 1) * GOLDEN));
      volatile float prod = (float)z * s; /* no contraction: one rounding, then the add */
      j->out[r * j->ncols + c] = f32_to_bf16_rne(prod + j->offset);
    }
  }
  return 0;
}

/* Fill the sub-block rows [row0,row0+nrows) x cols [col0,col0+ncols) of the full tensor
 * (seed, tensor_id) whose row length is ld, into out (row-major [nrows, ncols], bf16 bits).
 * gain_id != 0 applies the per-row gain (table: 49 fp32 values, step: IH units per quarter octave).
 * A 1-D tensor is ld = n, nrows = 1.  Threads: 1..64 (host cores). */
void synth_fill_bf16(uint64_t seed, uint64_t tensor_id, uint64_t ld, uint64_t row0, uint64_t nrows,
                     uint64_t col0, uint64_t ncols, float scale, float offset, uint64_t gain_id, int32_t step,
                     const float* table, uint16_t* out, int threads) {
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
    jobs[t].seed = seed;
    jobs[t].gain_id = gain_id;
    jobs[t].step = step;
    jobs[t].table = table;
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
