// decode_kernels.cu — bandwidth-bound decode kernels for sm_100a.
//
//  * gemv_stream_kernel   : row-streaming GEMV.  One elected producer lane streams whole weight rows
//                           (d*2 bytes, contiguous) HBM -> shared memory with 1-D bulk async copies
//                           (cp.async.bulk, the TMA engine) into an mbarrier ring; consumer warps
//                           compute warp-shuffle dot products.  Prologue fuses residual add +
//                           RMSNorm (or the embedding gather); epilogues: store, or packed argmax.
//  * ffn_fused_kernel     : the CATS-sparse MLP of one layer in one
//                           cooperative launch: dense gate GEMV + SiLU + per-layer magnitude
//                           threshold + warp-ballot compaction of each 32-neuron chunk, then only
//                           the ACTIVE rows of W_up and W_down are streamed (HBM bytes scale with
//                           density); grid barrier; deterministic column reduction of the per-CTA
//                           partial down-projections.
//  * attn_decode_kernel   : RoPE of q/k, K/V append at pos, split-K flash-decode over the cache,
//                           last-arriving CTA combines the splits.
// Numeric contract (D15): bf16 weights and bf16 KV-cache storage (k after RoPE, v);
// every activation fp32 (residual, RMSNorm outputs, q, attention output, g, a, u, m, scores,
// softmax, logits), fp32 accumulation.
#include "common.cuh"
#include "decode_kernels.cuh"

namespace sirius {

// consumer-only named barrier (the producer warp never joins)
SIRIUS_DEV void cbar(int nthreads) { asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory"); }

// Prologue: build the fp32 activation rows h[b, 0:K) in shared memory.  Executed by the NT
// consumer threads only.  Deterministic fixed-order reductions.
template <int B>
SIRIUS_DEV void run_prologue(const Prologue& p, int K, float* h_s, float* red_s, int tid, int NT, bool store_res) {
  const int nwarp = NT / 32, warp = tid / 32, lane = tid % 32;
  if (p.mode == IN_F32) {
    const float4* src = reinterpret_cast<const float4*>(p.in_f32);
    float4* dst = reinterpret_cast<float4*>(h_s);
    for (int i = tid; i < B * K / 4; i += NT) dst[i] = src[i];
    cbar(NT);
    return;
  }
  for (int b = 0; b < B; ++b) {
    const float* base = p.mode == IN_RESID ? p.base + (size_t)b * K : nullptr;
    const float* delta = (p.mode == IN_RESID && p.delta) ? p.delta + (size_t)b * K : nullptr;
    const uint16_t* erow = nullptr;
    if (p.mode == IN_EMBED) {
      int tok = p.tokens[b];
      tok = tok < 0 ? 0 : (tok >= p.vocab ? p.vocab - 1 : tok);
      erow = p.embed + (size_t)tok * K;
    }
    auto xval = [&](int k) -> float {
      if (erow) return __uint_as_float((uint32_t)erow[k] << 16);
      float v = base[k];
      if (delta) v += delta[k];
      return v;
    };
    float ss = 0.f;
    for (int k = tid; k < K; k += NT) {
      float v = xval(k);
      ss = fmaf(v, v, ss);
      if (store_res && p.res_out) p.res_out[(size_t)b * K + k] = v;
    }
    ss = warp_sum(ss);
    if (lane == 0) red_s[warp] = ss;
    cbar(NT);
    float tot = 0.f;
    for (int w = 0; w < nwarp; ++w) tot += red_s[w];
    const float r = 1.0f / sqrtf(tot / (float)K + p.eps);
    for (int k = tid; k < K; k += NT) {
      float w = __uint_as_float((uint32_t)p.norm_w[k] << 16);
      h_s[(size_t)b * K + k] = (xval(k) * r) * w;
    }
    cbar(NT);  // red_s reuse + h_s complete
  }
}

// consumer-only "last CTA" election (see arrive_last in common.cuh)
SIRIUS_DEV bool arrive_last_c(unsigned* counter, unsigned n, int tid, int NT, unsigned* flag_s) {
  cbar(NT);
  if (tid == 0) {
    __threadfence();
    unsigned old = atomicAdd(counter, 1u);
    bool last = old == n - 1;
    if (last) {
      atomicExch(counter, 0u);
      __threadfence();
    }
    *flag_s = last ? 1u : 0u;
  }
  cbar(NT);
  return *flag_s != 0;
}

// ===================================================================== streaming GEMV
template <int B, int NW>
__global__ void __launch_bounds__((NW + 1) * 32, 1) gemv_stream_kernel(GemvArgs a, int nslot) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int NT = NW * 32;
  const int K = a.K, rowbytes = K * 2;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  uint8_t* ring = smem;
  float* h_s = reinterpret_cast<float*>(smem + (size_t)nslot * rowbytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(h_s + (size_t)B * K);
  uint64_t* empty = full + nslot;
  float* red_s = reinterpret_cast<float*>(empty + nslot);
  unsigned long long* key_s = reinterpret_cast<unsigned long long*>(red_s + 32);  // [NW][B]
  unsigned* flag_s = reinterpret_cast<unsigned*>(key_s + NW * B);

  const int r0 = (int)((long long)a.rows * blockIdx.x / gridDim.x);
  const int r1 = (int)((long long)a.rows * (blockIdx.x + 1) / gridDim.x);
  const int nrows = r1 - r0;

  if (tid == 0) {
    for (int i = 0; i < nslot; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == NW) {  // ---------------- producer: stream rows [r0, r1) through the ring
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      for (int i = 0; i < nrows; ++i) {
        const int slot = i % nslot;
        const uint32_t ph = (uint32_t)(i / nslot) & 1u;
        mbar_wait(&empty[slot], ph ^ 1u);
        mbar_arrive_expect_tx(&full[slot], rowbytes);
        bulk_g2s(ring + (size_t)slot * rowbytes, a.W + (size_t)(r0 + i) * K, rowbytes, &full[slot], pol);
      }
    }
    return;
  }

  // ---------------- consumers
  run_prologue<B>(a.pro, K, h_s, red_s, tid, NT, blockIdx.x == 0);
  unsigned long long best[B];
#pragma unroll
  for (int b = 0; b < B; ++b) best[b] = 0ull;
  const int nch = K / 8;
  for (int i = warp; i < nrows; i += NW) {
    const int slot = i % nslot;
    mbar_wait(&full[slot], (uint32_t)(i / nslot) & 1u);
    const uint4* w = reinterpret_cast<const uint4*>(ring + (size_t)slot * rowbytes);
    float acc[B];
#pragma unroll
    for (int b = 0; b < B; ++b) acc[b] = 0.f;
#pragma unroll 4
    for (int c = lane; c < nch; c += 32) {
      const uint4 wv = w[c];
#pragma unroll
      for (int b = 0; b < B; ++b) acc[b] += dot8(wv, h_s + (size_t)b * K + c * 8);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
#pragma unroll
    for (int b = 0; b < B; ++b) acc[b] = warp_sum(acc[b]);
    const int row = r0 + i;
    if (lane == 0) {
#pragma unroll
      for (int b = 0; b < B; ++b) {
        if (a.out) a.out[(size_t)b * a.ldo + row] = acc[b];
        if (a.epi == EPI_ARGMAX) {
          unsigned long long k = argmax_key(acc[b], a.index_offset + (uint32_t)row);
          best[b] = k > best[b] ? k : best[b];
        }
      }
    }
  }
  if (a.epi != EPI_ARGMAX) return;
  if (lane == 0)
    for (int b = 0; b < B; ++b) key_s[warp * B + b] = best[b];
  cbar(NT);
  if (tid < B) {
    unsigned long long k = 0ull;
    for (int w = 0; w < NW; ++w) k = key_s[w * B + tid] > k ? key_s[w * B + tid] : k;
    atomicMax(a.amax + tid, k);
  }
  if (a.finalize) {
    if (arrive_last_c(a.done_counter, gridDim.x, tid, NT, flag_s)) {
      if (tid < B) {
        unsigned long long k = atomicExch(a.amax + tid, 0ull);  // read + reset for the next step
        a.token_out[tid] = (int32_t)argmax_key_index(k);
      }
    }
  }
}

// amax -> token (after a cross-rank max of the packed keys); resets amax.
__global__ void argmax_finalize_kernel(unsigned long long* amax, int B, int32_t* token_out) {
  int b = threadIdx.x;
  if (b < B) {
    unsigned long long k = amax[b];
    amax[b] = 0ull;
    token_out[b] = (int32_t)argmax_key_index(k);
  }
}

// ===================================================================== fused CATS FFN
constexpr int kFfnMaxChunks = 8;  // <= 256 neurons per CTA
constexpr int kFfnMaxN = kFfnMaxChunks * 32;

template <int B, int NW, int CPT>
__global__ void __launch_bounds__((NW + 1) * 32, 1) ffn_fused_kernel(FfnArgs a, int nslot) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int NT = NW * 32;
  const int d = a.d, rowbytes = d * 2;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int G = gridDim.x, cta = blockIdx.x;
  const int n0 = (int)((long long)a.F * cta / G), n1 = (int)((long long)a.F * (cta + 1) / G);
  const int nch = (n1 - n0 + 31) / 32;

  uint8_t* ring = smem;
  float* h_s = reinterpret_cast<float*>(smem + (size_t)nslot * rowbytes);        // [B][d]
  float* a_s = reinterpret_cast<float*>(h_s + (size_t)B * d);                    // [B][kFfnMaxN]
  float* m_s = a_s + B * kFfnMaxN;                                                // [B][32]
  float* red_s = m_s + B * 32;                                                    // [32]
  int* list_s = reinterpret_cast<int*>(red_s + 32);                               // [kFfnMaxChunks][32]
  unsigned* act_s = reinterpret_cast<unsigned*>(list_s + kFfnMaxN);               // [kFfnMaxChunks][B]
  int* cnt_s = reinterpret_cast<int*>(act_s + kFfnMaxChunks * B);                 // [kFfnMaxChunks]
  int* nact_s = cnt_s + kFfnMaxChunks;                                            // [B]
  uint64_t* full = reinterpret_cast<uint64_t*>(((uintptr_t)(nact_s + B) + 15) & ~(uintptr_t)15);
  uint64_t* empty = full + nslot;
  uint64_t* listbar = empty + nslot;  // [kFfnMaxChunks]

  if (tid == 0) {
    for (int i = 0; i < nslot; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NW);  // single-warp consumers arrive with count NW, all-warp consumers with 1
    }
    for (int c = 0; c < kFfnMaxChunks; ++c) mbar_init(&listbar[c], 1);
    for (int b = 0; b < B; ++b) nact_s[b] = 0;
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == NW) {  // ---------------- producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int op = 0;
      auto issue = [&](const uint16_t* src) {
        const int slot = op % nslot;
        mbar_wait(&empty[slot], ((uint32_t)(op / nslot) & 1u) ^ 1u);
        mbar_arrive_expect_tx(&full[slot], rowbytes);
        bulk_g2s(ring + (size_t)slot * rowbytes, src, rowbytes, &full[slot], pol);
        ++op;
      };
      // order: G0, G1, U0, D0, G2, U1, D1, ...: the next chunk's gate rows are in flight while the
      // consumers threshold the current chunk, so the ring never drains at a chunk boundary.
      for (int s = 0; s <= nch; ++s) {
        if (s < nch) {
          const int nb = n0 + s * 32, ne = min(n1, nb + 32);
          for (int n = nb; n < ne; ++n) issue(a.w_gate + (size_t)n * d);
        }
        if (s >= 1) {
          const int c = s - 1;
          mbar_wait(&listbar[c], 0);
          const int cnt = cnt_s[c];
          for (int k = 0; k < cnt; ++k) issue(a.w_up + (size_t)list_s[c * 32 + k] * d);
          for (int k = 0; k < cnt; ++k) issue(a.w_down + (size_t)list_s[c * 32 + k] * d);
        }
      }
    }
    return;
  }

  // ---------------- consumers
  run_prologue<B>(a.pro, d, h_s, red_s, tid, NT, cta == 0);
  const float t = a.dense ? 0.f : *a.threshold;
  float y[B][CPT * 8];
#pragma unroll
  for (int b = 0; b < B; ++b)
#pragma unroll
    for (int e = 0; e < CPT * 8; ++e) y[b][e] = 0.f;
  const int nchunk16 = d / 8;
  int op = 0;
  for (int s = 0; s <= nch; ++s) {
    if (s < nch) {
      const int nb = n0 + s * 32, ne = min(n1, nb + 32), rows = ne - nb;
      // ---- gate rows (dense): g = h2 . W_gate[n];  a = SiLU(g)
      for (int r = warp; r < rows; r += NW) {
        const int o = op + r, slot = o % nslot;
        mbar_wait(&full[slot], (uint32_t)(o / nslot) & 1u);
        const uint4* w = reinterpret_cast<const uint4*>(ring + (size_t)slot * rowbytes);
        float acc[B];
#pragma unroll
        for (int b = 0; b < B; ++b) acc[b] = 0.f;
#pragma unroll 4
        for (int c = lane; c < nchunk16; c += 32) {
          const uint4 wv = w[c];
#pragma unroll
          for (int b = 0; b < B; ++b) acc[b] += dot8(wv, h_s + (size_t)b * d + c * 8);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot], NW);
#pragma unroll
        for (int b = 0; b < B; ++b) {
          const float g = warp_sum(acc[b]);
          if (lane == 0) a_s[b * kFfnMaxN + s * 32 + r] = g / (1.0f + expf(-g));  // SiLU
        }
      }
      op += rows;
      cbar(NT);
      // ---- CATS threshold + warp-ballot compaction (every warp derives the same masks)
      const bool valid = lane < rows;
      unsigned um = 0u;
      unsigned mb[B];
      float av[B];
#pragma unroll
      for (int b = 0; b < B; ++b) {
        av[b] = valid ? a_s[b * kFfnMaxN + s * 32 + lane] : 0.f;
        const bool act = valid && (a.dense || fabsf(av[b]) >= t);
        mb[b] = __ballot_sync(0xffffffffu, act);
        um |= mb[b];
      }
      if (warp == 0) {
        if ((um >> lane) & 1u) list_s[s * 32 + __popc(um & ((1u << lane) - 1u))] = nb + lane;
        if (a.gate_out && valid)
          for (int b = 0; b < B; ++b) a.gate_out[(size_t)b * a.gate_stride + nb + lane] = av[b];
        if (lane == 0) {
          cnt_s[s] = __popc(um);
          for (int b = 0; b < B; ++b) {
            act_s[s * B + b] = mb[b];
            nact_s[b] += __popc(mb[b]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&listbar[s]);  // release: the producer may now gather this chunk
      }
    }
    if (s >= 1) {
      const int c = s - 1, cb = n0 + c * 32;
      cbar(NT);  // list_s[c], act_s[c] visible; every warp is done with the previous D loop (m_s)
      const int cnt = cnt_s[c];
      // ---- up rows (active only): u = h2 . W_up[n];  m = a * u
      for (int k = warp; k < cnt; k += NW) {
        const int o = op + k, slot = o % nslot;
        mbar_wait(&full[slot], (uint32_t)(o / nslot) & 1u);
        const uint4* w = reinterpret_cast<const uint4*>(ring + (size_t)slot * rowbytes);
        float acc[B];
#pragma unroll
        for (int b = 0; b < B; ++b) acc[b] = 0.f;
#pragma unroll 4
        for (int ch = lane; ch < nchunk16; ch += 32) {
          const uint4 wv = w[ch];
#pragma unroll
          for (int b = 0; b < B; ++b) acc[b] += dot8(wv, h_s + (size_t)b * d + ch * 8);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot], NW);
        const int nl = list_s[c * 32 + k] - cb;
#pragma unroll
        for (int b = 0; b < B; ++b) {
          const float u = warp_sum(acc[b]);
          if (lane == 0) {
            const bool act = (act_s[c * B + b] >> nl) & 1u;
            m_s[b * 32 + k] = act ? a_s[b * kFfnMaxN + c * 32 + nl] * u : 0.f;
          }
        }
      }
      op += cnt;
      cbar(NT);  // m_s complete
      // ---- down rows (active only): y += m * W_down[n]   (every warp owns a column slice)
      for (int k = 0; k < cnt; ++k) {
        const int o = op + k, slot = o % nslot;
        mbar_wait(&full[slot], (uint32_t)(o / nslot) & 1u);
        const uint4* w = reinterpret_cast<const uint4*>(ring + (size_t)slot * rowbytes);
        float mk[B];
#pragma unroll
        for (int b = 0; b < B; ++b) mk[b] = m_s[b * 32 + k];
#pragma unroll
        for (int j = 0; j < CPT; ++j) {
          const int ch = tid + j * NT;
          if (ch < nchunk16) {
            const uint4 wv = w[ch];
            const float wf[8] = {bf16_lo(wv.x), bf16_hi(wv.x), bf16_lo(wv.y), bf16_hi(wv.y),
                                 bf16_lo(wv.z), bf16_hi(wv.z), bf16_lo(wv.w), bf16_hi(wv.w)};
#pragma unroll
            for (int b = 0; b < B; ++b)
#pragma unroll
              for (int e = 0; e < 8; ++e) y[b][j * 8 + e] = fmaf(mk[b], wf[e], y[b][j * 8 + e]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot], 1);
      }
      op += cnt;
    }
  }
  // ---- per-CTA partials -> grid barrier -> deterministic column reduction
#pragma unroll
  for (int j = 0; j < CPT; ++j) {
    const int ch = tid + j * NT;
    if (ch < nchunk16) {
#pragma unroll
      for (int b = 0; b < B; ++b) {
        float4* dst = reinterpret_cast<float4*>(a.part + ((size_t)cta * B + b) * d + ch * 8);
        dst[0] = make_float4(y[b][j * 8 + 0], y[b][j * 8 + 1], y[b][j * 8 + 2], y[b][j * 8 + 3]);
        dst[1] = make_float4(y[b][j * 8 + 4], y[b][j * 8 + 5], y[b][j * 8 + 6], y[b][j * 8 + 7]);
      }
    }
  }
  if (tid < B) a.part_cnt[cta * B + tid] = nact_s[tid];
  cbar(NT);
  if (tid == 0) {
    __threadfence();
    unsigned long long old = atomicAdd(a.barrier, 1ull);
    const unsigned long long target = (old / (unsigned)G + 1) * (unsigned)G;
    while (ld_acquire_u64(a.barrier) < target) __nanosleep(32);
    __threadfence();
  }
  cbar(NT);
  const int units = B * d / 4;  // float4 columns
  const int u0 = (int)((long long)units * cta / G), u1 = (int)((long long)units * (cta + 1) / G);
  for (int u = u0 + warp; u < u1; u += NW) {
    const int b = u / (d / 4), c4 = u % (d / 4);
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int p = lane; p < G; p += 32) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(a.part + ((size_t)p * B + b) * d) + c4);
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    s.x = warp_sum(s.x); s.y = warp_sum(s.y); s.z = warp_sum(s.z); s.w = warp_sum(s.w);
    if (lane == 0) reinterpret_cast<float4*>(a.out + (size_t)b * d)[c4] = s;
  }
  if (cta == 0 && a.n_active_out && tid < B) {
    int tot = 0;
    for (int p = 0; p < G; ++p) tot += __ldcg(a.part_cnt + p * B + tid);
    a.n_active_out[(size_t)tid * a.n_active_stride] = tot;
  }
}

// ===================================================================== decode attention
template <int HD, int G>
__global__ void __launch_bounds__(128) attn_decode_kernel(AttnArgs a, float scale) {
  constexpr int EPL = HD / 32;
  const int split = blockIdx.x, kvh = blockIdx.y, b = blockIdx.z;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  __shared__ float q_s[G][HD];
  __shared__ float kn_s[HD], vn_s[HD];
  __shared__ float wm[4][G], wl[4][G];
  __shared__ float wacc[4][G][HD];

  const int S = a.splits, Hr = a.Hr, KVr = a.KVr;
  const int qkv_stride = (Hr + 2 * KVr) * HD;
  int pos = a.pos[b];
  const bool bad = pos < 0 || pos >= a.max_seq;
  if (bad) {
    if (tid == 0 && split == 0) atomicOr(a.err, 1);
    pos = 0;
  }
  const int nkeys = bad ? 0 : pos + 1;
  const int chunk = (nkeys + S - 1) / S;
  const int k0 = min(nkeys, split * chunk), k1 = min(nkeys, k0 + chunk);

  // RoPE (rotate-half) on q and k at position pos; k (and v) rounded to bf16 as stored in the cache
  const float* qkv = a.qkv + (size_t)b * qkv_stride;
  const float* cs = a.rope_cos + (size_t)pos * (HD / 2);
  const float* sn = a.rope_sin + (size_t)pos * (HD / 2);
  for (int idx = tid; idx < G * (HD / 2); idx += 128) {
    const int g = idx / (HD / 2), i = idx % (HD / 2);
    const float* q = qkv + (kvh * G + g) * HD;
    const float x0 = q[i], x1 = q[i + HD / 2], c = cs[i], s = sn[i];
    q_s[g][i] = x0 * c - x1 * s;
    q_s[g][i + HD / 2] = x1 * c + x0 * s;
  }
  if (tid < HD / 2) {
    const float* k = qkv + (Hr + kvh) * HD;
    const float x0 = k[tid], x1 = k[tid + HD / 2], c = cs[tid], s = sn[tid];
    kn_s[tid] = round_bf16(x0 * c - x1 * s);
    kn_s[tid + HD / 2] = round_bf16(x1 * c + x0 * s);
  }
  for (int i = tid; i < HD; i += 128) vn_s[i] = round_bf16(qkv[(Hr + KVr + kvh) * HD + i]);
  __syncthreads();
  const size_t head_base = ((size_t)b * KVr + kvh) * a.max_seq;
  uint16_t* kc = a.k_cache + head_base * HD;
  uint16_t* vc = a.v_cache + head_base * HD;
  if (!bad && k0 <= pos && pos < k1) {  // this split owns slot pos: append the new K/V row
    for (int i = tid; i < HD; i += 128) {
      kc[(size_t)pos * HD + i] = f2bf_bits(kn_s[i]);
      vc[(size_t)pos * HD + i] = f2bf_bits(vn_s[i]);
    }
  }
  __syncthreads();

  float qr[G][EPL];
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int e = 0; e < EPL; ++e) qr[g][e] = q_s[g][lane * EPL + e];
  float m[G], l[G], acc[G][EPL];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    m[g] = -INFINITY;
    l[g] = 0.f;
#pragma unroll
    for (int e = 0; e < EPL; ++e) acc[g][e] = 0.f;
  }
  for (int p = k0 + warp; p < k1; p += 4) {
    float kf[EPL], vf[EPL];
    if constexpr (EPL == 4) {
      const uint2 kv = *reinterpret_cast<const uint2*>(kc + (size_t)p * HD + lane * 4);
      const uint2 vv = *reinterpret_cast<const uint2*>(vc + (size_t)p * HD + lane * 4);
      kf[0] = bf16_lo(kv.x); kf[1] = bf16_hi(kv.x); kf[2] = bf16_lo(kv.y); kf[3] = bf16_hi(kv.y);
      vf[0] = bf16_lo(vv.x); vf[1] = bf16_hi(vv.x); vf[2] = bf16_lo(vv.y); vf[3] = bf16_hi(vv.y);
    } else {
      const uint32_t kv = *reinterpret_cast<const uint32_t*>(kc + (size_t)p * HD + lane * 2);
      const uint32_t vv = *reinterpret_cast<const uint32_t*>(vc + (size_t)p * HD + lane * 2);
      kf[0] = bf16_lo(kv); kf[1] = bf16_hi(kv);
      vf[0] = bf16_lo(vv); vf[1] = bf16_hi(vv);
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float s = 0.f;
#pragma unroll
      for (int e = 0; e < EPL; ++e) s = fmaf(qr[g][e], kf[e], s);
      s = warp_sum(s) * scale;
      const float mn = fmaxf(m[g], s);
      const float corr = expf(m[g] - mn);
      const float pe = expf(s - mn);
      l[g] = l[g] * corr + pe;
#pragma unroll
      for (int e = 0; e < EPL; ++e) acc[g][e] = fmaf(pe, vf[e], acc[g][e] * corr);
      m[g] = mn;
    }
  }
  if (lane == 0)
#pragma unroll
    for (int g = 0; g < G; ++g) {
      wm[warp][g] = m[g];
      wl[warp][g] = l[g];
    }
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int e = 0; e < EPL; ++e) wacc[warp][g][lane * EPL + e] = acc[g][e];
  __syncthreads();
  // CTA partial (M, L, A[HD]) per q head of the group
  float* part = a.part + (((size_t)b * KVr + kvh) * S + split) * G * (HD + 2);
  for (int idx = tid; idx < G * HD; idx += 128) {
    const int g = idx / HD, i = idx % HD;
    float M = -INFINITY;
    for (int w = 0; w < 4; ++w) M = fmaxf(M, wm[w][g]);
    float L = 0.f, A = 0.f;
    if (M != -INFINITY)
      for (int w = 0; w < 4; ++w)
        if (wm[w][g] != -INFINITY) {
          const float f = expf(wm[w][g] - M);
          L += wl[w][g] * f;
          A += wacc[w][g][i] * f;
        }
    float* pg = part + g * (HD + 2);
    if (i == 0) {
      pg[0] = M;
      pg[1] = L;
    }
    pg[2 + i] = A;
  }
  if (!arrive_last(a.counters + b * KVr + kvh, S)) return;
  // last CTA for (b, kvh): combine the S splits
  const float* pb = a.part + ((size_t)b * KVr + kvh) * S * G * (HD + 2);
  for (int idx = tid; idx < G * HD; idx += 128) {
    const int g = idx / HD, i = idx % HD;
    float M = -INFINITY;
    for (int sp = 0; sp < S; ++sp) M = fmaxf(M, __ldcg(pb + (sp * G + g) * (HD + 2)));
    float L = 0.f, A = 0.f;
    if (M != -INFINITY)
      for (int sp = 0; sp < S; ++sp) {
        const float* ps = pb + (sp * G + g) * (HD + 2);
        const float Ms = __ldcg(ps);
        if (Ms == -INFINITY) continue;
        const float f = expf(Ms - M);
        L += __ldcg(ps + 1) * f;
        A += __ldcg(ps + 2 + i) * f;
      }
    const float o = L > 0.f ? A / L : 0.f;
    a.out[(size_t)b * Hr * HD + (kvh * G + g) * HD + i] = o;
  }
}

// ===================================================================== host-side launchers
namespace launch {

constexpr int kNW = 8;

static size_t gemv_fixed_smem(int B, int K) { return (size_t)B * K * 4 + 32 * 4 + kNW * B * 8 + 16 + 64; }

int gemv_nslot(int B, int K, size_t smem_budget) {
  size_t fixed = gemv_fixed_smem(B, K);
  size_t per = (size_t)K * 2 + 16;
  long n = (long)((smem_budget - fixed) / per);
  if (n > 32) n = 32;
  return (int)n;
}

template <int B>
static cudaError_t gemv_b(const GemvArgs& a, int grid, int nslot, cudaStream_t st) {
  auto kern = gemv_stream_kernel<B, kNW>;
  size_t smem = (size_t)nslot * (a.K * 2 + 16) + gemv_fixed_smem(B, a.K);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, (kNW + 1) * 32, smem, st>>>(a, nslot);
  return cudaGetLastError();
}

cudaError_t gemv(const GemvArgs& a, int B, int grid, int nslot, cudaStream_t st) {
  switch (B) {
    case 1: return gemv_b<1>(a, grid, nslot, st);
    case 2: return gemv_b<2>(a, grid, nslot, st);
    case 4: return gemv_b<4>(a, grid, nslot, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t argmax_finalize(unsigned long long* amax, int B, int32_t* token_out, cudaStream_t st) {
  argmax_finalize_kernel<<<1, 32, 0, st>>>(amax, B, token_out);
  return cudaGetLastError();
}

static size_t ffn_fixed_smem(int B, int d) {
  return (size_t)B * d * 4 + (size_t)B * kFfnMaxN * 4 + B * 32 * 4 + 32 * 4 + kFfnMaxN * 4 + kFfnMaxChunks * B * 4 +
         kFfnMaxChunks * 4 + B * 4 + 16 + kFfnMaxChunks * 8 + 64;
}

int ffn_nslot(int B, int d, size_t smem_budget) {
  long n = (long)((smem_budget - ffn_fixed_smem(B, d)) / ((size_t)d * 2 + 16));
  if (n > 32) n = 32;
  return (int)n;
}

int ffn_grid(int F, int num_sms) {
  int g = (F + 7) / 8;
  if (g > num_sms) g = num_sms;
  // at most kFfnMaxN neurons per CTA
  if ((F + g - 1) / g > kFfnMaxN) return -1;
  return g;
}

template <int B, int CPT>
static cudaError_t ffn_bc(const FfnArgs& a, int grid, int nslot, cudaStream_t st) {
  auto kern = ffn_fused_kernel<B, kNW, CPT>;
  size_t smem = (size_t)nslot * (a.d * 2 + 16) + ffn_fixed_smem(B, a.d);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3((kNW + 1) * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // co-residency for the grid barrier
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a, nslot);
}

template <int B>
static cudaError_t ffn_b(const FfnArgs& a, int grid, int nslot, cudaStream_t st) {
  const int chunks = a.d / 8, NT = kNW * 32;
  const int cpt = (chunks + NT - 1) / NT;
  if (cpt <= 1) return ffn_bc<B, 1>(a, grid, nslot, st);
  if (cpt <= 2) return ffn_bc<B, 2>(a, grid, nslot, st);
  if (cpt <= 4) return ffn_bc<B, 4>(a, grid, nslot, st);
  return cudaErrorInvalidValue;
}

cudaError_t ffn(const FfnArgs& a, int B, int grid, int nslot, cudaStream_t st) {
  switch (B) {
    case 1: return ffn_b<1>(a, grid, nslot, st);
    case 2: return ffn_b<2>(a, grid, nslot, st);
    case 4: return ffn_b<4>(a, grid, nslot, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t attn_decode(const AttnArgs& a, int B, int hd, int group, cudaStream_t st) {
  dim3 grid(a.splits, a.KVr, B);
  const float scale = 1.0f / sqrtf((float)hd);
#define SIRIUS_ATTN(HD, GG)                                       \
  if (hd == HD && group == GG) {                                  \
    attn_decode_kernel<HD, GG><<<grid, 128, 0, st>>>(a, scale);   \
    return cudaGetLastError();                                    \
  }
  SIRIUS_ATTN(128, 1) SIRIUS_ATTN(128, 2) SIRIUS_ATTN(128, 4) SIRIUS_ATTN(128, 8)
  SIRIUS_ATTN(64, 1) SIRIUS_ATTN(64, 2) SIRIUS_ATTN(64, 4) SIRIUS_ATTN(64, 8)
#undef SIRIUS_ATTN
  return cudaErrorInvalidValue;
}

}  // namespace launch
}  // namespace sirius
