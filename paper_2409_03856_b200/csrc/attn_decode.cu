// attn_decode.cu — decode attention for sm_100a: RoPE of q/k, K/V append at
// the row's position in the static bf16 cache, split-K attention over [0, pos] with shared-memory
// staged 64-key blocks (one thread per (key, head) score, online softmax per block), last-arriving
// CTA combines the splits.  Also the packed-argmax finalize used after a cross-rank max.
// Numeric contract (D15): bf16 KV-cache storage (k after RoPE, v); q, scores, softmax and
// the attention output fp32.
#include "common.cuh"
#include "decode_kernels.cuh"

namespace sirius {

// amax -> token (after a cross-rank max of the packed keys); resets amax.
__global__ void argmax_finalize_kernel(unsigned long long* amax, int B, int32_t* token_out) {
  int b = threadIdx.x;
  if (b < B) {
    unsigned long long k = amax[b];
    amax[b] = 0ull;
    token_out[b] = (int32_t)argmax_key_index(k);
  }
}

// ===================================================================== decode attention
// grid (S splits, KVr, B), 128 threads.  Split `split` of sequence b / kv head kvh covers keys
// [k0, k1) of [0, pos]; it walks them in blocks of KB keys staged in shared memory.
template <int HD, int G>
__global__ void __launch_bounds__(128) attn_decode_kernel(AttnArgs a, float scale) {
  constexpr int KB = 64;
  constexpr int ROWB = HD * 2 + 16;                       // padded K row (bytes): conflict-free row reads
  constexpr int HPT = G / 2 > 1 ? G / 2 : 1;              // heads per thread in the score phase
  constexpr int NHO = (G * HD + 127) / 128;               // (head, dim) outputs per thread
  const int split = blockIdx.x, kvh = blockIdx.y, b = blockIdx.z;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  __shared__ __align__(16) float q_s[G][HD];
  __shared__ float kn_s[HD], vn_s[HD];
  __shared__ __align__(16) uint8_t k_s[KB * ROWB];
  __shared__ __align__(16) uint16_t v_s[KB][HD];
  __shared__ float sc[G][KB];
  __shared__ float m_s[G], l_s[G], c_s[G];
  __shared__ float cw[64][G];  // combine weights (M_s, then exp(M_s - M))
  __shared__ float cl2[64][G]; // L_s
  __shared__ float cl[G];

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
  const int s_active = chunk > 0 ? (nkeys + chunk - 1) / chunk : 0;

  // RoPE (rotate-half) on q and k at position pos; k (and v) rounded to bf16 as stored in the cache
  const float* qkv = a.qkv + (size_t)b * qkv_stride;
  const float* cs = a.rope_cos + (size_t)pos * (HD / 2);
  const float* sn = a.rope_sin + (size_t)pos * (HD / 2);
  for (int idx = tid; idx < G * (HD / 2); idx += 128) {
    const int g = idx / (HD / 2), i = idx % (HD / 2);
    const float* q = qkv + (kvh * G + g) * HD;
    const float x0 = q[i], x1 = q[i + HD / 2], c = cs[i], s = sn[i];
    q_s[g][i] = (x0 * c - x1 * s) * scale;  // the 1/sqrt(hd) score scale folded into q
    q_s[g][i + HD / 2] = (x1 * c + x0 * s) * scale;
  }
  if (tid < HD / 2) {
    const float* k = qkv + (Hr + kvh) * HD;
    const float x0 = k[tid], x1 = k[tid + HD / 2], c = cs[tid], s = sn[tid];
    kn_s[tid] = x0 * c - x1 * s;
    kn_s[tid + HD / 2] = x1 * c + x0 * s;
  }
  for (int i = tid; i < HD; i += 128) vn_s[i] = qkv[(Hr + KVr + kvh) * HD + i];
  if (tid < G) {
    m_s[tid] = -INFINITY;
    l_s[tid] = 0.f;
  }
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

  // output ownership: thread t -> dim t % HD, heads g = t / HD + 128/HD * j
  float acc[NHO];
#pragma unroll
  for (int j = 0; j < NHO; ++j) acc[j] = 0.f;
  const int od = tid % HD, og0 = tid / HD;
  constexpr int GSTEP = 128 / HD;

  for (int p0 = k0; p0 < k1; p0 += KB) {
    const int nb = min(KB, k1 - p0);
    // stage K (padded rows) and V for keys [p0, p0 + nb): 16-byte loads, all issued before use
    constexpr int VPR = HD / 8;  // uint4 per row
    constexpr int NL = KB * VPR / 128;  // uint4 per thread per operand; all loads issued first
    uint4 kv[NL], vv[NL];
#pragma unroll
    for (int j = 0; j < NL; ++j) {
      const int idx = tid + 128 * j, kk = idx / VPR, e = idx % VPR;
      if (kk < nb) {
        kv[j] = *reinterpret_cast<const uint4*>(kc + (size_t)(p0 + kk) * HD + e * 8);
        vv[j] = *reinterpret_cast<const uint4*>(vc + (size_t)(p0 + kk) * HD + e * 8);
      }
    }
#pragma unroll
    for (int j = 0; j < NL; ++j) {
      const int idx = tid + 128 * j, kk = idx / VPR, e = idx % VPR;
      if (kk < nb) {
        *reinterpret_cast<uint4*>(k_s + kk * ROWB + e * 16) = kv[j];
        *reinterpret_cast<uint4*>(&v_s[kk][e * 8]) = vv[j];
      }
    }
    __syncthreads();
    // scores: thread t -> key t % KB, heads (t / KB) * HPT + j
    {
      const int kk = tid % KB, hg = tid / KB;
      if (kk < nb && hg * HPT < G) {
        float s[HPT];
#pragma unroll
        for (int j = 0; j < HPT; ++j) s[j] = 0.f;
        const uint4* kr = reinterpret_cast<const uint4*>(k_s + kk * ROWB);
#pragma unroll 4
        for (int e = 0; e < HD / 8; ++e) {
          const uint4 w = kr[e];
          const float kf[8] = {bf16_lo(w.x), bf16_hi(w.x), bf16_lo(w.y), bf16_hi(w.y),
                               bf16_lo(w.z), bf16_hi(w.z), bf16_lo(w.w), bf16_hi(w.w)};
#pragma unroll
          for (int j = 0; j < HPT; ++j) {
            const int g = hg * HPT + j;
            if (g < G) {
              const float4 q0 = *reinterpret_cast<const float4*>(&q_s[g][e * 8]);
              const float4 q1 = *reinterpret_cast<const float4*>(&q_s[g][e * 8 + 4]);
              s[j] = fmaf(kf[0], q0.x, s[j]); s[j] = fmaf(kf[1], q0.y, s[j]);
              s[j] = fmaf(kf[2], q0.z, s[j]); s[j] = fmaf(kf[3], q0.w, s[j]);
              s[j] = fmaf(kf[4], q1.x, s[j]); s[j] = fmaf(kf[5], q1.y, s[j]);
              s[j] = fmaf(kf[6], q1.z, s[j]); s[j] = fmaf(kf[7], q1.w, s[j]);
            }
          }
        }
#pragma unroll
        for (int j = 0; j < HPT; ++j)
          if (hg * HPT + j < G) sc[hg * HPT + j][kk] = s[j];
      }
    }
    __syncthreads();
    // online softmax per head (warp w handles heads w, w + 4, ...)
    for (int g = warp; g < G; g += 4) {
      const float x0 = lane < nb ? sc[g][lane] : -INFINITY;
      const float x1 = lane + 32 < nb ? sc[g][lane + 32] : -INFINITY;
      const float bm = warp_max(fmaxf(x0, x1));
      const float mold = m_s[g];
      const float mn = fmaxf(mold, bm);
      const float p0v = lane < nb ? expf(x0 - mn) : 0.f;
      const float p1v = lane + 32 < nb ? expf(x1 - mn) : 0.f;
      sc[g][lane] = p0v;
      sc[g][lane + 32] = p1v;
      const float bs = warp_sum(p0v + p1v);
      if (lane == 0) {
        const float corr = mold == -INFINITY ? 0.f : expf(mold - mn);
        c_s[g] = corr;
        l_s[g] = l_s[g] * corr + bs;
        m_s[g] = mn;
      }
    }
    __syncthreads();
    // P.V: thread (dim od, heads og0 + GSTEP j)
#pragma unroll
    for (int j = 0; j < NHO; ++j) {
      const int g = og0 + GSTEP * j;
      if (g < G) {
        float s = acc[j] * c_s[g];
        for (int kk = 0; kk < nb; ++kk) s = fmaf(sc[g][kk], __uint_as_float((uint32_t)v_s[kk][od] << 16), s);
        acc[j] = s;
      }
    }
    __syncthreads();
  }
  // CTA partial (M, L, A[HD]) per q head of the group
  float* part = a.part + (((size_t)b * KVr + kvh) * S + split) * G * (HD + 2);
#pragma unroll
  for (int j = 0; j < NHO; ++j) {
    const int g = og0 + GSTEP * j;
    if (g < G) {
      part[g * (HD + 2) + 2 + od] = acc[j];
      if (od == 0) {
        part[g * (HD + 2)] = m_s[g];
        part[g * (HD + 2) + 1] = l_s[g];
      }
    }
  }
  group_barrier(a.group_bar + 2 * (b * KVr + kvh), S);
  // ---- distributed combine: split s finalises outputs (g, d) in [G HD s / S, G HD (s+1) / S)
  const float* pb = a.part + ((size_t)b * KVr + kvh) * S * G * (HD + 2);
  {  // (M_s, L_s) of every active split: one parallel round trip into shared memory
    constexpr int NMW = (64 * G + 127) / 128;
    float mv[NMW], lv[NMW];
#pragma unroll
    for (int j = 0; j < NMW; ++j) {
      const int idx = tid + 128 * j;
      if (idx < s_active * G) {
        const float* ps = pb + (size_t)idx * (HD + 2);  // idx = sp * G + g
        mv[j] = __ldcg(ps);
        lv[j] = __ldcg(ps + 1);
      }
    }
#pragma unroll
    for (int j = 0; j < NMW; ++j) {
      const int idx = tid + 128 * j;
      if (idx < s_active * G) {
        cw[idx / G][idx % G] = mv[j];
        cl2[idx / G][idx % G] = lv[j];
      }
    }
  }
  __syncthreads();
  if (tid < G) {
    float M = -INFINITY;
    for (int sp = 0; sp < s_active; ++sp) M = fmaxf(M, cw[sp][tid]);
    float L = 0.f;
    for (int sp = 0; sp < s_active; ++sp) {
      const float f = cw[sp][tid] == -INFINITY ? 0.f : expf(cw[sp][tid] - M);
      L += cl2[sp][tid] * f;
      cw[sp][tid] = f;
    }
    cl[tid] = L;
  }
  __syncthreads();
  const int oa = G * HD * split / S, oz = G * HD * (split + 1) / S;
  for (int o0 = oa + tid; o0 < oz; o0 += 128) {
    const int g = o0 / HD, d = o0 % HD;
    float o = 0.f;
    for (int sp0 = 0; sp0 < s_active; sp0 += 16) {  // 16 independent loads in flight
      float v[16];
#pragma unroll
      for (int u = 0; u < 16; ++u)
        v[u] = sp0 + u < s_active ? __ldcg(pb + ((size_t)(sp0 + u) * G + g) * (HD + 2) + 2 + d) : 0.f;
#pragma unroll
      for (int u = 0; u < 16; ++u)
        if (sp0 + u < s_active) o += v[u] * cw[sp0 + u][g];
    }
    a.out[(size_t)b * Hr * HD + (kvh * G + g) * HD + d] = cl[g] > 0.f ? o / cl[g] : 0.f;
  }
}

// ===================================================================== host-side launchers
namespace launch {

cudaError_t argmax_finalize(unsigned long long* amax, int B, int32_t* token_out, cudaStream_t st) {
  argmax_finalize_kernel<<<1, 32, 0, st>>>(amax, B, token_out);
  return cudaGetLastError();
}

int attn_splits(int B, int KVr, int num_sms) {
  int s = num_sms / (B * KVr);  // one wave
  return s < 1 ? 1 : (s > 64 ? 64 : s);
}

cudaError_t attn_decode(const AttnArgs& a, int B, int hd, int group, cudaStream_t st) {
  dim3 grid(a.splits, a.KVr, B);
  const float scale = 1.0f / sqrtf((float)hd);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(128);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // co-residency for the per-(b, kvh) split barrier
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = a.splits > 1 ? 1 : 0;
#define SIRIUS_ATTN(HD, GG) \
  if (hd == HD && group == GG) return cudaLaunchKernelEx(&cfg, attn_decode_kernel<HD, GG>, a, scale);
  SIRIUS_ATTN(128, 1) SIRIUS_ATTN(128, 2) SIRIUS_ATTN(128, 4) SIRIUS_ATTN(128, 8)
  SIRIUS_ATTN(64, 1) SIRIUS_ATTN(64, 2) SIRIUS_ATTN(64, 4) SIRIUS_ATTN(64, 8)
#undef SIRIUS_ATTN
  return cudaErrorInvalidValue;
}

}  // namespace launch
}  // namespace sirius
