// attn_rows.cu — causal multi-row attention of the verification / prefill forward (SURVEY.md §8(a)
// S8; "the full model takes in the last kernel size of tokens ... in parallel").
//
// Query rows of one (sequence, kv head) — R = rows_per_seq x G q-heads, up to 64 per row block —
// attend causally: row i (position T + i) sees cache[0, T) and the kernel's own rows [0, i] (verify:
// in the staging area; prefill: already in the cache).  grid (S splits, KVr x row_blocks, nseq),
// 256 threads, cooperative (one wave, all CTAs co-resident).  Each CTA walks its key range in
// 64-key blocks staged in shared memory:
//   scores   thread -> (keys lane, lane + 32; 8 rows)  k rows padded: conflict-free, q broadcast
//   softmax  warp   -> 8 rows, online (running max / sum per row)
//   P.V      thread -> (4 dims, 8 rows)               v: 8-byte reads, p broadcast
// then writes its partial (M, L, A) per row; after a barrier among the S splits of the group, split s
// combines rows [64 s / S, 64 (s+1) / S) and writes them as a bf16 hi/lo pair (the tensor-core
// operand of the O-projection).  fp32 throughout (D15).
#include "common.cuh"
#include "verify_kernels.cuh"

namespace sirius {
namespace {

constexpr int kRows = 64, kKB = 64, kThreads = 256;

SIRIUS_DEV void rstamp(const AttnRowsArgs& a, int slot) {  // debug phase stamps (a.trace != NULL)
  if (!a.trace) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const int cta = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    a.trace[(size_t)slot * 1024 + cta] = t;  // [8][1024]
  }
}

template <int HD>
__global__ void __launch_bounds__(kThreads, 1) attn_rows_kernel(AttnRowsArgs a, float scale) {
  constexpr int KROW = HD + 8;                     // padded bf16 K row (elements)
  constexpr int DPL = HD / 32;                     // P.V dims per thread (4 for HD=128)
  constexpr int RPW = kRows / (kThreads / 32);     // P.V rows per thread (8)
  extern __shared__ __align__(16) uint8_t smem[];
  float* q_s = reinterpret_cast<float*>(smem);                                   // [kRows][HD]
  uint16_t* k_s = reinterpret_cast<uint16_t*>(q_s + kRows * HD);                 // [kKB][KROW]
  uint16_t* v_s = k_s + kKB * KROW;                                              // [kKB][HD]
  float* p_s = reinterpret_cast<float*>(v_s + kKB * HD);                         // [kRows][kKB + 1]
  float* m_s = p_s + kRows * (kKB + 1);                                          // [kRows]
  float* l_s = m_s + kRows;
  float* c_s = l_s + kRows;

  pdl_trigger();
  pdl_wait();
  rstamp(a, 0);
  const int split = blockIdx.x, bz = blockIdx.z, b = a.b_base + bz;
  const int kvh = blockIdx.y % a.KVr, rb = blockIdx.y / a.KVr;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = a.G, rows = a.rows_per_seq;
  const int T = a.start[b];
  const int r_base = rb * kRows;                                  // row index r = i * G + g
  const int nr = min(kRows, rows * G - r_base);                   // valid rows in this block
  const int i_last = (r_base + nr - 1) / G;
  const int nkeys = max(0, T + a.stage_base + i_last + 1);  // own staging row = stage_base + i
  const int S = gridDim.x;
  const int chunk = (nkeys + S - 1) / S;
  const int k0 = min(nkeys, split * chunk), k1 = min(nkeys, k0 + chunk);
  const size_t hb = (size_t)b * a.KVr + kvh;
  const uint16_t* kc = a.k_cache + hb * a.max_seq * HD;
  const uint16_t* vc = a.v_cache + hb * a.max_seq * HD;
  const uint16_t* kf = a.fresh_in_cache ? kc + (size_t)T * HD : a.k_fresh + hb * a.fresh_stride * HD;
  const uint16_t* vf = a.fresh_in_cache ? vc + (size_t)T * HD : a.v_fresh + hb * a.fresh_stride * HD;

  // q rows (fp32, post-RoPE), score scale folded in; all loads issued first
  {
    constexpr int NQ = kRows * HD / 4 / kThreads;
    float4 qv[NQ];
#pragma unroll
    for (int j = 0; j < NQ; ++j) {
      const int idx = tid + kThreads * j, r = idx / (HD / 4), e4 = idx % (HD / 4);
      qv[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < nr) {
        const int rr = r_base + r, i = rr / G, g = rr % G;
        qv[j] = __ldcg(reinterpret_cast<const float4*>(a.q + (size_t)(bz * rows + i) * a.Hr * HD + (kvh * G + g) * HD) + e4);
      }
    }
#pragma unroll
    for (int j = 0; j < NQ; ++j)
      reinterpret_cast<float4*>(q_s)[tid + kThreads * j] =
          make_float4(qv[j].x * scale, qv[j].y * scale, qv[j].z * scale, qv[j].w * scale);
  }
  if (tid < kRows) {
    m_s[tid] = -INFINITY;
    l_s[tid] = 0.f;
  }
  rstamp(a, 1);
  const int dg = lane, rg = warp;  // P.V: dims 4 dg .. 4 dg + 3, rows 8 rg .. 8 rg + 7
  float acc[RPW][DPL];
#pragma unroll
  for (int j = 0; j < RPW; ++j)
#pragma unroll
    for (int e = 0; e < DPL; ++e) acc[j][e] = 0.f;

  for (int p0 = k0; p0 < k1; p0 += kKB) {
    const int nb = min(kKB, k1 - p0);
    __syncthreads();  // previous block's smem consumers done (and q_s / m_s init visible)
    constexpr int VPR = HD / 8;
    constexpr int NL = kKB * VPR / kThreads;  // uint4 per thread per operand; all loads issued first
    uint4 kv[NL], vv[NL];
#pragma unroll
    for (int j = 0; j < NL; ++j) {
      const int idx = tid + kThreads * j, kk = idx / VPR, e = idx % VPR, p = p0 + kk;
      if (kk < nb) {
        const uint16_t* ks = p < T ? kc + (size_t)p * HD : kf + (size_t)(p - T) * HD;
        const uint16_t* vs = p < T ? vc + (size_t)p * HD : vf + (size_t)(p - T) * HD;
        kv[j] = *reinterpret_cast<const uint4*>(ks + e * 8);
        vv[j] = *reinterpret_cast<const uint4*>(vs + e * 8);
      }
    }
#pragma unroll
    for (int j = 0; j < NL; ++j) {
      const int idx = tid + kThreads * j, kk = idx / VPR, e = idx % VPR;
      if (kk < nb) {
        *reinterpret_cast<uint4*>(k_s + kk * KROW + e * 8) = kv[j];
        *reinterpret_cast<uint4*>(v_s + kk * HD + e * 8) = vv[j];
      }
    }
    __syncthreads();
    rstamp(a, 2);
    // ---- scores s[r][kk] = q_r . k_kk  (masked: key p visible to row i iff p <= T + i)
    // thread -> keys (lane, lane + 32) x rows (warp + 8 j): per 8 dims 2 k reads (conflict-free rows)
    // and 2 q reads per row (warp-uniform: broadcast) feed 16 dot products; every dot product sums its
    // dims in ascending order
    {
      constexpr int KPT = kThreads / kKB == 4 ? 2 : 1;  // keys per thread
      constexpr int RW = kRows / (kThreads / 32);       // rows per thread (8)
      static_assert(KPT == 2 && RW == 8, "scores mapping: 256 threads, 64 rows x 64 keys");
      const int kk0 = lane, rr0 = warp;
      float s2[KPT][RW];
#pragma unroll
      for (int c = 0; c < KPT; ++c)
#pragma unroll
        for (int j = 0; j < RW; ++j) s2[c][j] = 0.f;
      if (kk0 < nb) {
        const uint16_t* kr0 = k_s + kk0 * KROW;
        const uint16_t* kr1 = k_s + (kk0 + 32) * KROW;  // rows >= nb hold stale data: masked below
#pragma unroll 2
        for (int e = 0; e < HD / 8; ++e) {
          float kf[KPT][8];
#pragma unroll
          for (int c = 0; c < KPT; ++c) {
            const uint4 w = *reinterpret_cast<const uint4*>((c == 0 ? kr0 : kr1) + e * 8);
            kf[c][0] = bf16_lo(w.x); kf[c][1] = bf16_hi(w.x); kf[c][2] = bf16_lo(w.y); kf[c][3] = bf16_hi(w.y);
            kf[c][4] = bf16_lo(w.z); kf[c][5] = bf16_hi(w.z); kf[c][6] = bf16_lo(w.w); kf[c][7] = bf16_hi(w.w);
          }
#pragma unroll
          for (int j = 0; j < RW; ++j) {
            const float4 qa = *reinterpret_cast<const float4*>(q_s + (rr0 + 8 * j) * HD + e * 8);
            const float4 qb = *reinterpret_cast<const float4*>(q_s + (rr0 + 8 * j) * HD + e * 8 + 4);
#pragma unroll
            for (int c = 0; c < KPT; ++c) {
              float t = s2[c][j];
              t = fmaf(kf[c][0], qa.x, t); t = fmaf(kf[c][1], qa.y, t); t = fmaf(kf[c][2], qa.z, t);
              t = fmaf(kf[c][3], qa.w, t); t = fmaf(kf[c][4], qb.x, t); t = fmaf(kf[c][5], qb.y, t);
              t = fmaf(kf[c][6], qb.z, t); t = fmaf(kf[c][7], qb.w, t);
              s2[c][j] = t;
            }
          }
        }
      }
#pragma unroll
      for (int c = 0; c < KPT; ++c)
#pragma unroll
        for (int j = 0; j < RW; ++j) {
          const int kk = kk0 + 32 * c, r = rr0 + 8 * j;
          const int i = (r_base + r) / G, p = p0 + kk;
          bool vis = kk < nb && r < nr;
          if (p >= T) vis = vis && (a.tree_vis ? ((a.tree_vis[a.stage_base + i] >> (p - T)) & 1ull) != 0 : p <= T + i);
          p_s[r * (kKB + 1) + kk] = vis ? s2[c][j] : -INFINITY;
        }
    }
    __syncthreads();
    rstamp(a, 3);
    // ---- online softmax per row: warp w -> rows 8w .. 8w+7
    for (int r = warp * (kRows / 8); r < (warp + 1) * (kRows / 8); ++r) {
      float* pr = p_s + r * (kKB + 1);
      const float x0 = pr[lane], x1 = pr[lane + 32];
      const float bm = warp_max(fmaxf(x0, x1));
      const float mold = m_s[r];
      const float mn = fmaxf(mold, bm);
      const float e0 = mn == -INFINITY ? 0.f : expf(x0 - mn);
      const float e1 = mn == -INFINITY ? 0.f : expf(x1 - mn);
      pr[lane] = e0;
      pr[lane + 32] = e1;
      const float bs = warp_sum(e0 + e1);
      __syncwarp();  // every lane has read m_s[r] / l_s[r] before lane 0 rewrites them
      if (lane == 0) {
        const float corr = mold == -INFINITY ? 0.f : expf(mold - mn);
        c_s[r] = corr;
        l_s[r] = l_s[r] * corr + bs;
        m_s[r] = mn;
      }
    }
    __syncthreads();
    // ---- P.V: thread -> (dims 4 dg.., rows 8 rg..)
#pragma unroll
    for (int j = 0; j < RPW; ++j) {
      const float c = c_s[rg * RPW + j];
#pragma unroll
      for (int e = 0; e < DPL; ++e) acc[j][e] *= c;
    }
    for (int kk = 0; kk < nb; ++kk) {
      float vf4[DPL];
      if constexpr (DPL == 4) {
        const uint2 w = *reinterpret_cast<const uint2*>(v_s + kk * HD + dg * 4);
        vf4[0] = bf16_lo(w.x); vf4[1] = bf16_hi(w.x); vf4[2] = bf16_lo(w.y); vf4[3] = bf16_hi(w.y);
      } else {
        const uint32_t w = *reinterpret_cast<const uint32_t*>(v_s + kk * HD + dg * 2);
        vf4[0] = bf16_lo(w); vf4[1] = bf16_hi(w);
      }
#pragma unroll
      for (int j = 0; j < RPW; ++j) {
        const float p = p_s[(rg * RPW + j) * (kKB + 1) + kk];
#pragma unroll
        for (int e = 0; e < DPL; ++e) acc[j][e] = fmaf(p, vf4[e], acc[j][e]);
      }
    }
  }
  __syncthreads();
  rstamp(a, 4);
  // ---- partial (M, L, A) of this split -> group barrier over the S splits
  const int RB = gridDim.y / a.KVr;
  const size_t grp = ((size_t)bz * a.KVr + kvh) * RB + rb;
  float* pbase = a.part + grp * S * kRows * (HD + 2);
  float* part = pbase + (size_t)split * kRows * (HD + 2);
#pragma unroll
  for (int j = 0; j < RPW; ++j) {
    float* pr = part + (rg * RPW + j) * (HD + 2) + 2 + dg * DPL;
#pragma unroll
    for (int e = 0; e < DPL; ++e) pr[e] = acc[j][e];
  }
  if (tid < kRows) {
    part[tid * (HD + 2)] = m_s[tid];
    part[tid * (HD + 2) + 1] = l_s[tid];
  }
  rstamp(a, 5);
  group_barrier(a.group_bar + 2 * grp, S);
  rstamp(a, 6);
  // ---- distributed combine: split s finalises rows [64 s / S, 64 (s+1) / S)
  const int s_active = chunk > 0 ? (nkeys + chunk - 1) / chunk : 0;
  const int ra = kRows * split / S, rz = kRows * (split + 1) / S, nrow = rz - ra;
  // (a) this thread's first two outputs' partial values A_s, requested before anything else (they do
  // not depend on the weights); (b) per-row weights w_s = e^(M_s - M) / sum_s e^(M_s - M) L_s, one warp
  // per row, into shared memory (p_s is free after P.V); (c) o = sum_s w_s A_s in split order
  const int nout = nrow * HD;
  float av[2][32];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int idx = tid + kThreads * q, rl = idx / HD, d = idx % HD, r = ra + rl;
    const bool ok = idx < nout && r < nr;
#pragma unroll
    for (int u = 0; u < 32; ++u)
      av[q][u] = (ok && u < s_active) ? __ldcg(pbase + ((size_t)u * kRows + r) * (HD + 2) + 2 + d) : 0.f;
  }
  float* wt = p_s;  // [nrow][kKB] (s_active <= S <= kKB)
  for (int rl = warp; rl < nrow; rl += kThreads / 32) {
    const int r = ra + rl;
    if (r >= nr) continue;  // warp-uniform
    const float* pr0 = pbase + ((size_t)lane * kRows + r) * (HD + 2);
    const float* pr1 = pbase + ((size_t)(lane + 32) * kRows + r) * (HD + 2);
    const float m0 = lane < s_active ? __ldcg(pr0) : -INFINITY, l0 = lane < s_active ? __ldcg(pr0 + 1) : 0.f;
    const float m1 = lane + 32 < s_active ? __ldcg(pr1) : -INFINITY, l1 = lane + 32 < s_active ? __ldcg(pr1 + 1) : 0.f;
    const float M = warp_max(fmaxf(m0, m1));
    const float f0 = m0 == -INFINITY ? 0.f : expf(m0 - M), f1 = m1 == -INFINITY ? 0.f : expf(m1 - M);
    const float Ls = warp_sum(l0 * f0 + l1 * f1);
    const float inv = Ls > 0.f ? 1.0f / Ls : 0.f;
    wt[rl * kKB + lane] = f0 * inv;
    wt[rl * kKB + lane + 32] = f1 * inv;
  }
  __syncthreads();
  auto emit = [&](int idx, float val) {
    const int rl = idx / HD, d = idx % HD, r = ra + rl;
    const int rr = r_base + r, i = rr / G, g = rr % G;
    const size_t off = (size_t)(bz * rows + i) * a.Hr * HD + (kvh * G + g) * HD + d;
    store_split3(a.out3, a.plane, off, val);
  };
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int idx = tid + kThreads * q, rl = idx / HD, d = idx % HD, r = ra + rl;
    if (idx >= nout || r >= nr) continue;
    float o = 0.f;
#pragma unroll
    for (int u = 0; u < 32; ++u) o = fmaf(wt[rl * kKB + u], av[q][u], o);
    for (int u = 32; u < s_active; ++u) o = fmaf(wt[rl * kKB + u], __ldcg(pbase + ((size_t)u * kRows + r) * (HD + 2) + 2 + d), o);
    emit(idx, o);
  }
  for (int idx = tid + 2 * kThreads; idx < nout; idx += kThreads) {  // few splits: more rows per split
    const int rl = idx / HD, d = idx % HD, r = ra + rl;
    if (r >= nr) continue;
    float o = 0.f;
    for (int u = 0; u < s_active; ++u) o = fmaf(wt[rl * kKB + u], __ldcg(pbase + ((size_t)u * kRows + r) * (HD + 2) + 2 + d), o);
    emit(idx, o);
  }
  rstamp(a, 7);
}

template <int HD>
size_t attn_rows_smem() {
  return (size_t)kRows * HD * 4 + (size_t)kKB * (HD + 8) * 2 + (size_t)kKB * HD * 2 + (size_t)kRows * (kKB + 1) * 4 +
         3 * kRows * 4;
}

template <int HD>
cudaError_t launch_hd(const AttnRowsArgs& a, dim3 grid, float scale, cudaStream_t st) {
  const size_t sm = attn_rows_smem<HD>();
  cudaError_t e = cudaFuncSetAttribute(attn_rows_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  // The per-group split barrier needs the S splits of a group co-resident: the grid is one wave
  // (attn_rows_splits); with PDL the predecessor's CTAs finish without waiting on this grid and the
  // successor launches only after every CTA of this grid has triggered (is resident).
  cudaLaunchAttribute attr[1];
  if (launch::g_chain_pdl) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
  } else {
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = (launch::g_chain_pdl || grid.x > 1) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, attn_rows_kernel<HD>, a, scale);
}

}  // namespace

namespace launch {

// splits per (sequence, kv head, row block): one wave of 1-CTA-per-SM blocks in total
int attn_rows_splits(int nseq, int KVr, int row_blocks, int max_keys, int num_sms) {
  int s = num_sms / (nseq * KVr * row_blocks);
  const int by_keys = (max_keys + kKB - 1) / kKB;  // no more splits than 64-key blocks
  if (s > by_keys) s = by_keys;
  if (s > kKB) s = kKB;                             // combine weights buffer
  return s < 1 ? 1 : s;
}

cudaError_t attn_rows(const AttnRowsArgs& a, int nseq, int hd, int splits, int row_blocks, cudaStream_t st) {
  dim3 grid(splits, a.KVr * row_blocks, nseq);
  const float scale = 1.0f / sqrtf((float)hd);
  if (hd == 128) return launch_hd<128>(a, grid, scale, st);
  if (hd == 64) return launch_hd<64>(a, grid, scale, st);
  return cudaErrorInvalidValue;
}

}  // namespace launch
}  // namespace sirius
