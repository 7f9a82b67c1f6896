// decode_step.cu — the whole decode step as ONE persistent kernel for
// tensor-parallel degree 1: one 512-thread CTA per SM, grid-wide barriers between the phases that
// have a grid-wide data dependency, and — the point of the design — every warp requests its first
// weight row of the NEXT phase before it arrives at the barrier.  Weights do not depend on the
// step's data, so HBM keeps streaming through each barrier and through each phase's activation
// prologue instead of idling for a kernel boundary (launch, drain, ramp-up: ~10 us per layer
// measured with one kernel per stage, r01 launch list).
//
// Per layer l (x = fp32 residual stream [B, d] in global memory):
//   P1  RMSNorm(x) -> QKV rows (warp per row)                        -> qkv   [B, (H+2KV) hd]
//   P2  RoPE q/k, K/V append at pos, split-K decode attention over [0, pos] (one (b, kv head,
//       split) item per CTA; split-group barrier + distributed combine) -> o [B, H hd]
//   P3  O-proj rows, residual add                                     -> x1 = x + o W_o^T
//   P4  CATS MLP of the CTA's neuron range: dense gate rows, a = SiLU(g),
//       |a| >= t_l, warp-ballot compaction, ACTIVE W_up / W_down rows only -> per-CTA partial
//   P5  deterministic column reduction of the partials                -> x = x1 + sum_c partial_c
// then final RMSNorm + LM head + packed (value, lowest index) argmax -> token_out.
// Arithmetic per element is the same as the one-kernel-per-stage path (gemv_ffn.cu,
// attn_stage_kernel below), which the TP > 1 path uses (its all-reduces sit between the stages).
// Numeric contract (D15): bf16 weights and KV cache, fp32 activations and accumulation.
#include "common.cuh"
#include "decode_kernels.cuh"
#include "gemv_dev.cuh"

namespace sirius {
namespace {

constexpr int kWarps = 16, kNT = kWarps * 32;
constexpr int kMaxN = 256;  // FFN neurons per CTA
constexpr int kMaxChunks = kMaxN / 32;
constexpr int kKB = 64;     // attention keys per shared-memory block
constexpr int kMaxSplits = 64;

using dev::prologue;
using dev::row_dot;
using dev::row_finish;
using dev::row_issue;
using dev::RowRegs;
using dev::after_all;
using dev::dot8p;

template <int B, int HD, int G>
struct StepSmem {
  // attention
  float q_s[G][HD];
  float kn_s[HD], vn_s[HD];
  __align__(16) uint8_t k_s[kKB * (HD * 2 + 16)];
  __align__(16) uint16_t v_s[kKB][HD];
  float sc[G][kKB];
  float m_s[G], l_s[G], c_s[G], cl[G];
  float cw[kMaxSplits][G], cl2[kMaxSplits][G];
  // FFN
  float a_s[B][kMaxN];
  float mm_s[B][kMaxN];
  int list_s[kMaxN];
  unsigned char bits_s[kMaxN];
  unsigned act_s[kMaxChunks][B];
  int cnt_s[kMaxChunks], off_s[kMaxChunks + 1];
  // misc
  float red_s[32];
  unsigned long long key_s[kWarps * B];
  unsigned flag_s;
};

SIRIUS_DEV int part_lo(int n, int c, int G) { return (int)((long long)n * c / G); }

// debug trace slots per layer (tools/step_trace.py): 0 P1 after prologue, 1 P1 arrive, 2 P1 exit,
// 3 P2 setup done, 4 P2 blocks done, 5 P2 group barrier done, 6 P2 arrive, 7 P2 exit, 8 P3 after
// prologue, 9 P3 arrive, 10 P3 exit, 11 P4 after prologue, 12 gate done, 13 compaction done,
// 14 up done, 15 P4 arrive, 16 P4 exit, 17 P5 arrive, 18 P5 exit; then 2 head slots.
constexpr int kTraceSlots = 20;
SIRIUS_DEV void stamp(const StepArgs& a, int slot) {
  if (!a.trace) return;
  __syncthreads();  // debug only: stamp when the whole CTA is done
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[(size_t)(1 + slot) * gridDim.x + blockIdx.x] = t;
  }
}

// ------------------------------------------------------------------------------------------ row streams
// A warp's stream of weight rows with DEPTH rows in flight: stream index k even -> registers, k odd ->
// the warp's shared-memory slot, filled by one 1-D bulk copy (TMA engine) completing on the warp's
// mbarrier.  Rows 0 and 1 of the NEXT phase are requested before the grid barrier, so the barrier,
// the phase's activation prologue and the first rows overlap with HBM transfers (r01 trace: one row
// in flight per warp left HBM idle ~1-3 us at every phase change).
template <int CPL, bool RING>
struct RowStream {
  static constexpr int DEPTH = RING ? 2 : 1;
  RowRegs<CPL> r;
  uint64_t pol;   // L2 policy of the weight loads
  uint4* slot;    // shared [32 CPL] uint4 (one row, RING only)
  uint64_t* bar;  // RING only
  uint32_t phase;
};

template <int CPL, bool RING>
SIRIUS_DEV void rs_issue(RowStream<CPL, RING>& s, int k, const uint16_t* row, int CH, int lane, bool valid) {
  if (!RING || (k & 1) == 0) {
    row_issue<CPL>(s.r, row, CH, lane, valid, s.pol);
  } else if (valid && lane == 0) {
    mbar_arrive_expect_tx(s.bar, (uint32_t)CH * 16u);
    bulk_g2s(s.slot, row, (uint32_t)CH * 16u, s.bar, policy_evict_first());
  }
}

template <int B, int CPL, bool RING>
SIRIUS_DEV void rs_finish(RowStream<CPL, RING>& s, int k, const uint16_t* row, const float4* hp, int CH, int lane,
                          float* acc) {
  if (!RING || (k & 1) == 0) {
    row_finish<B, CPL>(s.r, row, hp, CH, lane, acc);
    return;
  }
  mbar_wait(s.bar, s.phase);
  s.phase ^= 1u;
#pragma unroll
  for (int b = 0; b < B; ++b) acc[b] = 0.f;
#pragma unroll
  for (int u = 0; u < CPL; ++u) {  // same per-lane chunk order as row_finish
    const int c = lane + 32 * u;
    if (c < CH) {
      const uint4 w = s.slot[c];
#pragma unroll
      for (int b = 0; b < B; ++b) acc[b] = dot8p(w, hp[(b * 2) * CH + c], hp[(b * 2 + 1) * CH + c], acc[b]);
    }
  }
  __syncwarp();
  fence_proxy_async();  // the slot's generic-proxy reads precede the next bulk copy into it
}

// Rows 0 .. DEPTH-1 of a warp stream whose i-th row is row(i) (n rows).
template <int CPL, bool RING, class RowOf>
SIRIUS_DEV void rs_start(RowStream<CPL, RING>& s, int n, RowOf row, int CH, int lane) {
#pragma unroll
  for (int k = 0; k < RowStream<CPL, RING>::DEPTH; ++k) rs_issue<CPL, RING>(s, k, row(k), CH, lane, k < n);
}

// Consume the warp's n rows (started with rs_start): epi(i, acc) gets the warp-reduced dot products.
template <int B, int CPL, bool RING, class RowOf, class Epi>
SIRIUS_DEV void rs_run(RowStream<CPL, RING>& s, int n, RowOf row, const float4* hp, int CH, int lane, Epi epi) {
  constexpr int D = RowStream<CPL, RING>::DEPTH;
  for (int i = 0; i < n; ++i) {
    float acc[B];
    rs_finish<B, CPL, RING>(s, i, row(i), hp, CH, lane, acc);
    rs_issue<CPL, RING>(s, i + D, row(i + D) + after_all<B>(acc), CH, lane, i + D < n);
#pragma unroll
    for (int b = 0; b < B; ++b) acc[b] = warp_sum(acc[b]);
    epi(i, acc);
  }
}

SIRIUS_DEV int warp_rows(int r0, int r1, int warp) { return r1 - r0 > warp ? (r1 - r0 - warp + kWarps - 1) / kWarps : 0; }

// ------------------------------------------------------------------------------------------ P2
// The CTA's attention work item (b, kv head, split) and its key range [k0, k1) of [0, pos].
struct AttnItem {
  int active, b, kvh, split, pos, bad, k0, k1, s_active;
};

template <int B>
SIRIUS_DEV AttnItem attn_item(const StepArgs& a) {
  AttnItem it = {};
  const int S = a.splits, KVr = a.KVr, c = blockIdx.x;
  it.active = c < B * KVr * S;
  if (!it.active) return it;
  it.split = c % S;
  it.kvh = (c / S) % KVr;
  it.b = c / (S * KVr);
  int pos = a.pos[it.b];
  it.bad = pos < 0 || pos >= a.max_seq;
  if (it.bad) pos = 0;
  it.pos = pos;
  const int nkeys = it.bad ? 0 : pos + 1;
  const int chunk = (nkeys + S - 1) / S;
  it.k0 = min(nkeys, it.split * chunk);
  it.k1 = min(nkeys, it.k0 + chunk);
  it.s_active = chunk > 0 ? (nkeys + chunk - 1) / chunk : 0;
  return it;
}

// K/V rows [p0, p0 + 64) of the item (cached keys only: slot pos is this step's key, taken from
// shared memory).  Issued for the first block BEFORE the barrier that precedes the attention phase:
// the cache rows below pos were final before this step started.
template <int HD>
SIRIUS_DEV void attn_load_block(const StepArgs& a, int l, const AttnItem& it, int p0, uint4* kv, uint4* vv) {
  constexpr int VPR = HD / 8;
  constexpr int NL = (kKB * VPR + kNT - 1) / kNT;
  const int tid = threadIdx.x, nb = min(kKB, it.k1 - p0);
  const size_t hb = ((size_t)it.b * a.KVr + it.kvh) * a.max_seq;
  const uint16_t* kc = a.k_cache + (size_t)l * a.kv_layer + hb * HD;
  const uint16_t* vc = a.v_cache + (size_t)l * a.kv_layer + hb * HD;
#pragma unroll
  for (int j = 0; j < NL; ++j) {
    const int idx = tid + kNT * j, kk = idx / VPR, e = idx % VPR;
    if (kk < nb && p0 + kk != it.pos) {
      kv[j] = __ldcg(reinterpret_cast<const uint4*>(kc + (size_t)(p0 + kk) * HD + e * 8));
      vv[j] = __ldcg(reinterpret_cast<const uint4*>(vc + (size_t)(p0 + kk) * HD + e * 8));
    }
  }
}

// L1OK: the combine may read the (M_s, L_s) partials through L1 — only in the one-launch-per-layer
// item kernel (L1 does not survive kernel boundaries); the persistent step kernel reuses the
// partial buffer every layer within one launch, so it bypasses L1.
template <int B, int HD, int G, bool L1OK>
SIRIUS_DEV void attention_phase(const StepArgs& a, int l, StepSmem<B, HD, G>& sm, const AttnItem& it, uint4* kv,
                                uint4* vv) {
  constexpr int ROWB = HD * 2 + 16;  // padded K row (bytes): conflict-free row reads
  constexpr int VPR = HD / 8;        // uint4 per K/V row
  constexpr int NL = (kKB * VPR + kNT - 1) / kNT;
  if (!it.active) return;
  const int S = a.splits, KVr = a.KVr, Hr = a.Hr;
  const int split = it.split, kvh = it.kvh, b = it.b, pos = it.pos, k0 = it.k0, k1 = it.k1;
  const int s_active = it.s_active;
  const bool bad = it.bad;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (bad && tid == 0 && split == 0) atomicOr(a.err, 1);
  const size_t head_base = ((size_t)b * KVr + kvh) * a.max_seq;
  uint16_t* kc = a.k_cache + (size_t)l * a.kv_layer + head_base * HD;
  uint16_t* vc = a.v_cache + (size_t)l * a.kv_layer + head_base * HD;
  (void)NL;

  const float* qkv = a.qkv + (size_t)b * (Hr + 2 * KVr) * HD;
  const float* cs = a.rope_cos + (size_t)pos * (HD / 2);
  const float* sn = a.rope_sin + (size_t)pos * (HD / 2);
  for (int idx = tid; idx < G * (HD / 2); idx += kNT) {
    const int g = idx / (HD / 2), i = idx % (HD / 2);
    const float* q = qkv + (kvh * G + g) * HD;
    const float x0 = __ldcg(q + i), x1 = __ldcg(q + i + HD / 2), cc = cs[i], s = sn[i];
    sm.q_s[g][i] = (x0 * cc - x1 * s) * a.attn_scale;  // 1/sqrt(hd) folded into q
    sm.q_s[g][i + HD / 2] = (x1 * cc + x0 * s) * a.attn_scale;
  }
  if (tid < HD / 2) {
    const float* k = qkv + (Hr + kvh) * HD;
    const float x0 = __ldcg(k + tid), x1 = __ldcg(k + tid + HD / 2), cc = cs[tid], s = sn[tid];
    sm.kn_s[tid] = x0 * cc - x1 * s;
    sm.kn_s[tid + HD / 2] = x1 * cc + x0 * s;
  } else if (tid >= 64 && tid < 64 + HD) {
    sm.vn_s[tid - 64] = __ldcg(qkv + (Hr + KVr + kvh) * HD + tid - 64);
  }
  if (tid < G) {
    sm.m_s[tid] = -INFINITY;
    sm.l_s[tid] = 0.f;
  }
  __syncthreads();
  if (!bad && k0 <= pos && pos < k1) {  // this split owns slot pos: append the new K/V row
    for (int i = tid; i < HD; i += kNT) {
      kc[(size_t)pos * HD + i] = f2bf_bits(sm.kn_s[i]);
      vc[(size_t)pos * HD + i] = f2bf_bits(sm.vn_s[i]);
    }
  }
  stamp(a, l * kTraceSlots + 3);
  constexpr int NHO = (G * HD + kNT - 1) / kNT;  // (head, dim) outputs per thread
  float acc[NHO];
#pragma unroll
  for (int j = 0; j < NHO; ++j) acc[j] = 0.f;

  for (int p0 = k0; p0 < k1; p0 += kKB) {
    const int nb = min(kKB, k1 - p0);
#pragma unroll
    for (int j = 0; j < NL; ++j) {
      const int idx = tid + kNT * j, kk = idx / VPR, e = idx % VPR;
      if (kk < nb) {
        uint4 kw = kv[j], vw = vv[j];
        if (p0 + kk == pos) {
          const float* kn = sm.kn_s + e * 8;
          const float* vn = sm.vn_s + e * 8;
          kw = make_uint4(pack_bf16(kn[0], kn[1]), pack_bf16(kn[2], kn[3]), pack_bf16(kn[4], kn[5]),
                          pack_bf16(kn[6], kn[7]));
          vw = make_uint4(pack_bf16(vn[0], vn[1]), pack_bf16(vn[2], vn[3]), pack_bf16(vn[4], vn[5]),
                          pack_bf16(vn[6], vn[7]));
        }
        *reinterpret_cast<uint4*>(sm.k_s + kk * ROWB + e * 16) = kw;
        *reinterpret_cast<uint4*>(&sm.v_s[kk][e * 8]) = vw;
      }
    }
    __syncthreads();
    if (p0 + kKB < k1) attn_load_block<HD>(a, l, it, p0 + kKB, kv, vv);
    // scores: thread t -> (key t % kKB, head t / kKB)
    for (int t = tid; t < kKB * G; t += kNT) {
      const int kk = t % kKB, g = t / kKB;
      if (kk < nb) {
        float s = 0.f;
        const uint4* kr = reinterpret_cast<const uint4*>(sm.k_s + kk * ROWB);
#pragma unroll 4
        for (int e = 0; e < HD / 8; ++e) {
          const uint4 w = kr[e];
          const float4 q0 = *reinterpret_cast<const float4*>(&sm.q_s[g][e * 8]);
          const float4 q1 = *reinterpret_cast<const float4*>(&sm.q_s[g][e * 8 + 4]);
          s = fmaf(bf16_lo(w.x), q0.x, s); s = fmaf(bf16_hi(w.x), q0.y, s);
          s = fmaf(bf16_lo(w.y), q0.z, s); s = fmaf(bf16_hi(w.y), q0.w, s);
          s = fmaf(bf16_lo(w.z), q1.x, s); s = fmaf(bf16_hi(w.z), q1.y, s);
          s = fmaf(bf16_lo(w.w), q1.z, s); s = fmaf(bf16_hi(w.w), q1.w, s);
        }
        sm.sc[g][kk] = s;
      }
    }
    __syncthreads();
    // online softmax, warp g <-> head g
    for (int g = warp; g < G; g += kWarps) {
      const float x0 = lane < nb ? sm.sc[g][lane] : -INFINITY;
      const float x1 = lane + 32 < nb ? sm.sc[g][lane + 32] : -INFINITY;
      const float bm = warp_max(fmaxf(x0, x1));
      const float mold = sm.m_s[g];
      const float mn = fmaxf(mold, bm);
      const float p0v = lane < nb ? expf(x0 - mn) : 0.f;
      const float p1v = lane + 32 < nb ? expf(x1 - mn) : 0.f;
      sm.sc[g][lane] = p0v;
      sm.sc[g][lane + 32] = p1v;
      const float bs = warp_sum(p0v + p1v);
      __syncwarp();  // every lane has read m_s[g] before lane 0 rewrites it
      if (lane == 0) {
        const float corr = mold == -INFINITY ? 0.f : expf(mold - mn);
        sm.c_s[g] = corr;
        sm.l_s[g] = sm.l_s[g] * corr + bs;
        sm.m_s[g] = mn;
      }
    }
    __syncthreads();
    // P.V: thread -> outputs o = tid + kNT j = (head o / HD, dim o % HD)
#pragma unroll
    for (int j = 0; j < NHO; ++j) {
      const int o = tid + kNT * j;
      if (o < G * HD) {
        const int g = o / HD, dd = o % HD;
        float s = acc[j] * sm.c_s[g];
        for (int kk = 0; kk < nb; ++kk) s = fmaf(sm.sc[g][kk], __uint_as_float((uint32_t)sm.v_s[kk][dd] << 16), s);
        acc[j] = s;
      }
    }
    __syncthreads();
  }
  stamp(a, l * kTraceSlots + 4);
  // CTA partial (M, L, A[HD]) per q head of the group
  float* part = a.attn_part + (((size_t)b * KVr + kvh) * S + split) * G * (HD + 2);
#pragma unroll
  for (int j = 0; j < NHO; ++j) {
    const int o = tid + kNT * j;
    if (o < G * HD) {
      const int g = o / HD, dd = o % HD;
      part[g * (HD + 2) + 2 + dd] = acc[j];
      if (dd == 0) {
        part[g * (HD + 2)] = sm.m_s[g];
        part[g * (HD + 2) + 1] = sm.l_s[g];
      }
    }
  }
  // The LAST split of (b, kvh) to finish combines all of them; the others move on to the grid
  // barrier at once (no split-group wait).
  __syncthreads();  // this CTA's partial is written
  if (tid == 0) {
    unsigned* cnt = a.group_bar + 2 * (b * KVr + kvh);
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(old) : "l"(cnt) : "memory");
    const bool last = old == (unsigned)S - 1;
    if (last) *cnt = 0u;  // next use is after a grid barrier
    sm.flag_s = last ? 1u : 0u;
  }
  __syncthreads();
  stamp(a, l * kTraceSlots + 5);
  if (!sm.flag_s) return;
  // every thread: its outputs' partial values AND the (M, L) of the same head for all splits in
  // one round trip (batches of 32 splits), then M = max M_s, o = sum_s e^(M_s - M) A_s / sum_s e^(M_s - M) L_s
  const float* pb = a.attn_part + ((size_t)b * KVr + kvh) * S * G * (HD + 2);
  for (int o0 = tid; o0 < G * HD; o0 += kNT) {
    const int g = o0 / HD, dd = o0 % HD;
    float M = -INFINITY, Ls = 0.f, o = 0.f;
    for (int sp0 = 0; sp0 < s_active; sp0 += 32) {
      float mv[32], lv[32], av[32];
#pragma unroll
      for (int u = 0; u < 32; ++u) {
        const float* ps = pb + ((size_t)(sp0 + u) * G + g) * (HD + 2);
        const bool ok = sp0 + u < s_active;
        // (M_s, L_s) are shared by the HD threads of a head (L1-cached where that is safe)
        mv[u] = ok ? (L1OK ? __ldca(ps) : __ldcg(ps)) : -INFINITY;
        lv[u] = ok ? (L1OK ? __ldca(ps + 1) : __ldcg(ps + 1)) : 0.f;
        av[u] = ok ? __ldcg(ps + 2 + dd) : 0.f;
      }
      float Mb = M;
#pragma unroll
      for (int u = 0; u < 32; ++u) Mb = fmaxf(Mb, mv[u]);
      const float r = M == -INFINITY ? 0.f : expf(M - Mb);  // rescale the previous batches (s_active > 32)
      Ls *= r;
      o *= r;
#pragma unroll
      for (int u = 0; u < 32; ++u) {
        const float f = mv[u] == -INFINITY ? 0.f : expf(mv[u] - Mb);
        Ls += lv[u] * f;
        o += av[u] * f;
      }
      M = Mb;
    }
    const float val = Ls > 0.f ? o / Ls : 0.f;
    const size_t off = (size_t)b * Hr * HD + (kvh * G + g) * HD + dd;
    if (a.o3) {  // the row path's O-proj GEMM operand: val as three bf16 terms (exact)
      store_split3(a.o3, a.o3_plane, off, val);
    } else {
      a.o[off] = val;
    }
  }
}

// ------------------------------------------------------------------------------------------ P4
// CATS MLP of neurons [n0, n1) (same arithmetic as ffn_kernel phases A-D); the warp's first gate row
// was requested before the barrier (pf).  Writes the CTA's partial [B, d] and active counts.
template <int B, int CPL, bool RING, int HD, int G>
SIRIUS_DEV void ffn_phase(const StepArgs& a, int l, StepSmem<B, HD, G>& sm, const float4* hp,
                          RowStream<CPL, RING>& st) {
  constexpr int CPT = (CPL * 32 + kNT - 1) / kNT;          // down-proj column chunks per thread
  constexpr int RU = CPT == 1 ? 16 : (CPT == 2 ? 8 : 4);  // down rows in flight per thread
  const int d = a.d, CH = d / 8, Gd = gridDim.x, cta = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n0 = part_lo(a.F, cta, Gd), n1 = part_lo(a.F, cta + 1, Gd), nn = n1 - n0;
  const int nch = (nn + 31) / 32;
  const uint16_t* w_gate = a.w_gate[l];
  const uint16_t* w_up = a.w_up[l];
  const uint16_t* w_down = a.w_down[l];
  const float t = a.dense ? 0.f : a.thresholds[l];
  // A: dense gate rows -> a = SiLU(g)  (rows 0, 1 of the warp's stream requested before the barrier)
  auto gate_row = [&](int i) { return w_gate + (size_t)(n0 + warp + kWarps * i) * d; };
  rs_run<B, CPL, RING>(st, warp_rows(0, nn, warp), gate_row, hp, CH, lane, [&](int i, const float* acc) {
    if (lane == 0) {
#pragma unroll
      for (int b = 0; b < B; ++b) sm.a_s[b][warp + kWarps * i] = acc[b] / (1.0f + expf(-acc[b]));
    }
  });
  __syncthreads();
  stamp(a, l * kTraceSlots + 12);
  // B: CATS threshold |a| >= t, warp-ballot compaction (warp c <-> 32-neuron chunk c)
  unsigned um = 0u;
  for (int cw = warp; cw < nch; cw += kWarps) {  // nch <= 8 < kWarps: one chunk per warp
    const int i = cw * 32 + lane;
    const bool valid = i < nn;
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const float av = valid ? sm.a_s[b][i] : 0.f;
      const bool on = valid && (a.dense || fabsf(av) >= t);
      const unsigned mb = __ballot_sync(0xffffffffu, on);
      um |= mb;
      if (lane == 0) sm.act_s[cw][b] = mb;
      if (a.gate_out && valid) a.gate_out[(size_t)b * a.gate_stride + (size_t)l * a.F + n0 + i] = av;
    }
    if (lane == 0) sm.cnt_s[cw] = __popc(um);
  }
  __syncthreads();
  if (tid == 0) {
    int s = 0;
    for (int cc = 0; cc < nch; ++cc) {
      sm.off_s[cc] = s;
      s += sm.cnt_s[cc];
    }
    sm.off_s[nch] = s;
  }
  __syncthreads();
  if (warp < nch && ((um >> lane) & 1u)) {
    const int k = sm.off_s[warp] + __popc(um & ((1u << lane) - 1u));
    sm.list_s[k] = warp * 32 + lane;
    unsigned char bits = 0;
#pragma unroll
    for (int b = 0; b < B; ++b) bits |= (unsigned char)(((sm.act_s[warp][b] >> lane) & 1u) << b);
    sm.bits_s[k] = bits;
  }
  __syncthreads();
  const int nact = sm.off_s[nch];
  stamp(a, l * kTraceSlots + 13);
  // C: ACTIVE up rows only: m = a * u (inactive (b, n) pairs contribute 0)
  {
    auto up_row = [&](int i) {
      const int k = warp + kWarps * i;
      return w_up + (size_t)(n0 + sm.list_s[k < nact ? k : 0]) * d;
    };
    const int nw = warp_rows(0, nact, warp);
    rs_start<CPL, RING>(st, nw, up_row, CH, lane);
    rs_run<B, CPL, RING>(st, nw, up_row, hp, CH, lane, [&](int i, const float* acc) {
      const int k = warp + kWarps * i, n = sm.list_s[k];
      if (lane == 0) {
#pragma unroll
        for (int b = 0; b < B; ++b) sm.mm_s[b][k] = ((sm.bits_s[k] >> b) & 1u) ? sm.a_s[b][n] * acc[b] : 0.f;
      }
    });
  }
  __syncthreads();
  stamp(a, l * kTraceSlots + 14);
  // D: ACTIVE down rows only, thread owns column chunks tid + kNT j
  float y[B][CPT * 8];
#pragma unroll
  for (int b = 0; b < B; ++b)
#pragma unroll
    for (int e = 0; e < CPT * 8; ++e) y[b][e] = 0.f;
  for (int k0 = 0; k0 < nact; k0 += RU) {
    uint4 wv[RU][CPT];
#pragma unroll
    for (int r = 0; r < RU; ++r) {
      const int k = k0 + r;
      const uint16_t* wrow = w_down + (size_t)(n0 + (k < nact ? sm.list_s[k] : 0)) * d;
#pragma unroll
      for (int j = 0; j < CPT; ++j) {
        const int ch = tid + kNT * j;
        wv[r][j] = (k < nact && ch < CH) ? ld_nc_v4_ef(wrow + (size_t)ch * 8, st.pol) : make_uint4(0u, 0u, 0u, 0u);
      }
    }
#pragma unroll
    for (int r = 0; r < RU; ++r) {
      const int k = k0 + r;
      if (k < nact) {
#pragma unroll
        for (int j = 0; j < CPT; ++j) {
          const uint4 w = wv[r][j];
          const float wf[8] = {bf16_lo(w.x), bf16_hi(w.x), bf16_lo(w.y), bf16_hi(w.y),
                               bf16_lo(w.z), bf16_hi(w.z), bf16_lo(w.w), bf16_hi(w.w)};
#pragma unroll
          for (int b = 0; b < B; ++b) {
            const float mk = sm.mm_s[b][k];
#pragma unroll
            for (int e = 0; e < 8; ++e) y[b][j * 8 + e] = fmaf(mk, wf[e], y[b][j * 8 + e]);
          }
        }
      }
    }
  }
  // y_c added into the residual stream (x1, in place) with vector float atomics: the sum over the
  // CTAs' partials needs no separate reduction pass or barrier (its order varies run to run)
#pragma unroll
  for (int j = 0; j < CPT; ++j) {
    const int ch = tid + kNT * j;
    if (ch < CH && nact > 0) {
#pragma unroll
      for (int b = 0; b < B; ++b) {
        float4* dst = reinterpret_cast<float4*>(a.x + (size_t)b * d + ch * 8);
        atomicAdd(dst, make_float4(y[b][j * 8 + 0], y[b][j * 8 + 1], y[b][j * 8 + 2], y[b][j * 8 + 3]));
        atomicAdd(dst + 1, make_float4(y[b][j * 8 + 4], y[b][j * 8 + 5], y[b][j * 8 + 6], y[b][j * 8 + 7]));
      }
    }
  }
  if (a.n_active_out && tid < B) {
    int cnt = 0;
    for (int cc = 0; cc < nch; ++cc) cnt += __popc(sm.act_s[cc][tid]);
    atomicAdd(a.n_active_out + (size_t)tid * a.L + l, cnt);
  }
}

// ------------------------------------------------------------------------------------------ kernel
// Per-warp shared-memory row slot (2 rows in flight per warp): measured SLOWER on B200 (3.29 vs
// 2.88 ms per 8B step: the bulk-copied half of the rows and the L1 carve-out cost more than the
// extra depth gains), so it is compiled out; kept for the record / re-measurement.
template <int B, int CPL>
constexpr bool step_ring() {
  return false && CPL <= 16 && B <= 2;
}

template <int B, int CPL, int HD, int G>
constexpr size_t step_smem_bytes(int d) {
  constexpr size_t head = (sizeof(StepSmem<B, HD, G>) + 127) / 128 * 128;
  constexpr size_t ring = step_ring<B, CPL>() ? (size_t)kWarps * (CPL * 32 * 16 + 16) : 0;
  return head + ring + (size_t)B * d * 4;
}

template <int B, int CPL, int HD, int G>
__global__ void __launch_bounds__(kNT, 1) decode_step_kernel(StepArgs a) {
  constexpr bool RING = step_ring<B, CPL>();
  constexpr int kPG = CPL * 64 / kNT > 0 ? CPL * 64 / kNT : 1;  // prologue float4 groups per thread
  constexpr size_t kHead = (sizeof(StepSmem<B, HD, G>) + 127) / 128 * 128;
  constexpr size_t kSlot = (size_t)CPL * 32 * 16;  // one row: 32 CPL uint4 (= d bf16)
  extern __shared__ __align__(128) uint8_t smem_raw[];
  StepSmem<B, HD, G>& sm = *reinterpret_cast<StepSmem<B, HD, G>*>(smem_raw);
  uint8_t* ring = smem_raw + kHead;  // [kWarps] row slots, then [kWarps] mbarriers
  float* h_s = reinterpret_cast<float*>(ring + (RING ? kWarps * (kSlot + 16) : 0));  // [B][2][CH] float4 planes
  const int d = a.d, CH = d / 8, L = a.L, Gd = gridDim.x, cta = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int Nqkv = (a.Hr + 2 * a.KVr) * HD;
  const float4* hp = reinterpret_cast<const float4*>(h_s);
  RowStream<CPL, RING> st;
  st.slot = reinterpret_cast<uint4*>(ring + warp * kSlot);
  st.bar = reinterpret_cast<uint64_t*>(ring + kWarps * kSlot) + warp;
  st.phase = 0u;
  st.pol = (a.tune & 1) ? policy_evict_first() : policy_evict_unchanged();
  if (RING && lane == 0) mbar_init(st.bar, 1);
  fence_mbar_init();
  __syncthreads();
  const int q0 = part_lo(Nqkv, cta, Gd), q1 = part_lo(Nqkv, cta + 1, Gd);
  const int o0 = part_lo(d, cta, Gd), o1 = part_lo(d, cta + 1, Gd);
  const int f0 = part_lo(a.F, cta, Gd), f1 = part_lo(a.F, cta + 1, Gd);
  const int v0 = part_lo(a.Vr, cta, Gd), v1 = part_lo(a.Vr, cta + 1, Gd);
  const int nq = warp_rows(q0, q1, warp), no = warp_rows(o0, o1, warp), nf = warp_rows(f0, f1, warp);
  const int nv = warp_rows(v0, v1, warp);
  auto qkv_row = [&](int l) { return [=](int i) { return a.w_qkv[l] + (size_t)(q0 + warp + kWarps * i) * d; }; };
  auto o_row = [&](int l) { return [=](int i) { return a.w_o[l] + (size_t)(o0 + warp + kWarps * i) * d; }; };
  auto gate_row = [&](int l) { return [=](int i) { return a.w_gate[l] + (size_t)(f0 + warp + kWarps * i) * d; }; };
  auto head_row = [&](int i) { return a.lm_head + (size_t)(v0 + warp + kWarps * i) * d; };
  rs_start<CPL, RING>(st, nq, qkv_row(0), CH, lane);
  const AttnItem it = attn_item<B>(a);  // this CTA's attention work item (same every layer)
  stamp(a, -1);

  for (int l = 0; l < L; ++l) {
    // ---------------- P1: RMSNorm(y) + QKV rows
    {
      Prologue p = {};
      if (l == 0) {
        p.mode = IN_EMBED;
        p.tokens = a.tokens;
        p.embed = a.embed;
        p.vocab = a.vocab;
        p.res_out = a.x;  // CTA 0 stores the residual stream y = E[tok]
      } else {
        p.mode = IN_RESID;
        p.base = a.x;
      }
      p.norm_w = a.attn_norm[l];
      p.eps = a.eps;
      prologue<B, kPG>(p, d, h_s, sm.red_s, cta == 0);
      stamp(a, l * kTraceSlots + 0);
      rs_run<B, CPL, RING>(st, nq, qkv_row(l), hp, CH, lane, [&](int i, const float* acc) {
        if (lane == 0) {
#pragma unroll
          for (int b = 0; b < B; ++b) a.qkv[(size_t)b * Nqkv + q0 + warp + kWarps * i] = acc[b];
        }
      });
    }
    // first K/V block of this CTA's attention item, requested before the barrier
    uint4 kv[kKB * HD / 8 / kNT > 0 ? kKB * HD / 8 / kNT : 1], vv[kKB * HD / 8 / kNT > 0 ? kKB * HD / 8 / kNT : 1];
    if (it.active && it.k0 < it.k1) attn_load_block<HD>(a, l, it, it.k0, kv, vv);
    stamp(a, l * kTraceSlots + 1);
    grid_sync(a.grid_bar, Gd);
    stamp(a, l * kTraceSlots + 2);
    // ---------------- P2: attention (RoPE, K/V append, split-K, last-split combine)
    attention_phase<B, HD, G, false>(a, l, sm, it, kv, vv);
    rs_start<CPL, RING>(st, no, o_row(l), CH, lane);
    stamp(a, l * kTraceSlots + 6);
    grid_sync(a.grid_bar, Gd);
    stamp(a, l * kTraceSlots + 7);
    // ---------------- P3: O-proj + residual add: x1 = y + o W_o^T
    {
      Prologue p = {};
      p.mode = IN_F32;
      p.in_f32 = a.o;
      prologue<B, kPG>(p, d, h_s, sm.red_s, false);
      stamp(a, l * kTraceSlots + 8);
      rs_run<B, CPL, RING>(st, no, o_row(l), hp, CH, lane, [&](int i, const float* acc) {
        if (lane == 0) {
          const int row = o0 + warp + kWarps * i;
#pragma unroll
          for (int b = 0; b < B; ++b) {  // in place in the residual stream y (the FFN adds into it),
            const float x1 = __ldcg(a.x + (size_t)b * d + row) + acc[b];  // and a stable copy for the FFN
            a.x[(size_t)b * d + row] = x1;
            a.x1[(size_t)b * d + row] = x1;
          }
        }
      });
    }
    rs_start<CPL, RING>(st, nf, gate_row(l), CH, lane);
    stamp(a, l * kTraceSlots + 9);
    grid_sync(a.grid_bar, Gd);
    stamp(a, l * kTraceSlots + 10);
    // ---------------- P4: CATS MLP, partial added into y
    {
      Prologue p = {};
      p.mode = IN_RESID;
      p.base = a.x1;
      p.norm_w = a.ffn_norm[l];
      p.eps = a.eps;
      prologue<B, kPG>(p, d, h_s, sm.red_s, false);
      stamp(a, l * kTraceSlots + 11);
      ffn_phase<B, CPL, RING, HD, G>(a, l, sm, hp, st);
    }
    if (l + 1 < L) rs_start<CPL, RING>(st, nq, qkv_row(l + 1), CH, lane);
    else rs_start<CPL, RING>(st, nv, head_row, CH, lane);
    stamp(a, l * kTraceSlots + 15);
    grid_sync(a.grid_bar, Gd);
    stamp(a, l * kTraceSlots + 16);
  }
  // ---------------- final RMSNorm + LM head + packed argmax
  {
    stamp(a, L * kTraceSlots);
    Prologue p = {};
    p.mode = IN_RESID;
    p.base = a.x;
    p.norm_w = a.final_norm;
    p.eps = a.eps;
    prologue<B, kPG>(p, d, h_s, sm.red_s, false);
    unsigned long long best[B];
#pragma unroll
    for (int b = 0; b < B; ++b) best[b] = 0ull;
    rs_run<B, CPL, RING>(st, nv, head_row, hp, CH, lane, [&](int i, const float* acc) {
      if (lane == 0) {
        const int row = v0 + warp + kWarps * i;
#pragma unroll
        for (int b = 0; b < B; ++b) {
          if (a.logits_out) a.logits_out[(size_t)b * a.Vr + row] = acc[b];
          const unsigned long long k = argmax_key(acc[b], (uint32_t)row);
          best[b] = k > best[b] ? k : best[b];
        }
      }
    });
    if (lane == 0) {
#pragma unroll
      for (int b = 0; b < B; ++b) sm.key_s[warp * B + b] = best[b];
    }
    __syncthreads();
    if (tid < B) {
      unsigned long long k = 0ull;
      for (int w = 0; w < kWarps; ++w) k = sm.key_s[w * B + tid] > k ? sm.key_s[w * B + tid] : k;
      atomicMax(a.amax + tid, k);
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      const unsigned old = atomicAdd(a.head_cnt, 1u);
      const bool last = old == (unsigned)Gd - 1;
      if (last) {
        atomicExch(a.head_cnt, 0u);
        __threadfence();
      }
      sm.flag_s = last ? 1u : 0u;
    }
    __syncthreads();
    if (sm.flag_s && tid < B) {
      const unsigned long long k = atomicExch(a.amax + tid, 0ull);  // read + reset for the next step
      a.token_out[tid] = (int32_t)argmax_key_index(k);
    }
    stamp(a, L * kTraceSlots + 1);
  }
}

// The attention phase alone, as the per-stage schedule's attention kernel (one (b, kv head, split)
// item per CTA, RoPE + K/V append + split-K + last-split combine; no co-residency needed).
template <int B, int HD, int G>
__global__ void __launch_bounds__(kNT, 1) attn_stage_kernel(StepArgs a, int l) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  StepSmem<B, HD, G>& sm = *reinterpret_cast<StepSmem<B, HD, G>*>(smem_raw);
  const AttnItem it = attn_item<B>(a);
  constexpr int NL = kKB * HD / 8 / kNT > 0 ? kKB * HD / 8 / kNT : 1;
  uint4 kv[NL], vv[NL];
  if (it.active && it.k0 < it.k1) attn_load_block<HD>(a, l, it, it.k0, kv, vv);
  // PDL (decode chain): the positions are inputs of the step and the cached K/V rows below pos were
  // final before the step; the q / k / v of the QKV GEMV (the predecessor) only after the wait
  pdl_wait();
  pdl_trigger();
  attention_phase<B, HD, G, true>(a, l, sm, it, kv, vv);
}

template <int B, int HD, int G>
cudaError_t launch_attn_stage(const StepArgs& a, int l, cudaStream_t st) {
  auto kern = attn_stage_kernel<B, HD, G>;
  const size_t smem = (sizeof(StepSmem<B, HD, G>) + 127) / 128 * 128;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch::launch_pdl(launch::g_decode_pdl, kern, dim3(B * a.KVr * a.splits), dim3(kNT), smem, st, a, l);
}

template <int HD, int G>
cudaError_t attn_stage_b(const StepArgs& a, int l, int B, cudaStream_t st) {
  switch (B) {
    case 1: return launch_attn_stage<1, HD, G>(a, l, st);
    case 2: return launch_attn_stage<2, HD, G>(a, l, st);
    case 4: return launch_attn_stage<4, HD, G>(a, l, st);
    case 8: return launch_attn_stage<8, HD, G>(a, l, st);
    case 16: return launch_attn_stage<16, HD, G>(a, l, st);
    case 32: return launch_attn_stage<32, HD, G>(a, l, st);
    default: return cudaErrorInvalidValue;
  }
}

template <int B, int CPL, int HD, int G>
cudaError_t launch_step(const StepArgs& a, int grid, cudaStream_t st) {
  auto kern = decode_step_kernel<B, CPL, HD, G>;
  const size_t smem = step_smem_bytes<B, CPL, HD, G>(a.d);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kNT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // co-residency for the grid barriers
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

template <int CPL, int HD, int G>
cudaError_t launch_b(const StepArgs& a, int B, int grid, cudaStream_t st) {
  switch (B) {
    case 1: return launch_step<1, CPL, HD, G>(a, grid, st);
    case 2: return launch_step<2, CPL, HD, G>(a, grid, st);
    case 4: return launch_step<4, CPL, HD, G>(a, grid, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

namespace launch {

// The persistent step covers the shapes it is instantiated for: Llama-3-8B / 70B (hd 128, GQA group
// 4 / 8, d 4096 / 8192) and the tiny test decoder (d 256, hd 64, group 2), TP 1, H hd == d.
bool decode_step_supported(int d, int H, int KV, int hd, int F, int num_sms) {
  if (H * hd != d || (F + num_sms - 1) / num_sms > kMaxN) return false;
  const int G = H / KV;
  return (d == 4096 && hd == 128 && G == 4) || (d == 8192 && hd == 128 && G == 8) || (d == 256 && hd == 64 && G == 2);
}

int decode_step_splits(int B, int KV, int num_sms) {
  int s = num_sms / (B * KV);
  return s < 1 ? 1 : (s > kMaxSplits ? kMaxSplits : s);
}

bool attn_stage_supported(int hd, int G) { return (hd == 128 && (G == 4 || G == 8)) || (hd == 64 && G == 2); }

cudaError_t attn_stage(const StepArgs& a, int l, int B, cudaStream_t st) {
  const int G = a.Hr / a.KVr;
  if (a.hd == 128 && G == 4) return attn_stage_b<128, 4>(a, l, B, st);
  if (a.hd == 128 && G == 8) return attn_stage_b<128, 8>(a, l, B, st);
  if (a.hd == 64 && G == 2) return attn_stage_b<64, 2>(a, l, B, st);
  return cudaErrorInvalidValue;
}

cudaError_t decode_step(const StepArgs& a, int B, int grid, cudaStream_t st) {
  const int G = a.Hr / a.KVr;
  if (a.d == 4096 && a.hd == 128 && G == 4) return launch_b<16, 128, 4>(a, B, grid, st);
  if (a.d == 8192 && a.hd == 128 && G == 8) return launch_b<32, 128, 8>(a, B, grid, st);
  if (a.d == 256 && a.hd == 64 && G == 2) return launch_b<1, 64, 2>(a, B, grid, st);
  return cudaErrorInvalidValue;
}

}  // namespace launch
}  // namespace sirius
