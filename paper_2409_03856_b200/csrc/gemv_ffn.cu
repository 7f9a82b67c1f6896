// gemv_ffn.cu — the HBM-bound weight-streaming kernels of the decode step.
//
//  * gemv_kernel : y[b, r] = sum_k W[r, k] h[b, k] for the QKV, O-proj and LM-head GEMVs.  One warp per
//                  row; every lane issues all of its 128-bit weight loads for the row before using
//                  them (16 KB+ in flight per warp, 2 CTAs x 8 warps per SM), the fp32 activation rows
//                  sit in shared memory as two float4 "planes" so the per-chunk reads are
//                  bank-conflict free; warp-shuffle reduction.  Prologue fuses residual add + RMSNorm
//                  (or the embedding gather).  Epilogues: store, or packed (value, lowest index) argmax.
//  * ffn_kernel  : the CATS-sparse MLP of one layer in one
//                  launch, neurons split evenly over the CTAs:
//                    A  dense gate rows -> g -> a = SiLU(g)                        (warp per row)
//                    B  CATS threshold |a| >= t_l, warp-ballot compaction per 32-neuron chunk
//                    C  ACTIVE W_up rows only -> u -> m = a * u                    (warp per row)
//                    D  ACTIVE W_down rows only -> y += m * W_down[n]   (threads own output columns)
//                  so HBM bytes scale with the density.  Default (atomic mode): 8-warp CTAs, 2 per SM,
//                  partials added into the pre-zeroed output with float4 atomics.  SIRIUS_FFN_ATOMIC=0:
//                  16-warp CTAs, one per SM, cooperative launch, grid barrier and a deterministic
//                  fixed-order column reduction of the per-CTA partials.
// Decode chain: both kernels are launched with programmatic dependent launch; each warp's
// first weight row is requested before griddepcontrol.wait (weights only), the dependent is triggered
// right after it.  TP > 1 with sirius_par_enable: the rank partial is all-reduced in the kernel's tail
// over NVLink peer memory (peer_ar.cuh).
// Design note: 1-D bulk-copy (TMA) staging of 8 KB rows caps at ~3.3 TB/s with a reader
// (TMA ops have a fixed per-op cost; tools/bw_probe.cu, profiles/r02_bw_probe*.txt), direct 128-bit
// loads with many rows in flight reach ~7.3 TB/s.
// Numeric contract (D15): bf16 weights, fp32 activations and accumulation.
#include "common.cuh"
#include "decode_kernels.cuh"
#include "gemv_dev.cuh"
#include "peer_ar.cuh"

namespace sirius {
namespace {

constexpr int kGemvWarps = 8;   // 2 CTAs per SM
constexpr int kFfnWarps = 16;   // 1 CTA per SM (cooperative)
constexpr int kFfnMaxN = 256;   // neurons per CTA
constexpr int kFfnMaxChunks = kFfnMaxN / 32;
using dev::after_all;
using dev::prologue;
using dev::row_dot;
using dev::row_finish;
using dev::row_issue;
using dev::RowRegs;

// ===================================================================== dense GEMV
template <int B, int CPL>
__global__ void __launch_bounds__(kGemvWarps * 32, 2) gemv_kernel(GemvArgs a) {
  extern __shared__ __align__(16) float h_s[];  // [B][2][CH] float4
  __shared__ float red_s[32];
  __shared__ unsigned long long key_s[kGemvWarps * B];
  __shared__ unsigned flag_s;
  const int K = a.K, CH = K / 8;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint64_t pol = policy_evict_first();  // weights: read once per step
  const int r0 = (int)((long long)a.rows * blockIdx.x / gridDim.x);
  const int r1 = (int)((long long)a.rows * (blockIdx.x + 1) / gridDim.x);
  // the warp's first weight row is requested before the activation prologue (it does not depend on
  // it); afterwards each row's loads go out before the previous row's reduction
  RowRegs<CPL> pf;
  row_issue<CPL>(pf, a.W + (size_t)(r0 + warp) * K, CH, lane, r0 + warp < r1, pol);
  // PDL (decode chain): everything above reads weights only; the predecessor's outputs after the wait
  pdl_wait();
  pdl_trigger();
  if (a.zero_out) {  // the next FFN's accumulator (its previous contents were consumed upstream)
    const int z0 = (int)((long long)a.zero_n * blockIdx.x / gridDim.x);
    const int z1 = (int)((long long)a.zero_n * (blockIdx.x + 1) / gridDim.x);
    for (int i = z0 + tid; i < z1; i += blockDim.x) a.zero_out[i] = 0.f;
  }
  constexpr int MG = CPL / 4 > 0 ? CPL / 4 : 1;  // prologue float4 groups per thread (K <= 256 CPL)
  prologue<B, MG>(a.pro, K, h_s, red_s, blockIdx.x == 0);
  const float4* hp = reinterpret_cast<const float4*>(h_s);
  unsigned long long best[B];
#pragma unroll
  for (int b = 0; b < B; ++b) best[b] = 0ull;
  for (int row = r0 + warp; row < r1; row += kGemvWarps) {
    float acc[B];
    row_finish<B, CPL>(pf, a.W + (size_t)row * K, hp, CH, lane, acc);
    row_issue<CPL>(pf, a.W + (size_t)(row + kGemvWarps) * K + after_all<B>(acc), CH, lane, row + kGemvWarps < r1,
                   pol);
#pragma unroll
    for (int b = 0; b < B; ++b) acc[b] = warp_sum(acc[b]);
    if (lane == 0) {
#pragma unroll
      for (int b = 0; b < B; ++b) {
        if (a.out) a.out[(size_t)b * a.ldo + row] = acc[b];
        if (a.epi == EPI_ARGMAX) {
          const unsigned long long k = argmax_key(acc[b], a.index_offset + (uint32_t)row);
          best[b] = k > best[b] ? k : best[b];
        }
      }
    }
  }
  if (a.epi != EPI_ARGMAX) {
    if (a.par.world) par::push_last(a.par, a.out, B * a.ldo, nullptr, 0, nullptr);  // fused all-reduce (TP > 1)
    return;
  }
  if (lane == 0)
    for (int b = 0; b < B; ++b) key_s[warp * B + b] = best[b];
  __syncthreads();
  if (tid < B) {
    unsigned long long k = 0ull;
    for (int w = 0; w < kGemvWarps; ++w) k = key_s[w * B + tid] > k ? key_s[w * B + tid] : k;
    atomicMax(a.amax + tid, k);
  }
  if (a.par.world) {  // TP > 1: the rank's packed keys go to every rank, max-reduced -> token (fused)
    par::push_last(a.par, nullptr, 0, a.amax, B, a.token_out);
    return;
  }
  if (a.finalize) {
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      const unsigned old = atomicAdd(a.done_counter, 1u);
      const bool last = old == gridDim.x - 1;
      if (last) {
        atomicExch(a.done_counter, 0u);
        __threadfence();
      }
      flag_s = last ? 1u : 0u;
    }
    __syncthreads();
    if (flag_s && tid < B) {
      const unsigned long long k = atomicExch(a.amax + tid, 0ull);  // read + reset for the next step
      a.token_out[tid] = (int32_t)argmax_key_index(k);
    }
  }
}

// TP > 1: the per-rank packed keys were max-reduced across ranks (NCCL) -> token, amax reset
__global__ void argmax_finalize_kernel(unsigned long long* amax, int B, int32_t* token_out) {
  const int b = threadIdx.x;
  if (b < B) {
    const unsigned long long k = amax[b];
    amax[b] = 0ull;
    token_out[b] = (int32_t)argmax_key_index(k);
  }
}

// Single-GPU TP emulation of the fused all-reduce (PeerAr.fused = 0): after every emulated rank's
// producer has pushed, each rank's reduction runs here — the same wait + rank-order reduction the
// producer's last CTA runs when fused (dst: the partial, all-reduced in place; keys -> token_out)
__global__ void par_reduce_kernel(PeerAr p, float* dst, int n, int nk, int32_t* token_out) {
  const unsigned long long s = __ldcg(p.seq);
  par::wait_flags(p, s);
  par::reduce(p, (int)(s & 1ull), dst, n, nk, nullptr, token_out);
}

// ===================================================================== fused CATS FFN
SIRIUS_DEV void fstamp(const FfnArgs& a, int slot) {  // debug phase stamps (a.trace != NULL)
  if (!a.trace) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[(size_t)slot * 1024 + blockIdx.x] = t;
  }
}

// NW warps per CTA: 16 with one CTA per SM (deterministic mode: cooperative grid barrier + column
// reduction), 8 with several small CTAs per SM (atomic mode: the hardware scheduler balances the
// data-dependent up/down work across SMs and one CTA's prologue overlaps another's weight stream).
template <int B, int CPL, int CPT, int NW>
__global__ void __launch_bounds__(NW * 32, NW == 8 ? 2 : 1) ffn_kernel(FfnArgs a) {
  constexpr int kFfnWarps = NW;
  fstamp(a, 0);
  extern __shared__ __align__(16) float h_s[];  // [B][2][CH] float4
  __shared__ float red_s[32];
  __shared__ float a_s[B][kFfnMaxN];            // a = SiLU(g) of the CTA's neurons
  __shared__ float m_s[B][kFfnMaxN];            // m = a * u, in active-list order
  __shared__ int list_s[kFfnMaxN];              // active neurons (local index), ascending
  __shared__ unsigned char bits_s[kFfnMaxN];    // per active neuron: which batch rows are active
  __shared__ unsigned act_s[kFfnMaxChunks][B];
  __shared__ int cnt_s[kFfnMaxChunks], off_s[kFfnMaxChunks + 1];
  constexpr int NT = kFfnWarps * 32;
  const int d = a.d, CH = d / 8;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = gridDim.x, cta = blockIdx.x;
  const int n0 = (int)((long long)a.F * cta / G), n1 = (int)((long long)a.F * (cta + 1) / G), nn = n1 - n0;
  const int nch = (nn + 31) / 32;

  const uint64_t pol = policy_evict_first();
  RowRegs<CPL> pf;  // first gate row of the warp, requested before the activation prologue
  row_issue<CPL>(pf, a.w_gate + (size_t)(n0 + warp) * d, CH, lane, warp < nn && !a.a_in, pol);
  pdl_wait();  // PDL (decode chain): only weights were read above
  pdl_trigger();
  constexpr int MG = CPL * 2 / NW > 0 ? CPL * 2 / NW : 1;  // prologue float4 groups per thread (d = 256 CPL)
  prologue<B, MG>(a.pro, d, h_s, red_s, cta == 0);
  fstamp(a, 1);
  const float4* hp = reinterpret_cast<const float4*>(h_s);
  const float t = a.dense ? 0.f : *a.threshold;

  // ---- A: dense gate rows: g = h2 . W_gate[n];  a = SiLU(g)  (precomputed-gate mode: loaded)
  if (a.a_in) {
    for (int i = tid; i < nn; i += NT)
#pragma unroll
      for (int b = 0; b < B; ++b) a_s[b][i] = __ldcg(a.a_in + (size_t)b * a.a_ld + n0 + i);
  }
  for (int i = warp; i < nn && !a.a_in; i += kFfnWarps) {
    float acc[B];
    row_finish<B, CPL>(pf, a.w_gate + (size_t)(n0 + i) * d, hp, CH, lane, acc);
    row_issue<CPL>(pf, a.w_gate + (size_t)(n0 + i + kFfnWarps) * d + after_all<B>(acc), CH, lane, i + kFfnWarps < nn,
                   pol);
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const float g = warp_sum(acc[b]);
      if (lane == 0) a_s[b][i] = g / (1.0f + expf(-g));
    }
  }
  __syncthreads();
  fstamp(a, 2);
  // ---- B: CATS threshold |a| >= t and warp-ballot compaction (warp c <-> 32-neuron chunk c)
  unsigned um = 0u;
  if (warp < nch) {
    const int i = warp * 32 + lane;
    const bool valid = i < nn;
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const float av = valid ? a_s[b][i] : 0.f;
      bool sel = fabsf(av) >= t;
      if (a.mask_in && valid) sel = (__ldcg(a.mask_in + (size_t)b * a.m_ld + ((n0 + i) >> 5)) >> ((n0 + i) & 31)) & 1u;
      const bool on = valid && (a.dense || sel);
      const unsigned mb = __ballot_sync(0xffffffffu, on);
      um |= mb;
      if (lane == 0) act_s[warp][b] = mb;
      if (a.gate_out && valid) a.gate_out[(size_t)b * a.gate_stride + n0 + i] = av;
    }
    if (lane == 0) cnt_s[warp] = __popc(um);
  }
  __syncthreads();
  if (tid == 0) {
    int s = 0;
    for (int c = 0; c < nch; ++c) {
      off_s[c] = s;
      s += cnt_s[c];
    }
    off_s[nch] = s;
  }
  __syncthreads();
  if (warp < nch && ((um >> lane) & 1u)) {
    const int k = off_s[warp] + __popc(um & ((1u << lane) - 1u));
    list_s[k] = warp * 32 + lane;
    unsigned char bits = 0;
#pragma unroll
    for (int b = 0; b < B; ++b) bits |= (unsigned char)(((act_s[warp][b] >> lane) & 1u) << b);
    bits_s[k] = bits;
  }
  __syncthreads();
  const int nact = off_s[nch];
  fstamp(a, 3);
  // ---- C: active up rows only: u = h2 . W_up[n];  m = a * u  (inactive (b, n) pairs contribute 0)
  // (each warp's next up row requested before the current row's reduction, as for the gate rows)
  row_issue<CPL>(pf, a.w_up + (size_t)(n0 + list_s[warp < nact ? warp : 0]) * d, CH, lane, warp < nact, pol);
  for (int k = warp; k < nact; k += kFfnWarps) {
    const int i = list_s[k];
    float acc[B];
    row_finish<B, CPL>(pf, a.w_up + (size_t)(n0 + i) * d, hp, CH, lane, acc);
    const int kn = k + kFfnWarps < nact ? k + kFfnWarps : k;
    row_issue<CPL>(pf, a.w_up + (size_t)(n0 + list_s[kn]) * d + after_all<B>(acc), CH, lane, k + kFfnWarps < nact,
                   pol);
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const float u = warp_sum(acc[b]);
      if (lane == 0) m_s[b][k] = ((bits_s[k] >> b) & 1u) ? a_s[b][i] * u : 0.f;
    }
  }
  __syncthreads();
  fstamp(a, 4);
  // ---- D: active down rows only: y += m * W_down[n]; thread owns column chunks tid + NT j
  // rows in flight per thread (fewer for B = 8: the y[B][.] accumulators share the registers)
  constexpr int RU = (CPT == 1 ? 16 : (CPT == 2 ? 8 : 4)) / (B >= 8 ? 2 : 1);
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
      const uint16_t* wrow = a.w_down + (size_t)(n0 + (k < nact ? list_s[k] : 0)) * d;
#pragma unroll
      for (int j = 0; j < CPT; ++j) {
        const int ch = tid + NT * j;
        wv[r][j] = (k < nact && ch < CH) ? ld_nc_v4_ef(wrow + (size_t)ch * 8, pol) : make_uint4(0u, 0u, 0u, 0u);
      }
    }
#pragma unroll
    for (int r = 0; r < RU; ++r) {
      const int k = k0 + r;
      if (k < nact) {  // ascending neuron order, same for every column
#pragma unroll
        for (int j = 0; j < CPT; ++j) {
          const uint4 w = wv[r][j];
          const float wf[8] = {bf16_lo(w.x), bf16_hi(w.x), bf16_lo(w.y), bf16_hi(w.y),
                               bf16_lo(w.z), bf16_hi(w.z), bf16_lo(w.w), bf16_hi(w.w)};
#pragma unroll
          for (int b = 0; b < B; ++b) {
            const float mk = m_s[b][k];
#pragma unroll
            for (int e = 0; e < 8; ++e) y[b][j * 8 + e] = fmaf(mk, wf[e], y[b][j * 8 + e]);
          }
        }
      }
    }
  }
  fstamp(a, 5);
  if (a.atomic_out) {  // ---- partials added into out (zeroed by the O-proj GEMV); order varies run to run
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
      const int ch = tid + NT * j;
      if (ch < CH && nact > 0) {
#pragma unroll
        for (int b = 0; b < B; ++b) {
          float4* dst = reinterpret_cast<float4*>(a.out + (size_t)b * d + ch * 8);
          atomicAdd(dst, make_float4(y[b][j * 8 + 0], y[b][j * 8 + 1], y[b][j * 8 + 2], y[b][j * 8 + 3]));
          atomicAdd(dst + 1, make_float4(y[b][j * 8 + 4], y[b][j * 8 + 5], y[b][j * 8 + 6], y[b][j * 8 + 7]));
        }
      }
    }
    if (a.n_active_out && tid < B) {
      int cnt = 0;
      for (int c = 0; c < nch; ++c) cnt += __popc(act_s[c][tid]);
      if (cnt) atomicAdd(a.n_active_out + (size_t)tid * a.n_active_stride, cnt);
    }
    if (a.par.world) par::push_last(a.par, a.out, B * d, nullptr, 0, nullptr);  // fused all-reduce (TP > 1)
    fstamp(a, 6);
    return;
  }
  // ---- per-CTA partials -> grid barrier -> deterministic column reduction
#pragma unroll
  for (int j = 0; j < CPT; ++j) {
    const int ch = tid + NT * j;
    if (ch < CH) {
#pragma unroll
      for (int b = 0; b < B; ++b) {
        float4* dst = reinterpret_cast<float4*>(a.part + ((size_t)cta * B + b) * d + ch * 8);
        dst[0] = make_float4(y[b][j * 8 + 0], y[b][j * 8 + 1], y[b][j * 8 + 2], y[b][j * 8 + 3]);
        dst[1] = make_float4(y[b][j * 8 + 4], y[b][j * 8 + 5], y[b][j * 8 + 6], y[b][j * 8 + 7]);
      }
    }
  }
  if (tid < B) {
    int cnt = 0;
    for (int c = 0; c < nch; ++c) cnt += __popc(act_s[c][tid]);
    a.part_cnt[cta * B + tid] = cnt;
  }
  grid_barrier(a.barrier, G);
  const int units = B * d / 4;  // float4 columns
  const int u0 = (int)((long long)units * cta / G), u1 = (int)((long long)units * (cta + 1) / G);
  for (int u = u0 + warp; u < u1; u += kFfnWarps) {
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
    atomicAdd(a.n_active_out + (size_t)tid * a.n_active_stride, tot);
  }
  if (a.par.world) par::push_last(a.par, a.out, B * d, nullptr, 0, nullptr);  // fused all-reduce (TP > 1)
}

}  // namespace

// ===================================================================== host-side launchers
namespace launch {

template <int B, int CPL>
static cudaError_t gemv_bc(const GemvArgs& a, int grid, cudaStream_t st) {
  auto kern = gemv_kernel<B, CPL>;
  const size_t smem = (size_t)B * a.K * 4;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(g_decode_pdl, kern, dim3(grid), dim3(kGemvWarps * 32), smem, st, a);
}

template <int B>
static cudaError_t gemv_b(const GemvArgs& a, int grid, cudaStream_t st) {
  const int cpl = (a.K / 8 + 31) / 32;
  if (cpl <= 1) return gemv_bc<B, 1>(a, grid, st);
  if (cpl <= 2) return gemv_bc<B, 2>(a, grid, st);
  if (cpl <= 4) return gemv_bc<B, 4>(a, grid, st);
  if (cpl <= 8) return gemv_bc<B, 8>(a, grid, st);
  if (cpl <= 16) return gemv_bc<B, 16>(a, grid, st);
  if (cpl <= 32) return gemv_bc<B, 32>(a, grid, st);
  return cudaErrorInvalidValue;
}

cudaError_t par_reduce(const PeerAr& p, float* dst, int n, int nk, int32_t* token_out, cudaStream_t st) {
  par_reduce_kernel<<<1, 256, 0, st>>>(p, dst, n, nk, token_out);
  return cudaGetLastError();
}

cudaError_t argmax_finalize(unsigned long long* amax, int B, int32_t* token_out, cudaStream_t st) {
  argmax_finalize_kernel<<<1, 32, 0, st>>>(amax, B, token_out);
  return cudaGetLastError();
}

int gemv_grid(int rows, int num_sms) {
  const int g = 2 * num_sms;
  return rows < g ? rows : g;
}

cudaError_t gemv(const GemvArgs& a, int B, int grid, cudaStream_t st) {
  if (a.K % 8) return cudaErrorInvalidValue;
  switch (B) {
    case 1: return gemv_b<1>(a, grid, st);
    case 2: return gemv_b<2>(a, grid, st);
    case 4: return gemv_b<4>(a, grid, st);
    case 8: return gemv_b<8>(a, grid, st);
    default: return cudaErrorInvalidValue;
  }
}

int ffn_grid(int F, int num_sms) {
  int g = (F + 7) / 8;
  if (g > num_sms) g = num_sms;
  if ((F + g - 1) / g > kFfnMaxN) return -1;
  return g;
}

template <int B, int CPL, int CPT, int NW>
static cudaError_t ffn_bc(const FfnArgs& a, int grid, cudaStream_t st) {
  auto kern = ffn_kernel<B, CPL, CPT, NW>;
  const size_t smem = (size_t)B * a.d * 4;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NW * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // co-residency for the grid barrier (deterministic mode)
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (a.atomic_out) {  // no grid barrier: PDL instead of the cooperative attribute (decode chain)
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.numAttrs = g_decode_pdl ? 1 : 0;
  }
  return cudaLaunchKernelEx(&cfg, kern, a);
}

template <int B>
static cudaError_t ffn_b(const FfnArgs& a, int grid, cudaStream_t st) {
  const int CH = a.d / 8;
  const int cpl = (CH + 31) / 32;
  if (a.atomic_out) {  // 8 warps: CPT = d / 2048 column chunks per thread
    if (cpl <= 1) return ffn_bc<B, 1, 1, 8>(a, grid, st);
    if (cpl <= 2) return ffn_bc<B, 2, 1, 8>(a, grid, st);
    if (cpl <= 4) return ffn_bc<B, 4, 1, 8>(a, grid, st);
    if (cpl <= 8) return ffn_bc<B, 8, 1, 8>(a, grid, st);
    if (cpl <= 16) return ffn_bc<B, 16, 2, 8>(a, grid, st);  // d = 4096
    if (cpl <= 32) return ffn_bc<B, 32, 4, 8>(a, grid, st);  // d = 8192
    return cudaErrorInvalidValue;
  }
  const int cpt = (CH + 16 * 32 - 1) / (16 * 32);
  if (cpl <= 1) return ffn_bc<B, 1, 1, 16>(a, grid, st);
  if (cpl <= 2) return ffn_bc<B, 2, 1, 16>(a, grid, st);
  if (cpl <= 4) return ffn_bc<B, 4, 1, 16>(a, grid, st);
  if (cpl <= 8) return ffn_bc<B, 8, 1, 16>(a, grid, st);
  if (cpl <= 16) return ffn_bc<B, 16, 1, 16>(a, grid, st);  // d = 4096
  if (cpl <= 32 && cpt <= 2) return ffn_bc<B, 32, 2, 16>(a, grid, st);  // d = 8192
  return cudaErrorInvalidValue;
}

cudaError_t ffn(const FfnArgs& a, int B, int grid, cudaStream_t st) {
  if (a.d % 8) return cudaErrorInvalidValue;
  switch (B) {
    case 1: return ffn_b<1>(a, grid, st);
    case 2: return ffn_b<2>(a, grid, st);
    case 4: return ffn_b<4>(a, grid, st);
    case 8: return ffn_b<8>(a, grid, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace launch
}  // namespace sirius
