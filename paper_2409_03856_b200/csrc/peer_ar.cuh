// peer_ar.cuh — the fused peer all-reduce of the tensor-parallel decode step (SURVEY.md §8(e) phase 2;
// the all-reduces of S3 / S6 / S7 in SURVEY.md §8(a)): device side of the protocol documented at
// PeerAr (decode_kernels.cuh).  It runs in the tail of the kernel that computes the rank partial
// (O-proj GEMV, CATS FFN, LM-head argmax): the CTA that completes the partial pushes it over NVLink
// (peer stores through CUDA-IPC mappings), waits for the peers' pushes and reduces them in place — no
// collective launch, and the next kernel's prologue reads the all-reduced delta as at TP 1.
#pragma once
#include "common.cuh"
#include "decode_kernels.cuh"

namespace sirius {
namespace par {

constexpr int kMaxWorld = 8;
constexpr int kErrTimeout = 8;  // device error word bit: a peer never arrived (runtime: SIRIUS_ERR_NCCL)

SIRIUS_DEV size_t off_keys(const PeerAr& p) { return (size_t)2 * p.world * p.slot_n * sizeof(float); }
SIRIUS_DEV size_t off_flags(const PeerAr& p) { return off_keys(p) + (size_t)2 * p.world * p.key_n * 8; }

SIRIUS_DEV void st_release_sys(unsigned long long* a, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
SIRIUS_DEV unsigned long long ld_acquire_sys(const unsigned long long* a) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
  return v;
}
SIRIUS_DEV unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// threads < world acquire-wait for flags (par, 0..world-1) >= s on this rank's buffer; CTA barrier.
// A rank that does not arrive within timeout_ns (10 s) sets kErrTimeout and the wait gives up (the
// results are then garbage, the next ABI call reports SIRIUS_ERR_NCCL); once the bit is set every
// later wait gives up at once, so a dead peer costs one timeout, not one per sync point.
SIRIUS_DEV void wait_flags(const PeerAr& p, unsigned long long s) {
  const int par = (int)(s & 1ull);
  if (threadIdx.x < (unsigned)p.world) {
    const unsigned long long* f =
        reinterpret_cast<const unsigned long long*>(p.self + off_flags(p)) + (size_t)par * p.world + threadIdx.x;
    // acquire polling (measured faster than relaxed polling + a fence); the CTA barrier orders the
    // other threads' slot reads after it
    if (ld_acquire_sys(f) < s && !(*(volatile const int*)p.err & kErrTimeout)) {
      const unsigned long long t0 = globaltimer();
      int n = 0;
      while (ld_acquire_sys(f) < s) {
        if (++n == 4096) {
          n = 0;
          if (globaltimer() - t0 > p.timeout_ns || (*(volatile const int*)p.err & kErrTimeout)) {
            atomicOr(p.err, kErrTimeout);
            break;
          }
        }
      }
    }
  }
  __syncthreads();
}

// every thread of the CTA: dst[0, n) = scale * ((slot_0 + slot_1) + ... + slot_{world-1}) of parity par
// (rank order, as the emulated in-order sum), and for the keys: the max over the ranks -> token_out
// (argmax_key_index) when token_out != NULL, else -> keys_out
SIRIUS_DEV void reduce(const PeerAr& p, int par, float* dst, int n, int nk, unsigned long long* keys_out,
                       int32_t* token_out) {
  const int W = p.world;
  const float* slots = reinterpret_cast<const float*>(p.self) + (size_t)par * W * p.slot_n;
  constexpr int GU = 2;  // float4 groups per thread per round: GU * kMaxWorld loads in flight
  for (int i0 = threadIdx.x; i0 < n / 4; i0 += GU * blockDim.x) {
    float4 v[GU][kMaxWorld];
#pragma unroll
    for (int u = 0; u < GU; ++u)
#pragma unroll
      for (int r = 0; r < kMaxWorld; ++r) {
        const int i = i0 + u * blockDim.x;
        if (r < W && i < n / 4) v[u][r] = __ldcg(reinterpret_cast<const float4*>(slots + (size_t)r * p.slot_n) + i);
      }
#pragma unroll
    for (int u = 0; u < GU; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i >= n / 4) continue;
      float4 a = v[u][0];
#pragma unroll
      for (int r = 1; r < kMaxWorld; ++r)
        if (r < W) {
          a.x += v[u][r].x; a.y += v[u][r].y; a.z += v[u][r].z; a.w += v[u][r].w;
        }
      a.x *= p.scale; a.y *= p.scale; a.z *= p.scale; a.w *= p.scale;
      reinterpret_cast<float4*>(dst)[i] = a;
    }
  }
  const unsigned long long* ks =
      reinterpret_cast<const unsigned long long*>(p.self + off_keys(p)) + (size_t)par * W * p.key_n;
  for (int b = threadIdx.x; b < nk; b += blockDim.x) {
    unsigned long long m = 0ull;
    for (int r = 0; r < W; ++r) m = ks[(size_t)r * p.key_n + b] > m ? ks[(size_t)r * p.key_n + b] : m;
    if (token_out) token_out[b] = (int32_t)argmax_key_index(m);
    else keys_out[b] = m;
  }
}

// Producer: every thread of every CTA calls it once the CTA's contribution to src (n floats, n % 4 ==
// 0, written by plain stores or atomics) / to the packed keys (nk words, atomicMax) is complete.  The
// CTA that arrives last pushes src and keys to every rank (the keys are reset to 0 for the next step),
// publishes the new sequence number and, fused, waits for every rank's push and writes the reduced
// sum over src (keys: the global argmax -> token_out).
SIRIUS_DEV void push_last(const PeerAr& p, float* src, int n, unsigned long long* keys_io, int nk, int32_t* token_out) {
  __shared__ unsigned last_s;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned old = atomicAdd(p.done, 1u);
    const unsigned last = old == gridDim.x - 1 ? 1u : 0u;
    if (last) {
      atomicExch(p.done, 0u);
      __threadfence();
    }
    last_s = last;
  }
  __syncthreads();
  if (!last_s) return;
  const int W = p.world;
  char* pb[kMaxWorld];
#pragma unroll
  for (int q = 0; q < kMaxWorld; ++q) pb[q] = q < W ? p.peers[q] : nullptr;
  const unsigned long long s = __ldcg(p.seq) + 1ull;
  const int par = (int)(s & 1ull);
  const size_t slot0 = (size_t)par * W * p.slot_n;
  constexpr int GU = 8;  // float4 groups per thread loaded before any store
  for (int i0 = threadIdx.x; i0 < n / 4; i0 += GU * blockDim.x) {
    float4 v[GU];
#pragma unroll
    for (int u = 0; u < GU; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i < n / 4) v[u] = __ldcg(reinterpret_cast<const float4*>(src) + i);
    }
#pragma unroll
    for (int q = 0; q < kMaxWorld; ++q)
      if (q < W) {
        float4* dq = reinterpret_cast<float4*>(reinterpret_cast<float*>(pb[q]) + slot0 +
                                               (size_t)(p.loopback ? q : p.rank) * p.slot_n);
#pragma unroll
        for (int u = 0; u < GU; ++u) {
          const int i = i0 + u * blockDim.x;
          if (i < n / 4) dq[i] = v[u];
        }
      }
  }
  for (int i = threadIdx.x; i < nk; i += blockDim.x) {
    const unsigned long long k = atomicExch(keys_io + i, 0ull);  // read + reset for the next step
#pragma unroll
    for (int q = 0; q < kMaxWorld; ++q)
      if (q < W) {
        const int si = p.loopback ? q : p.rank;
        reinterpret_cast<unsigned long long*>(pb[q] + off_keys(p))[((size_t)par * W + si) * p.key_n + i] = k;
      }
  }
  // the CTA barrier orders every thread's stores before the flag lanes' sys-scope release stores (PTX
  // memory model: bar.sync is morally strong, a release is cumulative over what its thread observed);
  // lanes 0..W-1 of warp 0 release in one instruction (measured: faster than one fence + W relaxed
  // stores by one thread, tools/tp_proxy.py A/B on one box)
  __syncthreads();
  if (threadIdx.x < (unsigned)W)
    st_release_sys(reinterpret_cast<unsigned long long*>(pb[threadIdx.x] + off_flags(p)) + (size_t)par * W +
                       (p.loopback ? threadIdx.x : p.rank), s);
  if (threadIdx.x == 0) *p.seq = s;
  if (!p.fused) return;
  wait_flags(p, s);
  reduce(p, par, src, n, nk, keys_io, token_out);
}

}  // namespace par
}  // namespace sirius
