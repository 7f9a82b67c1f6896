// peer_ar.cuh — the fused peer all-reduce of the tensor-parallel decode step (SURVEY.md §8(e) phase 2;
// the all-reduces of S3 / S6 / S7 in SURVEY.md §8(a)): device side of the protocol documented at
// PeerAr (decode_kernels.cuh).  The producer half runs in the epilogue of the kernel that computes the
// rank partial (O-proj GEMV, CATS FFN, LM-head argmax), the consumer half in the activation prologue of
// the kernel that needs the sum (FFN, next layer's QKV GEMV, LM head) — no separate collective launch:
// the push goes out over NVLink (peer stores through CUDA-IPC mappings) the moment the partial is
// complete, and the consumer's wait overlaps its first weight rows already in flight.
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

// Consumer: every thread of the CTA calls it.  Waits until every source rank's push of this rank's
// current sync point s (= *seq, incremented by the producer kernel that ran just before in stream
// order) has landed, then returns this rank's slot array of parity s & 1 ([world][slot_n], local
// memory).  A rank that does not arrive within 10 s sets kErrTimeout and the wait gives up (the
// results are then garbage, the next ABI call reports the error).
SIRIUS_DEV const float* wait(const PeerAr& p) {
  const unsigned long long s = __ldcg(p.seq);
  const int par = (int)(s & 1ull);
  if (threadIdx.x < (unsigned)p.world) {
    const unsigned long long* f =
        reinterpret_cast<const unsigned long long*>(p.self + off_flags(p)) + (size_t)par * p.world + threadIdx.x;
    if (ld_acquire_sys(f) < s) {
      const unsigned long long t0 = globaltimer();
      int n = 0;
      while (ld_acquire_sys(f) < s) {
        if (++n == 4096) {
          n = 0;
          if (globaltimer() - t0 > 10000000000ull) {
            atomicOr(p.err, kErrTimeout);
            break;
          }
        }
      }
    }
  }
  __syncthreads();
  return reinterpret_cast<const float*>(p.self) + (size_t)par * p.world * p.slot_n;
}

// this rank's received key slots of parity par ([world][key_n])
SIRIUS_DEV const unsigned long long* keys(const PeerAr& p, int par) {
  return reinterpret_cast<const unsigned long long*>(p.self + off_keys(p)) + (size_t)par * p.world * p.key_n;
}

// Producer: every thread of every CTA calls it once the CTA's contribution to src (n floats, n % 4 ==
// 0, written by plain stores or atomics) / to the packed keys (nk words, atomicMax) is complete.  The
// CTA that arrives last pushes src and keys to every rank (the keys are reset to 0 for the next step),
// then publishes the new sequence number.
SIRIUS_DEV void push_last(const PeerAr& p, const float* src, int n, unsigned long long* keys_io, int nk) {
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
  for (int i = threadIdx.x; i < n / 4; i += blockDim.x) {
    const float4 v = __ldcg(reinterpret_cast<const float4*>(src) + i);
#pragma unroll
    for (int q = 0; q < kMaxWorld; ++q)
      if (q < W) {
        const int si = p.loopback ? q : p.rank;
        reinterpret_cast<float4*>(reinterpret_cast<float*>(pb[q]) + slot0 + (size_t)si * p.slot_n)[i] = v;
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
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x < (unsigned)W) {
    const int q = threadIdx.x, si = p.loopback ? q : p.rank;
    st_release_sys(reinterpret_cast<unsigned long long*>(pb[q] + off_flags(p)) + (size_t)par * W + si, s);
  }
  if (threadIdx.x == 0) *p.seq = s;
}

}  // namespace par
}  // namespace sirius
