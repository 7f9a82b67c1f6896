// common.cuh — device helpers for the sm_100a Sirius kernels (PTX wrappers, reductions,
// bf16 packing, grid barrier).  Product code: no oracle code is included or shared.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#define SIRIUS_DEV __device__ __forceinline__

namespace sirius {

constexpr int kWarp = 32;

SIRIUS_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// ------------------------------------------------------------------ mbarrier
SIRIUS_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
SIRIUS_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
SIRIUS_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

SIRIUS_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
SIRIUS_DEV void mbar_arrive(uint64_t* bar, uint32_t count = 1) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
SIRIUS_DEV bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
SIRIUS_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// ------------------------------------------------------------------ bulk async copies (TMA engine, 1-D)
// L2 eviction policy for weight streams: every weight byte is read once per step.
SIRIUS_DEV uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
SIRIUS_DEV uint64_t policy_evict_unchanged() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(p));
  return p;
}
SIRIUS_DEV uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// global -> shared, `bytes` multiple of 16, both addresses 16-byte aligned; completes tx on `bar`.
SIRIUS_DEV void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// ------------------------------------------------------------------ PDL (programmatic dependent launch)
// Kernels of the verify / prefill chain call pdl_trigger() then pdl_wait() before touching anything a
// predecessor writes (both are no-ops when a kernel is launched without the PDL attribute).
SIRIUS_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
SIRIUS_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

namespace launch {
extern bool g_chain_pdl;   // verify / prefill chain launched with PDL (runtime.cu; SIRIUS_VERIFY_PDL)
extern bool g_decode_pdl;  // per-stage decode chain (QKV / O / head GEMV, attention, CATS FFN) with PDL
                           // (runtime.cu; SIRIUS_DECODE_PDL): each kernel streams its first weight rows
                           // before griddepcontrol.wait and triggers its dependent right after it
// <<<grid, block, smem, st>>> with the programmatic-stream-serialization attribute when g_chain_pdl
template <class... KArgs, class... Args>
inline cudaError_t launch_chain(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_chain_pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<Args&&>(args)...);
}
// the same with an explicit PDL switch
template <class... KArgs, class... Args>
inline cudaError_t launch_pdl(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<Args&&>(args)...);
}
}  // namespace launch

// ------------------------------------------------------------------ loads
SIRIUS_DEV uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
// streamed weights read once per step: L2 lines marked evict-first on use
SIRIUS_DEV uint4 ld_nc_v4_ef(const void* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
SIRIUS_DEV unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// ------------------------------------------------------------------ bf16
SIRIUS_DEV float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }
SIRIUS_DEV float bf16_hi(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }
SIRIUS_DEV uint16_t f2bf_bits(float f) { return __bfloat16_as_ushort(__float2bfloat16_rn(f)); }
SIRIUS_DEV float round_bf16(float f) { return __bfloat162float(__float2bfloat16_rn(f)); }
SIRIUS_DEV uint32_t pack_bf16(float lo, float hi) { return (uint32_t)f2bf_bits(lo) | ((uint32_t)f2bf_bits(hi) << 16); }
// fp32 value as three bf16 terms x = t0 + t1 + t2 (exact for normal x: each residual is exact in fp32
// and the last one has <= 8 significant bits) — the tensor-core B operand of the verify / prefill
// GEMMs ("x3" operand planes, D15a).  t[0] = bf16(x), t[1] = bf16(x - t0), t[2] = bf16(x - t0 - t1).
SIRIUS_DEV void split3(float x, uint16_t* t) {
  t[0] = f2bf_bits(x);
  const float r1 = x - __uint_as_float((uint32_t)t[0] << 16);
  t[1] = f2bf_bits(r1);
  t[2] = f2bf_bits(r1 - __uint_as_float((uint32_t)t[1] << 16));
}
// store x at element off of the three planes (plane stride in elements)
SIRIUS_DEV void store_split3(uint16_t* x3, size_t plane, size_t off, float x) {
  uint16_t t[3];
  split3(x, t);
  x3[off] = t[0];
  x3[plane + off] = t[1];
  x3[2 * plane + off] = t[2];
}

// dot of 8 bf16 (packed in a uint4) with 8 floats
SIRIUS_DEV float dot8(const uint4 w, const float* x) {
  float s = 0.f;
  s = fmaf(bf16_lo(w.x), x[0], s);
  s = fmaf(bf16_hi(w.x), x[1], s);
  s = fmaf(bf16_lo(w.y), x[2], s);
  s = fmaf(bf16_hi(w.y), x[3], s);
  s = fmaf(bf16_lo(w.z), x[4], s);
  s = fmaf(bf16_hi(w.z), x[5], s);
  s = fmaf(bf16_lo(w.w), x[6], s);
  s = fmaf(bf16_hi(w.w), x[7], s);
  return s;
}
// dot of 8 bf16 weights with 8 bf16 activations
SIRIUS_DEV float dot8bf(const uint4 w, const uint4 h, float s) {
  s = fmaf(bf16_lo(w.x), bf16_lo(h.x), s);
  s = fmaf(bf16_hi(w.x), bf16_hi(h.x), s);
  s = fmaf(bf16_lo(w.y), bf16_lo(h.y), s);
  s = fmaf(bf16_hi(w.y), bf16_hi(h.y), s);
  s = fmaf(bf16_lo(w.z), bf16_lo(h.z), s);
  s = fmaf(bf16_hi(w.z), bf16_hi(h.z), s);
  s = fmaf(bf16_lo(w.w), bf16_lo(h.w), s);
  s = fmaf(bf16_hi(w.w), bf16_hi(h.w), s);
  return s;
}

// ------------------------------------------------------------------ warp / block reductions (fixed order)
SIRIUS_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
SIRIUS_DEV float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// order-preserving float -> uint32 (monotone), for packed argmax keys
SIRIUS_DEV uint32_t float_ordered(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
SIRIUS_DEV float ordered_float(uint32_t u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u);
}
// argmax key: larger value wins, then LOWER index wins (reading D13)
SIRIUS_DEV unsigned long long argmax_key(float v, uint32_t idx) {
  return ((unsigned long long)float_ordered(v) << 32) | (unsigned long long)(0xFFFFFFFFu - idx);
}
SIRIUS_DEV uint32_t argmax_key_index(unsigned long long k) { return 0xFFFFFFFFu - (uint32_t)(k & 0xFFFFFFFFull); }
SIRIUS_DEV unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w > v ? w : v;
  }
  return v;
}

// ------------------------------------------------------------------ grid-wide barrier
// All CTAs of the launch must be co-resident (cooperative launch).  Monotone 64-bit counter:
// generation g completes when the counter reaches (g+1)*nblocks; never reset, never wraps.
SIRIUS_DEV void grid_barrier(unsigned long long* counter, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned long long old = atomicAdd(counter, 1ull);
    unsigned long long target = (old / nblocks + 1) * nblocks;
    while (ld_acquire_u64(counter) < target) __nanosleep(20);
    __threadfence();
  }
  __syncthreads();
}

// Same contract as grid_barrier, one round trip cheaper: the arrival is a single release atomic
// (cumulative over the CTA's writes ordered before it by bar.sync), the wait an acquire spin.
SIRIUS_DEV void grid_sync(unsigned long long* counter, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long old, v;
    asm volatile("atom.add.release.gpu.u64 %0, [%1], 1;" : "=l"(old) : "l"(counter) : "memory");
    const unsigned long long target = (old / nblocks + 1) * nblocks;
    do {
      asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(v) : "l"(counter) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// Barrier among the n co-resident CTAs that share bar[0] (arrival count) / bar[1] (generation), a
// subset of a cooperative grid.  Self-resetting, so the same counter may be used by later launches
// with a different n (each counter is used at most once per launch).
SIRIUS_DEV void group_barrier(unsigned* bar, unsigned n) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vgen = bar + 1;
    const unsigned gen = *vgen;  // read the generation BEFORE arriving
    __threadfence();
    if (atomicAdd(bar, 1u) == n - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*vgen == gen) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

// "last CTA to arrive" election for split reductions; returns true in exactly one CTA per group
// of `n` arrivals.  The last arrival resets the counter to 0 for the next launch.
SIRIUS_DEV bool arrive_last(unsigned* counter, unsigned n) {
  __shared__ unsigned s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned old = atomicAdd(counter, 1u);
    bool last = old == n - 1;
    if (last) {
      atomicExch(counter, 0u);
      __threadfence();
    }
    s_last = last ? 1u : 0u;
  }
  __syncthreads();
  return s_last != 0;
}

}  // namespace sirius
