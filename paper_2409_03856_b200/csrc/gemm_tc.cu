// gemm_tc.cu — tcgen05 tensor-core GEMM for the gamma-row full-model verification forward
// ("memory-bound while rows <= 64", PAPER.md:70 / Table 10; the verify pass is
// the one place on the path that really is a dense contraction).
//
//   C[m, n] = sum_k X[m, k] * W[n, k]          X: activations [Mp, K] bf16, W: weights [N, K] bf16
//
// Swap-AB: the weights are the MMA "A" operand (M = 128 weight rows per tile), the Mp <= 256 token
// rows are the MMA "B" operand (N = Mp), so one tcgen05.mma.kind::f16 128 x Mp x 16 instruction
// covers every token of the kernel; accumulators (fp32) live in TMEM.  Operands arrive via 2-D TMA
// (cp.async.bulk.tensor, SWIZZLE_128B) into a multi-stage mbarrier ring.  Work is split stream-K
// style over the 148 SMs: CTA c owns the contiguous k-block range [W c / G, W (c+1) / G) of the
// (tile, k-block) space, so every SM streams the same number of weight bytes; tiles cut by a CTA
// boundary are reduced deterministically (fixed CTA order) by the last-arriving CTA.
//
// Roles (128 threads): warp 0 lane 0 = TMA producer, warp 1 lane 0 = MMA issuer, warp 2 = TMEM
// allocator; all four warps run the epilogue (TMEM lane = weight row = threadIdx.x).
// Epilogues: fp32 store, or SwiGLU m = SiLU(g) * u from two accumulators (gate, up), written as three
// bf16 terms.  Activations enter as three bf16 terms of fp32 values (split3: x = t0 + t1 + t2 exactly):
// three MMAs per k-step into one accumulator, free while the pass is HBM-bound (D15a).
#include <cuda.h>

#include "common.cuh"
#include "gemm_tc.cuh"
#include "peer_ar.cuh"

namespace sirius {

SIRIUS_DEV void tma_load_2d(void* smem_dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], "
      "[%4], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
SIRIUS_DEV void tma_load_3d(void* smem_dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar,
                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, "
      "%4}], [%5], %6;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
SIRIUS_DEV void tma_load_4d(void* smem_dst, const CUtensorMap* map, int c0, int c1, int c2, int c3, uint64_t* bar,
                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, "
      "%4, %5}], [%6], %7;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
SIRIUS_DEV void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// K-major, SWIZZLE_128B shared-memory matrix descriptor (sm_100 "version 1"):
// start>>4 [0,14), LBO>>4 [16,30) (unused for SW128 K-major), SBO>>4 [32,46) = 1024 B between
// 8-row core groups, version [46,48) = 1, layout [61,64) = 2 (SWIZZLE_128B).
SIRIUS_DEV uint64_t sw128_desc(const void* smem) {
  const uint32_t a = smem_u32(smem);
  return (uint64_t)((a & 0x3FFFFu) >> 4) | ((uint64_t)(1024u >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

SIRIUS_DEV void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
SIRIUS_DEV void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
SIRIUS_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
SIRIUS_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 32 lanes x 16 columns of fp32 from TMEM (this warp's lane quarter) -> 16 registers per thread.
SIRIUS_DEV void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// last CTA owning work item x (CTA c owns [floor(W c / G), floor(W (c+1) / G)))
SIRIUS_DEV int owner_of(long long x, long long W, int G) { return (int)(((x + 1) * G + W - 1) / W) - 1; }

// fused all-reduce destinations of this CTA's epilogue (read once, after the PDL wait): this rank's
// slot of parity (s + 1) on every rank
struct ParDst {
  float* slot[8];
};

template <bool DUAL>
SIRIUS_DEV void epi_store(const GemmArgs& g, int j, int n, float v0, float v1, const ParDst* pd = nullptr) {
  if (j >= g.M || n >= g.N) return;
  if (DUAL) {
    const float av = v0 / (1.0f + expf(-v0));  // a = SiLU(gate)
    const bool on = !g.thr || fabsf(av) >= *g.thr;
    const float m = on ? av * v1 : 0.f;        // a * up, CATS-masked (inactive pairs contribute exact 0)
    if (g.gate_out) g.gate_out[(size_t)j * g.gate_stride + n] = av;
    if (g.n_active && on) atomicAdd(g.n_active + (size_t)j * g.n_active_stride, 1);
    store_split3(reinterpret_cast<uint16_t*>(g.out), g.out_plane, (size_t)j * g.ldc + n, m);
  } else {
    reinterpret_cast<float*>(g.out)[(size_t)j * g.ldc + n] = v0;
    if (pd) {  // fused all-reduce: this rank's element into its slot on every rank
      const size_t off = (size_t)j * g.ldc + n;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q < g.par.world) pd->slot[q][off] = v0;
    }
  }
}

SIRIUS_DEV void gstamp(const GemmArgs& g, int slot) {
  if (!g.trace) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  g.trace[(size_t)slot * 1024 + blockIdx.x] = t;  // [8][1024]
}

// Epilogue-only barrier (warps 0-3) and "last of n arrivals" election among them.
SIRIUS_DEV void epi_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
SIRIUS_DEV bool epi_arrive_last(unsigned* counter, unsigned n, unsigned* flag_s) {
  epi_sync();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned old = atomicAdd(counter, 1u);
    const bool last = old == n - 1;
    if (last) {
      atomicExch(counter, 0u);
      __threadfence();
    }
    *flag_s = last ? 1u : 0u;
  }
  epi_sync();
  return *flag_s != 0;
}

// Warp-specialised (192 threads): warps 0-3 epilogue (TMEM lane = weight row = threadIdx.x), warp 4
// lane 0 TMA producer, warp 5 lane 0 MMA issuer (+ TMEM allocation).  The producer streams the CTA's
// whole stream-K range without stopping at tile (segment) boundaries, and the accumulator is double
// buffered in TMEM when 2 NACC MP <= 512 columns, so a segment's epilogue / fix-up overlaps the next
// segment's loads and MMAs (r01 trace: the second segment of a CTA used to wait for the first's
// epilogue and refill the pipeline, up to 17 us per GEMM).
template <bool DUAL, int KBOX>
__global__ void __launch_bounds__(192, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmA1,
                   const __grid_constant__ CUtensorMap tmB, GemmArgs g, int MP, int stages) {
  // KBOX: 64-wide K boxes per pipeline stage (one work unit = 64 KBOX of K): each weight row is read
  // 128 KBOX contiguous bytes at a time
  constexpr int NACC = DUAL ? 2 : 1;
  constexpr uint32_t BOX_BYTES = 128 * 64 * 2;      // one 128 x 64 bf16 weight box
  constexpr uint32_t A_BYTES = BOX_BYTES * KBOX;    // one operand's weight tiles of a stage
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int G = gridDim.x, c = blockIdx.x;
  const long long W = (long long)g.n_tiles * g.kb;
  const long long w0 = W * c / G, w1 = W * (c + 1) / G;
  if (w0 == w1) return;

  if (tid == 0) gstamp(g, 0);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const uint32_t b_bytes = (uint32_t)MP * 128 * KBOX;  // one activation term's boxes of a stage
  const int NB = g.nterms;
  const uint32_t stage_bytes = ((NACC * A_BYTES + NB * b_bytes) + 1023) & ~1023u;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * stage_bytes);
  uint64_t* empty = full + stages;
  uint64_t* acc_full = empty + stages;   // [2]
  uint64_t* acc_empty = acc_full + 2;    // [2]
  uint32_t* tmem_ptr_s = reinterpret_cast<uint32_t*>(acc_empty + 2);
  unsigned* flag_s = tmem_ptr_s + 1;
  // Activation terms side by side along N (one 128 x NB*MP x 16 MMA per k-step and operand instead of
  // NB MMAs of N = MP: the verify GEMMs at MP = 16 were bound by the MMA issue rate, not by HBM);
  // the epilogue sums the NB accumulator column groups.  NB*MP > 256: one MMA per term, one group.
  const bool cat = NB * MP <= 256;
  const int ACCW = cat ? NB * MP : MP;  // accumulator columns per operand
  const int NBUF = 2 * NACC * ACCW <= 512 ? 2 : 1;
  uint32_t ncols = 32;
  while (ncols < (uint32_t)(NBUF * NACC * ACCW)) ncols <<= 1;

  if (tid == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 4);  // one arrival per epilogue warp
    }
    fence_mbar_init();
    prefetch_tmap(&tmA0);
    if (DUAL) prefetch_tmap(&tmA1);
    prefetch_tmap(&tmB);
  }
  if (warp == 5) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_ptr_s)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr_s;
  // instruction descriptor, kind::f16: D fp32 [4,6)=1, A bf16 [7,10)=1, B bf16 [10,13)=1,
  // both K-major, N>>3 at [17,23), M>>4 at [24,29)
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)((cat ? NB * MP : MP) >> 3) << 17) |
                         ((128u >> 4) << 24);
  const uint32_t tx_bytes = NACC * A_BYTES + NB * b_bytes;
  const long long nq = w1 - w0;  // the CTA's k-iterations, over all its segments
  // weight tiles of a stage: [x][128 rows][128 B] — one 3-D op (box 64 x 128 rows x KBOX) per operand,
  // or KBOX 2-D boxes.  TMA ops have a fixed per-op cost (tools/bw_probe.cu: 1-D bulk copies of 4 / 8 /
  // 16 KB stream at 3.0 / 6.0 / 7.1 TB/s whatever the ring depth), so a stage is as few ops as possible.
  auto load_a = [&](uint8_t* st, int t, int kc, uint64_t* bar, uint64_t pol) {
    if (g.coarse) {
      tma_load_3d(st, &tmA0, 0, t * 128, kc / 64, bar, pol);
      if (DUAL) tma_load_3d(st + A_BYTES, &tmA1, 0, t * 128, kc / 64, bar, pol);
    } else {
#pragma unroll
      for (int x = 0; x < KBOX; ++x) {
        tma_load_2d(st + x * BOX_BYTES, &tmA0, kc + 64 * x, t * 128, bar, pol);
        if (DUAL) tma_load_2d(st + A_BYTES + x * BOX_BYTES, &tmA1, kc + 64 * x, t * 128, bar, pol);
      }
    }
  };
  pdl_trigger();

  if (warp == 4) {
    if (lane == 0) {  // ---------------- TMA producer
      const uint64_t pol_w = policy_evict_first(), pol_x = policy_evict_last();
      // PDL: weight (A) tiles of the first stages before the dependency wait, activations after it
      const int npre = (int)min((long long)stages, nq);
      for (int i = 0; i < npre; ++i) {
        const long long w = w0 + i;
        uint8_t* st = smem + (size_t)i * stage_bytes;
        mbar_arrive_expect_tx(&full[i], tx_bytes);
        const int t = (int)(w / g.kb), kc = (int)(w % g.kb) * 64 * KBOX;
        load_a(st, t, kc, &full[i], pol_w);
      }
      gstamp(g, 1);
      pdl_wait();
      gstamp(g, 2);
      for (long long q = 0; q < nq; ++q) {
        const long long w = w0 + q;
        const int s = (int)(q % stages);
        const int t = (int)(w / g.kb), kc = (int)(w % g.kb) * 64 * KBOX;
        uint8_t* st = smem + (size_t)s * stage_bytes;
        if (q >= npre) {
          mbar_wait(&empty[s], ((uint32_t)(q / stages) & 1u) ^ 1u);
          mbar_arrive_expect_tx(&full[s], tx_bytes);
          load_a(st, t, kc, &full[s], pol_w);
        }
        // B boxes of a stage: [x][term][MP rows][128 B]
        if (g.coarse) {  // all terms, rows and K boxes of the stage in one 4-D op
          tma_load_4d(st + NACC * A_BYTES, &tmB, 0, g.row0, 0, kc / 64, &full[s], pol_x);
        } else {
#pragma unroll
          for (int x = 0; x < KBOX; ++x) {
            uint8_t* bx = st + NACC * A_BYTES + (size_t)x * NB * MP * 128;
            for (int p = 0; p < NB; ++p)
              for (int r = 0; r < MP / 16; ++r)
                tma_load_2d(bx + (p * MP + r * 16) * 128, &tmB, kc + 64 * x, p * g.plane_rows + g.row0 + r * 16,
                            &full[s], pol_x);
          }
        }
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {  // ---------------- MMA issuer
      long long q = 0;
      int sidx = 0;
      for (long long w = w0; w < w1; ++sidx) {
        const int t = (int)(w / g.kb);
        const long long wend = min(w1, (long long)(t + 1) * g.kb);
        const int buf = sidx % NBUF;
        if (sidx >= NBUF) mbar_wait(&acc_empty[buf], (uint32_t)((sidx / NBUF) - 1) & 1u);
        tc_fence_after();
        const uint32_t acc = tmem + (uint32_t)(buf * NACC * ACCW);
        for (long long i = 0; w + i < wend; ++i, ++q) {
          const int s = (int)(q % stages);
          mbar_wait(&full[s], (uint32_t)(q / stages) & 1u);
          if (q == 0) gstamp(g, 3);
          tc_fence_after();
          uint8_t* st = smem + (size_t)s * stage_bytes;
#pragma unroll
          for (int x = 0; x < KBOX; ++x) {
            const uint64_t a0 = sw128_desc(st + x * BOX_BYTES);
            const uint64_t a1 = DUAL ? sw128_desc(st + A_BYTES + x * BOX_BYTES) : 0ull;
            uint8_t* bx = st + NACC * A_BYTES + (size_t)x * NB * MP * 128;
#pragma unroll
            for (int k = 0; k < 4; ++k) {  // 64 = 4 x UMMA_K(16); +32 bytes per step inside the swizzle atom
              if (cat) {  // all terms in one MMA (N = NB * MP), each into its own column group
                const uint64_t bp = sw128_desc(bx);
                const uint32_t accf = (i > 0 || x > 0 || k > 0) ? 1u : 0u;
                mma_bf16(acc, a0 + 2 * k, bp + 2 * k, idesc, accf);
                if (DUAL) mma_bf16(acc + ACCW, a1 + 2 * k, bp + 2 * k, idesc, accf);
              } else {
                for (int p = 0; p < NB; ++p) {  // the activation's bf16 terms, all into one accumulator
                  const uint64_t bp = sw128_desc(bx + p * MP * 128);
                  const uint32_t accf = (i > 0 || x > 0 || k > 0 || p > 0) ? 1u : 0u;
                  mma_bf16(acc, a0 + 2 * k, bp + 2 * k, idesc, accf);
                  if (DUAL) mma_bf16(acc + ACCW, a1 + 2 * k, bp + 2 * k, idesc, accf);
                }
              }
            }
          }
          mma_commit(&empty[s]);  // smem slot free once these MMAs have read it
        }
        mma_commit(&acc_full[buf]);  // this segment's accumulator complete
        w = wend;
      }
    }
  } else {  // ---------------- epilogue warps 0-3 (thread = TMEM lane = weight row of the tile)
    pdl_wait();
    ParDst pdst;
    const ParDst* pd = nullptr;
    if (!DUAL && g.par.world) {
      const unsigned long long s1 = __ldcg(g.par.seq) + 1ull;  // written by the previous producer
      const size_t base = (size_t)(s1 & 1ull) * g.par.world * g.par.slot_n;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        pdst.slot[q] = q < g.par.world ? reinterpret_cast<float*>(g.par.peers[q]) + base +
                                             (size_t)(g.par.loopback ? q : g.par.rank) * g.par.slot_n
                                       : nullptr;
      pd = &pdst;
    }
    int sidx = 0;
    for (long long w = w0; w < w1; ++sidx) {
      const int t = (int)(w / g.kb);
      const int kbeg = (int)(w % g.kb);
      const long long wend = min(w1, (long long)(t + 1) * g.kb);
      const int buf = sidx % NBUF;
      mbar_wait(&acc_full[buf], (uint32_t)(sidx / NBUF) & 1u);
      if (tid == 0 && sidx == 0) gstamp(g, 4);
      tc_fence_after();
      const uint32_t tbase = tmem + (uint32_t)(buf * NACC * ACCW) + ((uint32_t)(warp * 32) << 16);
      const int n = t * 128 + tid;
      const bool complete = (kbeg == 0 && wend == (long long)(t + 1) * g.kb);
      const int ngrp = cat ? NB : 1;
      // columns j0..j0+15 of operand a, the term column groups summed in term order
      auto acc_ld = [&](int a, int j0, float* v) {
        tmem_ld16(tbase + a * ACCW + j0, v);
        for (int p = 1; p < ngrp; ++p) {
          float u[16];
          tmem_ld16(tbase + a * ACCW + p * MP + j0, u);
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] += u[j];
        }
      };
      if (complete) {
        for (int j0 = 0; j0 < MP; j0 += 16) {
          float v0[16], v1[16];
          acc_ld(0, j0, v0);
          if (DUAL) acc_ld(1, j0, v1);
#pragma unroll
          for (int j = 0; j < 16; ++j) epi_store<DUAL>(g, j0 + j, n, v0[j], DUAL ? v1[j] : 0.f, pd);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[buf]);
      } else {
        const int slot = (w == w0) ? 0 : 1;
        float* mine = g.part + ((size_t)(c * 2 + slot) * NACC) * 256 * 128;
        for (int j0 = 0; j0 < MP; j0 += 16) {
          float v[16];
          for (int a = 0; a < NACC; ++a) {
            acc_ld(a, j0, v);
#pragma unroll
            for (int j = 0; j < 16; ++j) mine[((size_t)a * 256 + j0 + j) * 128 + tid] = v[j];
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[buf]);  // TMEM drained; the fix-up below reads global memory
        const int cf = owner_of((long long)t * g.kb, W, G);
        const int cl = owner_of(min(W, (long long)(t + 1) * g.kb) - 1, W, G);
        if (epi_arrive_last(g.counters + t, (unsigned)(cl - cf + 1), flag_s)) {
          for (int j0 = 0; j0 < MP; j0 += 16) {
            float s0[16], s1[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) s0[j] = s1[j] = 0.f;
            for (int cc = cf; cc <= cl; ++cc) {  // fixed CTA order -> deterministic
              const long long cw0 = W * cc / G;
              const int sl = ((int)(cw0 / g.kb) == t) ? 0 : 1;
              const float* p = g.part + ((size_t)(cc * 2 + sl) * NACC) * 256 * 128;
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                s0[j] += __ldcg(p + (size_t)(j0 + j) * 128 + tid);
                if (DUAL) s1[j] += __ldcg(p + ((size_t)256 + j0 + j) * 128 + tid);
              }
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) epi_store<DUAL>(g, j0 + j, n, s0[j], s1[j], pd);
          }
        }
      }
      w = wend;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (tid == 0) gstamp(g, 5);  // all segments (epilogue + fix-up) done
  if (g.par.world && warp == 0) {  // fused all-reduce: the last CTA with work publishes the sync point
    unsigned last = 0u;
    if (lane == 0) {
      __threadfence_system();  // this CTA's peer stores (ordered before by the barrier above)
      const unsigned old = atomicAdd(g.par.done, 1u);
      last = old == (unsigned)g.par_ctas - 1 ? 1u : 0u;
      if (last) {
        atomicExch(g.par.done, 0u);
        __threadfence_system();  // every CTA's stores: their fences precede their arrivals
      }
    }
    last = __shfl_sync(0xffffffffu, last, 0);  // warp-synchronising: lane 0's observations reach the lanes
    if (last) {
      const unsigned long long s1 = __ldcg(g.par.seq) + 1ull;
      const int W = g.par.world;
      if (lane < W)  // lanes 0..W-1 release the W flags in one instruction
        par::st_release_sys(reinterpret_cast<unsigned long long*>(g.par.peers[lane] + par::off_flags(g.par)) +
                                (size_t)(s1 & 1ull) * W + (g.par.loopback ? lane : g.par.rank),
                            s1);
      __syncwarp();
      if (lane == 0) *g.par.seq = s1;
    }
  }
  if (warp == 5) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(ncols) : "memory");
  }
}

// ===================================================================== host side
namespace launch {

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  }
  return fn;
}

// bf16 tensor map, SWIZZLE_128B (64-element = 128-byte inner box), rank 2..4; strides in bytes.
static bool encode(CUtensorMap* map, const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
                   const cuuint32_t* box) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) return false;
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, (cuuint32_t)rank, const_cast<void*>(base), dims, strides, box,
                   es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}
// weights [N, K] row-major.  coarse: 3-D view (64, N, K/64) — strides K*2 (rows), 128 B (K blocks) — with a
// box of 64 x 128 rows x kbox, so one op fetches a stage's [kbox][128 rows][64] tile; else 2-D box 64 x 128.
static bool map_weights(CUtensorMap* m, const void* w, int N, int K, int kbox, bool coarse) {
  if (coarse) {
    cuuint64_t dims[3] = {64, (cuuint64_t)N, (cuuint64_t)(K / 64)};
    cuuint64_t strides[2] = {(cuuint64_t)K * 2, 128};
    cuuint32_t box[3] = {64, 128, (cuuint32_t)kbox};
    return encode(m, w, 3, dims, strides, box);
  }
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)N};
  cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {64, 128};
  return encode(m, w, 2, dims, strides, box);
}
// activation term planes [nt][rows][K].  coarse: 4-D view (64, rows, nt, K/64) with a box of
// 64 x MP x nt x kbox -> smem [kbox][nt][MP][64] in one op; else 2-D [nt * rows, K], box 64 x 16 rows.
static bool map_acts(CUtensorMap* m, const void* x, int nt, int rows, int K, int MP, int kbox, bool coarse) {
  if (coarse) {
    cuuint64_t dims[4] = {64, (cuuint64_t)rows, (cuuint64_t)nt, (cuuint64_t)(K / 64)};
    cuuint64_t strides[3] = {(cuuint64_t)K * 2, (cuuint64_t)rows * K * 2, 128};
    cuuint32_t box[4] = {64, (cuuint32_t)MP, (cuuint32_t)nt, (cuuint32_t)kbox};
    return encode(m, x, 4, dims, strides, box);
  }
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)nt * rows};
  cuuint64_t strides[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {64, 16};
  return encode(m, x, 2, dims, strides, box);
}
int g_gemm_coarse = 1;  // SIRIUS_GEMM_COARSE=0: one TMA op per 64-wide box (A/B timing)

size_t gemm_workspace_bytes(int num_sms) { return (size_t)num_sms * 2 * 2 * 256 * 128 * sizeof(float); }

int g_gemm_kbox = 2;  // 64-wide K boxes per stage (SIRIUS_GEMM_KBOX)

template <bool DUAL, int KBOX>
static cudaError_t gemm_k(const void* w0, const void* w1, const void* x, GemmArgs g, int MP, int num_sms,
                          size_t smem_budget, cudaStream_t st) {
  const int NACC = DUAL ? 2 : 1;
  const int NB = g.nterms;
  g.kb = (g.K + 64 * KBOX - 1) / (64 * KBOX);
  // coarse boxes need whole 64-wide K blocks and <= 256 activation rows per box
  g.coarse = (g_gemm_coarse && g.K % 64 == 0 && MP <= 256) ? 1 : 0;
  CUtensorMap a0, a1, b;
  if (!map_weights(&a0, w0, g.N, g.K, KBOX, g.coarse) || (DUAL && !map_weights(&a1, w1, g.N, g.K, KBOX, g.coarse)) ||
      !map_acts(&b, x, NB, g.plane_rows, g.K, MP, KBOX, g.coarse))
    return cudaErrorInvalidValue;
  if (!DUAL) a1 = a0;
  const size_t stage_bytes = ((size_t)KBOX * (NACC * 16384 + (size_t)NB * MP * 128) + 1023) & ~(size_t)1023;
  const size_t extra = 1024 + 512;
  int stages = (int)((smem_budget - extra) / stage_bytes);
  if (stages > 8) stages = 8;
  if (stages < 2) return cudaErrorInvalidValue;
  const size_t smem = (size_t)stages * stage_bytes + extra;
  const long long W = (long long)g.n_tiles * g.kb;
  const int grid = (int)(W < num_sms ? W : num_sms);
  g.par_ctas = grid;  // every CTA of the grid has work (W >= grid)
  auto kern = gemm_tc_kernel<DUAL, KBOX>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_chain(kern, dim3(grid), dim3(192), smem, st, a0, a1, b, g, MP, stages);
}

cudaError_t gemm(const void* a0, const void* a1, const void* b, const GemmArgs& g, int MP, int num_sms,
                 size_t smem_budget, cudaStream_t st) {
  if (MP < 16 || MP > 256 || MP % 16 || g.nterms < 1 || g.nterms > 3) return cudaErrorInvalidValue;
  const bool dual = a1 != nullptr;
  // KBOX boxes per stage need room for >= 2 stages (dual operands at large MP fall back to fewer)
  auto fits = [&](int kb) {
    return (size_t)kb * ((dual ? 2 : 1) * 16384 + (size_t)g.nterms * MP * 128) * 2 + 1536 <= smem_budget;
  };
  int kbox = 1;
  if (g_gemm_kbox >= 4 && fits(4)) kbox = 4;
  else if (g_gemm_kbox >= 2 && fits(2)) kbox = 2;
  if (dual) {
    if (kbox == 4) return gemm_k<true, 4>(a0, a1, b, g, MP, num_sms, smem_budget, st);
    if (kbox == 2) return gemm_k<true, 2>(a0, a1, b, g, MP, num_sms, smem_budget, st);
    return gemm_k<true, 1>(a0, a1, b, g, MP, num_sms, smem_budget, st);
  }
  if (kbox == 4) return gemm_k<false, 4>(a0, a1, b, g, MP, num_sms, smem_budget, st);
  if (kbox == 2) return gemm_k<false, 2>(a0, a1, b, g, MP, num_sms, smem_budget, st);
  return gemm_k<false, 1>(a0, a1, b, g, MP, num_sms, smem_budget, st);
}

}  // namespace launch
}  // namespace sirius
