// gemv_dev.cuh — device building blocks of the HBM-streaming decode kernels (gemv_ffn.cu and the
// persistent decode-step kernel decode_step.cu): the activation prologue (residual add + RMSNorm /
// embedding gather into shared-memory float4 planes) and the warp-per-row bf16 dot product.
#pragma once
#include "common.cuh"
#include "decode_kernels.cuh"

namespace sirius {
namespace dev {

// plane layout of an fp32 activation row of K elements: chunk c = 8 consecutive elements,
// plane p = 0 holds elements 8c..8c+3, plane 1 holds 8c+4..8c+7 (float4 per chunk per plane)

// Prologue: activation rows h[b, :] (plane layout) in shared memory; all NT threads participate.
// Thread t owns the 4-element groups g = t + NT j (plane-aligned: a group is one float4 of a plane);
// all of its global loads are issued before any is used (one memory round trip, not K / NT).
constexpr int kMaxGroups = 8;  // K <= 32 * NT
template <int B, int MG = kMaxGroups>  // MG: groups per thread, >= K / (4 NT)
SIRIUS_DEV void prologue(const Prologue& p, int K, float* h_s, float* red_s, bool store_res) {
  const int tid = threadIdx.x, NT = blockDim.x, warp = tid >> 5, lane = tid & 31, nwarp = NT >> 5;
  const int CH = K / 8, NG = K / 4;
  float4* hp = reinterpret_cast<float4*>(h_s);
  auto slot = [&](int b, int g) { return (b * 2 + (g & 1)) * CH + (g >> 1); };  // group g = elements 4g..4g+3
  for (int b = 0; b < B; ++b) {
    float4 x[MG];
    if (p.mode == IN_F32) {
      const float4* src = reinterpret_cast<const float4*>(p.in_f32 + (size_t)b * K);
#pragma unroll
      for (int j = 0; j < MG; ++j) {
        const int g = tid + NT * j;
        if (g < NG) x[j] = __ldcg(src + g);
      }
#pragma unroll
      for (int j = 0; j < MG; ++j) {
        const int g = tid + NT * j;
        if (g < NG) hp[slot(b, g)] = x[j];
      }
      continue;
    }
    if (p.mode == IN_EMBED) {
      int tok = p.tokens[b];
      tok = tok < 0 ? 0 : (tok >= p.vocab ? p.vocab - 1 : tok);
      const uint2* erow = reinterpret_cast<const uint2*>(p.embed + (size_t)tok * K);
#pragma unroll
      for (int j = 0; j < MG; ++j) {
        const int g = tid + NT * j;
        if (g < NG) {
          const uint2 e = erow[g];
          x[j] = make_float4(bf16_lo(e.x), bf16_hi(e.x), bf16_lo(e.y), bf16_hi(e.y));
        }
      }
    } else {
      const float4* base = reinterpret_cast<const float4*>(p.base + (size_t)b * K);
      const float4* delta = p.delta ? reinterpret_cast<const float4*>(p.delta + (size_t)b * K) : nullptr;
      float4 dl[MG];
#pragma unroll
      for (int j = 0; j < MG; ++j) {
        const int g = tid + NT * j;
        if (g < NG) {
          x[j] = __ldcg(base + g);
          dl[j] = delta ? __ldcg(delta + g) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
      for (int j = 0; j < MG; ++j) {
        x[j].x += dl[j].x; x[j].y += dl[j].y; x[j].z += dl[j].z; x[j].w += dl[j].w;
      }
    }
    float ss = 0.f;
#pragma unroll
    for (int j = 0; j < MG; ++j) {  // sum of squares, fixed order
      const int g = tid + NT * j;
      if (g < NG) {
        ss = fmaf(x[j].x, x[j].x, ss); ss = fmaf(x[j].y, x[j].y, ss);
        ss = fmaf(x[j].z, x[j].z, ss); ss = fmaf(x[j].w, x[j].w, ss);
        if (store_res && p.res_out) reinterpret_cast<float4*>(p.res_out + (size_t)b * K)[g] = x[j];
      }
    }
    uint2 wn[MG];
    const uint2* nw = reinterpret_cast<const uint2*>(p.norm_w);
#pragma unroll
    for (int j = 0; j < MG; ++j) {
      const int g = tid + NT * j;
      if (g < NG) wn[j] = nw[g];
    }
    ss = warp_sum(ss);
    if (lane == 0) red_s[warp] = ss;
    __syncthreads();
    float tot = 0.f;
    for (int w = 0; w < nwarp; ++w) tot += red_s[w];
    const float r = 1.0f / sqrtf(tot / (float)K + p.eps);
#pragma unroll
    for (int j = 0; j < MG; ++j) {
      const int g = tid + NT * j;
      if (g < NG)
        hp[slot(b, g)] = make_float4((x[j].x * r) * bf16_lo(wn[j].x), (x[j].y * r) * bf16_hi(wn[j].x),
                                     (x[j].z * r) * bf16_lo(wn[j].y), (x[j].w * r) * bf16_hi(wn[j].y));
    }
    __syncthreads();  // red_s reuse
  }
  __syncthreads();
}

SIRIUS_DEV float dot8p(const uint4 w, const float4 x0, const float4 x1, float s) {
  s = fmaf(bf16_lo(w.x), x0.x, s);
  s = fmaf(bf16_hi(w.x), x0.y, s);
  s = fmaf(bf16_lo(w.y), x0.z, s);
  s = fmaf(bf16_hi(w.y), x0.w, s);
  s = fmaf(bf16_lo(w.z), x1.x, s);
  s = fmaf(bf16_hi(w.z), x1.y, s);
  s = fmaf(bf16_lo(w.w), x1.z, s);
  s = fmaf(bf16_hi(w.w), x1.w, s);
  return s;
}

// Warp-cooperative dot of one bf16 row (global) with the B activation rows (planes in smem).
// Lane l handles chunks l + 32 j; loads are issued in groups of U before use.  Result: lane sums
// (not yet reduced across the warp).
template <int B, int CPL>
SIRIUS_DEV void row_dot(const uint16_t* __restrict__ wrow, const float4* __restrict__ hp, int CH, int lane,
                        float* acc, uint64_t pol) {
  constexpr int U = CPL < 16 ? CPL : 16;
#pragma unroll
  for (int b = 0; b < B; ++b) acc[b] = 0.f;
#pragma unroll
  for (int j0 = 0; j0 < CPL; j0 += U) {
    uint4 wv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = lane + 32 * (j0 + u);
      wv[u] = c < CH ? ld_nc_v4_ef(wrow + (size_t)c * 8, pol) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = lane + 32 * (j0 + u);
      if (c < CH) {
#pragma unroll
        for (int b = 0; b < B; ++b) acc[b] = dot8p(wv[u], hp[(b * 2) * CH + c], hp[(b * 2 + 1) * CH + c], acc[b]);
      }
    }
  }
}


}  // namespace dev
}  // namespace sirius

namespace sirius {
namespace dev {

// ---- split row dot: issue a warp's 128-bit loads of one bf16 row (chunks lane + 32 u, u < PF) into
// registers now, finish (and stream any chunks u >= PF) later.  Lets a warp request its next row
// before reducing the current one, and request its first row of the next phase before a barrier.
template <int CPL>
struct RowRegs {
  static constexpr int PF = CPL < 16 ? CPL : 16;
  uint4 v[PF];
};

// 0, opaque to the compiler and data-dependent on `dep`: added to the next row's address it keeps
// that row's loads after the FMAs that produce dep (else they are hoisted and two rows' registers
// are live at once, which spills at 512 threads / 128 registers).
SIRIUS_DEV size_t after(float dep) {
  uint32_t z;
  asm volatile("{\n\t.reg .f32 t;\n\tmov.b32 t, %1;\n\tmov.b32 %0, 0;\n\t}" : "=r"(z) : "f"(dep));
  return z;
}
template <int B>
SIRIUS_DEV size_t after_all(const float* acc) {
  float dep = acc[0];
#pragma unroll
  for (int b = 1; b < B; ++b) dep += acc[b];
  return after(dep);
}

// Always overwrites every register of r (zeros when !valid), so stale rows are never live.
template <int CPL>
SIRIUS_DEV void row_issue(RowRegs<CPL>& r, const uint16_t* __restrict__ wrow, int CH, int lane, bool valid,
                          uint64_t pol) {
#pragma unroll
  for (int u = 0; u < RowRegs<CPL>::PF; ++u) {
    const int c = lane + 32 * u;
    r.v[u] = (valid && c < CH) ? ld_nc_v4_ef(wrow + (size_t)c * 8, pol) : make_uint4(0u, 0u, 0u, 0u);
  }
}

// acc[b] = lane's partial dot of the row with activation row b (planes in smem); same per-lane
// summation order as row_dot (chunks ascending).
template <int B, int CPL>
SIRIUS_DEV void row_finish(const RowRegs<CPL>& r, const uint16_t* __restrict__ wrow, const float4* __restrict__ hp,
                           int CH, int lane, float* acc) {
  constexpr int PF = RowRegs<CPL>::PF;
#pragma unroll
  for (int b = 0; b < B; ++b) acc[b] = 0.f;
#pragma unroll
  for (int u = 0; u < PF; ++u) {
    const int c = lane + 32 * u;
    if (c < CH) {
#pragma unroll
      for (int b = 0; b < B; ++b) acc[b] = dot8p(r.v[u], hp[(b * 2) * CH + c], hp[(b * 2 + 1) * CH + c], acc[b]);
    }
  }
#pragma unroll
  for (int j0 = PF; j0 < CPL; j0 += 16) {  // d = 8192: the second half of the row
    uint4 wv[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int c = lane + 32 * (j0 + u);
      wv[u] = c < CH ? ld_nc_v4(wrow + (size_t)c * 8) : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int c = lane + 32 * (j0 + u);
      if (c < CH) {
#pragma unroll
        for (int b = 0; b < B; ++b) acc[b] = dot8p(wv[u], hp[(b * 2) * CH + c], hp[(b * 2 + 1) * CH + c], acc[b]);
      }
    }
  }
}

}  // namespace dev
}  // namespace sirius
