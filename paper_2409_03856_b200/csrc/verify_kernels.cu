// verify_kernels.cu — the non-GEMM kernels of the full-model verification / prefill forward and of
// the Sirius accept / commit steps (Algorithm 1).
//
//  * norm_rows_kernel      residual add (or embedding gather) + RMSNorm of M token rows -> bf16
//  * rope_store_kernel     RoPE(q, k) at each row's position, bf16; K/V -> staging (verify) or cache
//  * accept_stats_kernel   per logits row (rank shard, vocab split): max, lowest-index argmax,
//                          sum of exp, and the draft token's logit
//  * accept_finalize_kernel  LSE, q_i = softmax(l_i)[d_{i+1}], first rejection j, interleaved token
//  * kv_rewrite_kernel     staging rows [0, n) -> cache slots [T, T + n) in every layer (commit +
//                          rollback, PAPER.md:257/:264/:294)
//  * transpose / rank-sum helpers
#include "common.cuh"
#include "verify_kernels.cuh"
#include "peer_ar.cuh"

namespace sirius {

// ===================================================================== norm rows
__global__ void __launch_bounds__(256) norm_rows_kernel(NormRowsArgs a) {
  pdl_trigger();
  pdl_wait();
  // thread t owns 4-element groups g = t + 256 j; every global load is issued before use
  constexpr int MG = 8;  // d <= 8192
  const int m = blockIdx.x, tid = threadIdx.x, d = a.d, NG = d / 4;
  __shared__ float red[8];
  float4 x[MG];
  if (a.tokens) {
    int tok = a.tokens[m];
    tok = tok < 0 ? 0 : (tok >= a.vocab ? a.vocab - 1 : tok);
    const uint2* erow = reinterpret_cast<const uint2*>(a.embed + (size_t)tok * d);
#pragma unroll
    for (int j = 0; j < MG; ++j) {
      const int g = tid + 256 * j;
      if (g < NG) {
        const uint2 e = erow[g];
        x[j] = make_float4(bf16_lo(e.x), bf16_hi(e.x), bf16_lo(e.y), bf16_hi(e.y));
      }
    }
  } else {
    const float4* base = reinterpret_cast<const float4*>(a.base + (size_t)m * d);
    const float4* delta = a.delta ? reinterpret_cast<const float4*>(a.delta + (size_t)m * d) : nullptr;
    float4 dl[MG];
#pragma unroll
    for (int j = 0; j < MG; ++j) {
      const int g = tid + 256 * j;
      if (g < NG) {
        x[j] = __ldcg(base + g);
        dl[j] = delta ? __ldcg(delta + g) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    if (a.par_consume) {  // fused peer all-reduce: ((s_0 + s_1) + ...) * scale, as the in-order sum
      const unsigned long long s = __ldcg(a.par.seq);
      par::wait_flags(a.par, s);
      const float* slots = reinterpret_cast<const float*>(a.par.self) + (size_t)(s & 1ull) * a.par.world * a.par.slot_n;
      for (int r0 = 0; r0 < a.par.world; r0 += 2) {  // two ranks' rows in flight per round
        float4 v[2][MG];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const float4* sr = reinterpret_cast<const float4*>(slots + (size_t)(r0 + u) * a.par.slot_n + (size_t)m * d);
#pragma unroll
          for (int j = 0; j < MG; ++j)
            if (r0 + u < a.par.world && tid + 256 * j < NG) v[u][j] = __ldcg(sr + tid + 256 * j);
        }
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int j = 0; j < MG; ++j)
            if (r0 + u < a.par.world && tid + 256 * j < NG) {
              if (r0 + u == 0) {
                dl[j] = v[u][j];
              } else {
                dl[j].x += v[u][j].x; dl[j].y += v[u][j].y; dl[j].z += v[u][j].z; dl[j].w += v[u][j].w;
              }
            }
      }
#pragma unroll
      for (int j = 0; j < MG; ++j) {
        dl[j].x *= a.par.scale; dl[j].y *= a.par.scale; dl[j].z *= a.par.scale; dl[j].w *= a.par.scale;
      }
    }
#pragma unroll
    for (int j = 0; j < MG; ++j) {
      x[j].x += dl[j].x; x[j].y += dl[j].y; x[j].z += dl[j].z; x[j].w += dl[j].w;
    }
  }
  uint2 wn[MG];
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < MG; ++j) {
    const int g = tid + 256 * j;
    if (g < NG) {
      wn[j] = reinterpret_cast<const uint2*>(a.norm_w)[g];
      ss = fmaf(x[j].x, x[j].x, ss); ss = fmaf(x[j].y, x[j].y, ss);
      ss = fmaf(x[j].z, x[j].z, ss); ss = fmaf(x[j].w, x[j].w, ss);
      if (a.res_out) reinterpret_cast<float4*>(a.res_out + (size_t)m * d)[g] = x[j];
    }
  }
  ss = warp_sum(ss);
  if ((tid & 31) == 0) red[tid >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
  for (int w = 0; w < 8; ++w) tot += red[w];
  const float r = 1.0f / sqrtf(tot / (float)d + a.eps);
#pragma unroll
  for (int j = 0; j < MG; ++j) {
    const int g = tid + 256 * j;
    if (g < NG) {
      const float h[4] = {(x[j].x * r) * bf16_lo(wn[j].x), (x[j].y * r) * bf16_hi(wn[j].x),
                          (x[j].z * r) * bf16_lo(wn[j].y), (x[j].w * r) * bf16_hi(wn[j].y)};
      uint16_t t[4][3];
#pragma unroll
      for (int e = 0; e < 4; ++e) split3(h[e], t[e]);
#pragma unroll
      for (int p = 0; p < 3; ++p)
        reinterpret_cast<uint2*>(a.out3 + p * a.plane + (size_t)m * d)[g] =
            make_uint2(t[0][p] | ((uint32_t)t[1][p] << 16), t[2][p] | ((uint32_t)t[3][p] << 16));
    }
  }
}

// ===================================================================== RoPE + K/V store
__global__ void __launch_bounds__(128) rope_store_kernel(RopeStoreArgs a) {
  pdl_trigger();
  pdl_wait();
  const int m = blockIdx.x, tid = threadIdx.x, hd = a.hd, half = hd / 2;
  const int b = a.b_base + m / a.rows_per_seq, i = m % a.rows_per_seq;
  const int pos = a.start[b] + (a.row_off ? a.row_off[i] : i);
  const int si = a.stage_base + i;  // staging row
  const bool bad = pos < 0 || pos >= a.max_seq || (a.to_cache == 0 && si >= a.max_gamma);
  if (bad) {
    if (tid == 0) atomicOr(a.err, 2);
    return;
  }
  const float* row = a.qkv + (size_t)m * (a.Hr + 2 * a.KVr) * hd;
  const float4* cs = reinterpret_cast<const float4*>(a.rope_cos + (size_t)pos * half);
  const float4* sn = reinterpret_cast<const float4*>(a.rope_sin + (size_t)pos * half);
  // rotate-half pairs (e, e + half) in groups of 4 consecutive e: items = (Hr + KVr) * half / 4
  constexpr int MI = 8;  // items per thread per round
  const int q4 = half / 4, items = (a.Hr + a.KVr) * q4;
  for (int it0 = 0; it0 < items; it0 += 128 * MI) {
  float4 x0[MI], x1[MI], c4[MI], s4[MI];
#pragma unroll
  for (int j = 0; j < MI; ++j) {
    const int it = it0 + tid + 128 * j;
    if (it < items) {
      const int h = it / q4, e4 = it % q4;
      x0[j] = __ldcg(reinterpret_cast<const float4*>(row + h * hd) + e4);
      x1[j] = __ldcg(reinterpret_cast<const float4*>(row + h * hd + half) + e4);
      c4[j] = cs[e4];
      s4[j] = sn[e4];
    }
  }
#pragma unroll
  for (int j = 0; j < MI; ++j) {
    const int it = it0 + tid + 128 * j;
    if (it >= items) continue;
    const int h = it / q4, e = (it % q4) * 4;
    const float4 a0 = x0[j], a1 = x1[j], c = c4[j], s = s4[j];
    const float4 y0 = make_float4(a0.x * c.x - a1.x * s.x, a0.y * c.y - a1.y * s.y, a0.z * c.z - a1.z * s.z,
                                  a0.w * c.w - a1.w * s.w);
    const float4 y1 = make_float4(a1.x * c.x + a0.x * s.x, a1.y * c.y + a0.y * s.y, a1.z * c.z + a0.z * s.z,
                                  a1.w * c.w + a0.w * s.w);
    if (h < a.Hr) {
      *reinterpret_cast<float4*>(a.q_out + (size_t)m * a.Hr * hd + h * hd + e) = y0;
      *reinterpret_cast<float4*>(a.q_out + (size_t)m * a.Hr * hd + h * hd + e + half) = y1;
    } else {
      const int kvh = h - a.Hr;
      uint16_t* dst = a.to_cache ? a.k_dst + (((size_t)b * a.KVr + kvh) * a.max_seq + pos) * hd
                                 : a.k_dst + (((size_t)b * a.KVr + kvh) * a.max_gamma + si) * hd;
      *reinterpret_cast<uint2*>(dst + e) = make_uint2(pack_bf16(y0.x, y0.y), pack_bf16(y0.z, y0.w));
      *reinterpret_cast<uint2*>(dst + e + half) = make_uint2(pack_bf16(y1.x, y1.y), pack_bf16(y1.z, y1.w));
    }
  }
  }
  const int v4 = a.KVr * hd / 4;
  for (int it0 = 0; it0 < v4; it0 += 128 * 4) {
  float4 vv[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int it = it0 + tid + 128 * j;
    if (it < v4) vv[j] = __ldcg(reinterpret_cast<const float4*>(row + (a.Hr + a.KVr) * hd) + it);
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int it = it0 + tid + 128 * j;
    if (it >= v4) continue;
    const int kvh = (it * 4) / hd, e = (it * 4) % hd;
    uint16_t* dst = a.to_cache ? a.v_dst + (((size_t)b * a.KVr + kvh) * a.max_seq + pos) * hd
                               : a.v_dst + (((size_t)b * a.KVr + kvh) * a.max_gamma + si) * hd;
    *reinterpret_cast<uint2*>(dst + e) = make_uint2(pack_bf16(vv[j].x, vv[j].y), pack_bf16(vv[j].z, vv[j].w));
  }
  }
}

// ===================================================================== acceptance
__global__ void __launch_bounds__(256) accept_stats_kernel(AcceptStatsArgs a) {
  pdl_trigger();
  pdl_wait();
  const int m = blockIdx.x, split = blockIdx.y, S = gridDim.y, tid = threadIdx.x;
  const int b = m / a.gamma, i = m % a.gamma;
  const int draft = (i < a.gamma - 1) ? a.tokens[b * a.gamma + i + 1] : -1;
  const int v0 = (int)((long long)a.Vr * split / S), v1 = (int)((long long)a.Vr * (split + 1) / S);
  const float* row = a.logits + (size_t)m * a.ldl;
  __shared__ float red_f[8];
  __shared__ unsigned long long red_k[8];
  float mx = -INFINITY;
  unsigned long long key = 0ull;
  for (int v = v0 + tid; v < v1; v += 256) {
    const float l = row[v];
    mx = fmaxf(mx, l);
    const unsigned long long k = argmax_key(l, (uint32_t)(a.voff + v));
    key = k > key ? k : key;
  }
  mx = warp_max(mx);
  key = warp_max_u64(key);
  if ((tid & 31) == 0) {
    red_f[tid >> 5] = mx;
    red_k[tid >> 5] = key;
  }
  __syncthreads();
  float M = -INFINITY;
  unsigned long long K = 0ull;
  for (int w = 0; w < 8; ++w) {
    M = fmaxf(M, red_f[w]);
    K = red_k[w] > K ? red_k[w] : K;
  }
  __syncthreads();
  float s = 0.f;
  for (int v = v0 + tid; v < v1; v += 256) s += expf(row[v] - M);
  s = warp_sum(s);
  if ((tid & 31) == 0) red_f[tid >> 5] = s;
  __syncthreads();
  if (tid == 0) {
    float tot = 0.f;
    for (int w = 0; w < 8; ++w) tot += red_f[w];
    RowStat st;
    st.mx = M;
    st.sum = tot;
    st.key = K;
    const int dl = draft - a.voff;
    st.ld = (draft >= 0 && dl >= v0 && dl < v1) ? row[dl] : -INFINITY;
    st.pad = 0.f;
    a.stats[((size_t)a.rank * a.M + m) * S + split] = st;
  }
}

// one CTA per sequence; thread i = verify row i (gamma <= 64)
__global__ void __launch_bounds__(64) accept_finalize_kernel(AcceptFinalArgs a) {
  pdl_wait();
  const int b = blockIdx.x, i = threadIdx.x, gam = a.gamma;
  __shared__ float q_s[64];
  __shared__ int am_s[64];
  if (i < gam) {
    const int m = b * gam + i;
    float M = -INFINITY, ld = -INFINITY;
    unsigned long long K = 0ull;
    for (int r = 0; r < a.nranks; ++r)
      for (int sp = 0; sp < a.S; ++sp) {
        const RowStat st = a.stats[((size_t)r * a.M + m) * a.S + sp];
        M = fmaxf(M, st.mx);
        K = st.key > K ? st.key : K;
        ld = fmaxf(ld, st.ld);
      }
    float tot = 0.f;
    for (int r = 0; r < a.nranks; ++r)
      for (int sp = 0; sp < a.S; ++sp) {
        const RowStat st = a.stats[((size_t)r * a.M + m) * a.S + sp];
        tot += st.sum * expf(st.mx - M);
      }
    const float lse = M + logf(tot);
    const float q = (i < gam - 1) ? expf(ld - lse) : expf(M - lse);
    q_s[i] = q;
    am_s[i] = (int)argmax_key_index(K);
    if (a.row_argmax) a.row_argmax[(size_t)b * gam + i] = am_s[i];
    if (a.q_out) a.q_out[(size_t)b * gam + i] = q;
  }
  __syncthreads();
  if (i == 0) {
    int j = gam - 1;
    for (int k = 0; k < gam - 1; ++k) {
      const int d = a.tokens[b * gam + k + 1];
      const bool ok = a.mode == 0 ? (q_s[k] >= a.r) : (d == am_s[k]);
      if (!ok) {
        j = k;
        break;
      }
    }
    a.n_accept[b] = j;
    a.next_token[b] = am_s[j];
  }
}

// ===================================================================== KV rewrite (commit + rollback)
__global__ void __launch_bounds__(128) kv_rewrite_kernel(KvRewriteArgs a) {
  const int l = blockIdx.x / (a.B * a.KVr), rem = blockIdx.x % (a.B * a.KVr);
  const int b = rem / a.KVr, kvh = rem % a.KVr;
  const int T = a.start[b], n = a.n_rows[b];
  if (n < 1 || n > a.gamma || T < 0 || T + n > a.max_seq) {
    if (threadIdx.x == 0) atomicOr(a.err, 4);
    return;
  }
  const size_t hb = ((size_t)l * a.B + b) * a.KVr + kvh;
  const uint4* ks = reinterpret_cast<const uint4*>(a.stage_k + hb * a.max_gamma * a.hd);
  const uint4* vs = reinterpret_cast<const uint4*>(a.stage_v + hb * a.max_gamma * a.hd);
  uint4* kd = reinterpret_cast<uint4*>(a.k_cache + (hb * a.max_seq + T) * a.hd);
  uint4* vd = reinterpret_cast<uint4*>(a.v_cache + (hb * a.max_seq + T) * a.hd);
  const int rv = a.hd / 8;  // uint4 per row
  const int nvec = n * rv;
  for (int e = threadIdx.x; e < nvec; e += 128) {
    const int r = e / rv, c = e % rv;
    const int src = a.rows ? a.rows[r] * rv + c : e;  // tree commit: the winning path's staging rows
    kd[e] = ks[src];
    vd[e] = vs[src];
  }
}

// ===================================================================== helpers
__global__ void transpose_bf16_kernel(const uint16_t* __restrict__ in, uint16_t* __restrict__ out, int R, int C) {
  __shared__ uint16_t tile[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int y = threadIdx.y; y < 32; y += 8) {
    const int r = r0 + y, c = c0 + threadIdx.x;
    if (r < R && c < C) tile[y][threadIdx.x] = in[(size_t)r * C + c];
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += 8) {
    const int c = c0 + y, r = r0 + threadIdx.x;
    if (r < R && c < C) out[(size_t)c * R + r] = tile[threadIdx.x][y];
  }
}

// in-order sum over emulated TP ranks; result written back to every rank's buffer
__global__ void sum_ranks_kernel(float* const* bufs, int nranks, size_t n, size_t ld, size_t width) {
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (size_t)gridDim.x * blockDim.x) {
    const size_t row = idx / width, col = idx % width, off = row * ld + col;
    float s = 0.f;
    for (int r = 0; r < nranks; ++r) s += bufs[r][off];
    for (int r = 0; r < nranks; ++r) bufs[r][off] = s;
  }
}

namespace launch {

bool g_chain_pdl = true;
bool g_decode_pdl = true;  // measured: Sirius 2.653 -> 2.572 ms/token (tools/ab_env.sh)
#define LAUNCH_CHECK(x)                 \
  do {                                  \
    const cudaError_t e_ = (x);         \
    if (e_ != cudaSuccess) return e_;   \
  } while (0)

cudaError_t norm_rows(const NormRowsArgs& a, int M, cudaStream_t st) {
  LAUNCH_CHECK(launch_chain(norm_rows_kernel, dim3(M), dim3(256), 0, st, a));
  return cudaGetLastError();
}
cudaError_t rope_store(const RopeStoreArgs& a, int M, cudaStream_t st) {
  LAUNCH_CHECK(launch_chain(rope_store_kernel, dim3(M), dim3(128), 0, st, a));
  return cudaGetLastError();
}
cudaError_t accept_stats(const AcceptStatsArgs& a, int splits, cudaStream_t st) {
  LAUNCH_CHECK(launch_chain(accept_stats_kernel, dim3(a.M, splits), dim3(256), 0, st, a));
  return cudaGetLastError();
}
cudaError_t accept_finalize(const AcceptFinalArgs& a, int B, cudaStream_t st) {
  LAUNCH_CHECK(launch_chain(accept_finalize_kernel, dim3(B), dim3(64), 0, st, a));
  return cudaGetLastError();
}
cudaError_t kv_rewrite(const KvRewriteArgs& a, int L, cudaStream_t st) {
  kv_rewrite_kernel<<<L * a.B * a.KVr, 128, 0, st>>>(a);
  return cudaGetLastError();
}
cudaError_t transpose_bf16(const uint16_t* in, uint16_t* out, int R, int C, cudaStream_t st) {
  dim3 grid((C + 31) / 32, (R + 31) / 32);
  transpose_bf16_kernel<<<grid, dim3(32, 8), 0, st>>>(in, out, R, C);
  return cudaGetLastError();
}
cudaError_t sum_ranks(float* const* bufs_dev, int nranks, size_t rows, size_t width, size_t ld, cudaStream_t st) {
  const size_t n = rows * width;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 1184) blocks = 1184;
  sum_ranks_kernel<<<blocks, 256, 0, st>>>(bufs_dev, nranks, n, ld, width);
  return cudaGetLastError();
}

}  // namespace launch
}  // namespace sirius
