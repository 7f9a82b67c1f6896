// verify_kernels.cu — the non-GEMM kernels of the full-model verification / prefill forward and of
// the Sirius accept / commit steps (Algorithm 1).
//
//  * norm_rows_kernel      residual add (or embedding gather) + RMSNorm of M token rows -> bf16
//  * rope_store_kernel     RoPE(q, k) at each row's position, bf16; K/V -> staging (verify) or cache
//  * attn_rows_kernel      causal multi-row attention: row i of a kernel sees cache[0, T) and the
//                          kernel's own rows [0, i]; split-K over keys + last-CTA combine
//  * accept_stats_kernel   per logits row (rank shard, vocab split): max, lowest-index argmax,
//                          sum of exp, and the draft token's logit
//  * accept_finalize_kernel  LSE, q_i = softmax(l_i)[d_{i+1}], first rejection j, interleaved token
//  * kv_rewrite_kernel     staging rows [0, n) -> cache slots [T, T + n) in every layer (commit +
//                          rollback, PAPER.md:257/:264/:294)
//  * transpose / rank-sum helpers
#include "common.cuh"
#include "verify_kernels.cuh"

namespace sirius {

// ===================================================================== norm rows
__global__ void __launch_bounds__(256) norm_rows_kernel(NormRowsArgs a) {
  const int m = blockIdx.x, tid = threadIdx.x, d = a.d;
  __shared__ float red[8];
  const float* base = a.base ? a.base + (size_t)m * d : nullptr;
  const float* delta = a.delta ? a.delta + (size_t)m * d : nullptr;
  const uint16_t* erow = nullptr;
  if (a.tokens) {
    int tok = a.tokens[m];
    tok = tok < 0 ? 0 : (tok >= a.vocab ? a.vocab - 1 : tok);
    erow = a.embed + (size_t)tok * d;
  }
  auto xval = [&](int k) -> float {
    if (erow) return __uint_as_float((uint32_t)erow[k] << 16);
    float v = base[k];
    if (delta) v += delta[k];
    return v;
  };
  float ss = 0.f;
  for (int k = tid; k < d; k += 256) {
    const float v = xval(k);
    ss = fmaf(v, v, ss);
    if (a.res_out) a.res_out[(size_t)m * d + k] = v;
  }
  ss = warp_sum(ss);
  if ((tid & 31) == 0) red[tid >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
  for (int w = 0; w < 8; ++w) tot += red[w];
  const float r = 1.0f / sqrtf(tot / (float)d + a.eps);
  for (int k = tid; k < d; k += 256) {
    const float w = __uint_as_float((uint32_t)a.norm_w[k] << 16);
    const float h = (xval(k) * r) * w;
    const uint16_t hi = f2bf_bits(h);
    a.out_hi[(size_t)m * d + k] = hi;
    a.out_lo[(size_t)m * d + k] = f2bf_bits(h - __uint_as_float((uint32_t)hi << 16));
  }
}

// ===================================================================== RoPE + K/V store
__global__ void __launch_bounds__(128) rope_store_kernel(RopeStoreArgs a) {
  const int m = blockIdx.x, tid = threadIdx.x, hd = a.hd, half = hd / 2;
  const int b = a.b_base + m / a.rows_per_seq, i = m % a.rows_per_seq;
  const int pos = a.start[b] + i;
  const bool bad = pos < 0 || pos >= a.max_seq || (a.to_cache == 0 && i >= a.max_gamma);
  if (bad) {
    if (tid == 0) atomicOr(a.err, 2);
    return;
  }
  const float* row = a.qkv + (size_t)m * (a.Hr + 2 * a.KVr) * hd;
  const float* cs = a.rope_cos + (size_t)pos * half;
  const float* sn = a.rope_sin + (size_t)pos * half;
  for (int idx = tid; idx < (a.Hr + a.KVr) * half; idx += 128) {
    const int h = idx / half, e = idx % half;
    const float x0 = row[h * hd + e], x1 = row[h * hd + e + half], c = cs[e], s = sn[e];
    const float y0 = x0 * c - x1 * s, y1 = x1 * c + x0 * s;
    if (h < a.Hr) {
      a.q_out[(size_t)m * a.Hr * hd + h * hd + e] = y0;
      a.q_out[(size_t)m * a.Hr * hd + h * hd + e + half] = y1;
    } else {
      const uint16_t r0 = f2bf_bits(y0), r1 = f2bf_bits(y1);
      const int kvh = h - a.Hr;
      uint16_t* dst = a.to_cache ? a.k_dst + (((size_t)b * a.KVr + kvh) * a.max_seq + pos) * hd
                                 : a.k_dst + (((size_t)b * a.KVr + kvh) * a.max_gamma + i) * hd;
      dst[e] = r0;
      dst[e + half] = r1;
    }
  }
  for (int idx = tid; idx < a.KVr * hd; idx += 128) {
    const int kvh = idx / hd, e = idx % hd;
    const float v = row[(a.Hr + a.KVr + kvh) * hd + e];
    uint16_t* dst = a.to_cache ? a.v_dst + (((size_t)b * a.KVr + kvh) * a.max_seq + pos) * hd
                               : a.v_dst + (((size_t)b * a.KVr + kvh) * a.max_gamma + i) * hd;
    dst[e] = f2bf_bits(v);
  }
}

// ===================================================================== multi-row causal attention
// grid (splits, KVr * row_blocks, B); 128 threads = 64 query rows x 2 halves of head_dim.
template <int HD>
__global__ void __launch_bounds__(128) attn_rows_kernel(AttnRowsArgs a, float scale) {
  constexpr int H2 = HD / 2, KB = 32, LD = H2 + 1;
  const int split = blockIdx.x, bz = blockIdx.z, b = a.b_base + bz;  // bz: sequence within this launch
  const int kvh = blockIdx.y % a.KVr, rb = blockIdx.y / a.KVr;
  const int tid = threadIdx.x, half = tid & 1;
  const int G = a.G, rows = a.rows_per_seq;
  const int r = rb * 64 + (tid >> 1);  // row index within (b, kvh): r = i * G + g
  const int i = r / G, g = r % G;
  const bool valid = i < rows;
  __shared__ float k_s[KB][2][LD];
  __shared__ float v_s[KB][2][LD];
  const int T = a.start[b];
  // keys 0..T-1 from the cache prefix, T.. from the fresh rows (staging or cache)
  const int i_last = min(rows - 1, (rb * 64 + 63) / G);
  const int nkeys = max(0, T + i_last + 1);
  const int S = gridDim.x;
  const int chunk = (nkeys + S - 1) / S;
  const int k0 = min(nkeys, split * chunk), k1 = min(nkeys, k0 + chunk);
  const size_t hb = (size_t)b * a.KVr + kvh;
  const uint16_t* kc = a.k_cache + hb * a.max_seq * HD;
  const uint16_t* vc = a.v_cache + hb * a.max_seq * HD;
  const uint16_t* kf = a.fresh_in_cache ? kc + (size_t)T * HD : a.k_fresh + hb * a.fresh_stride * HD;
  const uint16_t* vf = a.fresh_in_cache ? vc + (size_t)T * HD : a.v_fresh + hb * a.fresh_stride * HD;

  float q[H2], acc[H2];
  float mrun = -INFINITY, lrun = 0.f;
  {
    const int m = bz * rows + (valid ? i : 0);
    const float* qp = a.q + (size_t)m * a.Hr * HD + (kvh * G + g) * HD + half * H2;
#pragma unroll
    for (int e = 0; e < H2; ++e) {
      q[e] = qp[e];
      acc[e] = 0.f;
    }
  }
  const int vis = T + i;  // last visible key for this row
  for (int p0 = k0; p0 < k1; p0 += KB) {
    __syncthreads();
    for (int idx = tid; idx < KB * HD; idx += 128) {
      const int pp = idx / HD, e = idx % HD, p = p0 + pp;
      float kv = 0.f, vv = 0.f;
      if (p < k1) {
        const uint16_t* ks = p < T ? kc + (size_t)p * HD : kf + (size_t)(p - T) * HD;
        const uint16_t* vs = p < T ? vc + (size_t)p * HD : vf + (size_t)(p - T) * HD;
        kv = __uint_as_float((uint32_t)ks[e] << 16);
        vv = __uint_as_float((uint32_t)vs[e] << 16);
      }
      k_s[pp][e / H2][e % H2] = kv;
      v_s[pp][e / H2][e % H2] = vv;
    }
    __syncthreads();
    const int np = min(KB, k1 - p0);
    for (int pp = 0; pp < np; ++pp) {
      float s = 0.f;
#pragma unroll
      for (int e = 0; e < H2; ++e) s = fmaf(q[e], k_s[pp][half][e], s);
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s *= scale;
      if (valid && p0 + pp <= vis) {
        const float mn = fmaxf(mrun, s);
        const float corr = expf(mrun - mn), pe = expf(s - mn);
        lrun = lrun * corr + pe;
#pragma unroll
        for (int e = 0; e < H2; ++e) acc[e] = fmaf(pe, v_s[pp][half][e], acc[e] * corr);
        mrun = mn;
      }
    }
  }
  // partial (M, L, A) for this split
  const int RB = gridDim.y / a.KVr;
  float* part = a.part + ((((size_t)bz * a.KVr + kvh) * RB + rb) * S + split) * 64 * (HD + 2);
  float* pr = part + (tid >> 1) * (HD + 2);
  if (half == 0) {
    pr[0] = mrun;
    pr[1] = lrun;
  }
#pragma unroll
  for (int e = 0; e < H2; ++e) pr[2 + half * H2 + e] = acc[e];
  if (!arrive_last(a.counters + ((size_t)bz * a.KVr + kvh) * RB + rb, S)) return;
  if (!valid) return;
  const float* pb = a.part + (((size_t)bz * a.KVr + kvh) * RB + rb) * S * 64 * (HD + 2) + (tid >> 1) * (HD + 2);
  float M = -INFINITY;
  for (int sp = 0; sp < S; ++sp) M = fmaxf(M, __ldcg(pb + (size_t)sp * 64 * (HD + 2)));
  float L = 0.f;
  float o[H2];
#pragma unroll
  for (int e = 0; e < H2; ++e) o[e] = 0.f;
  for (int sp = 0; sp < S; ++sp) {
    const float* ps = pb + (size_t)sp * 64 * (HD + 2);
    const float Ms = __ldcg(ps);
    if (Ms == -INFINITY) continue;
    const float f = expf(Ms - M);
    L += __ldcg(ps + 1) * f;
#pragma unroll
    for (int e = 0; e < H2; ++e) o[e] += __ldcg(ps + 2 + half * H2 + e) * f;
  }
  const size_t off = (size_t)(bz * rows + i) * a.Hr * HD + (kvh * G + g) * HD + half * H2;
#pragma unroll
  for (int e = 0; e < H2; ++e) {
    const float v = L > 0.f ? o[e] / L : 0.f;
    const uint16_t hi = f2bf_bits(v);
    a.out_hi[off + e] = hi;
    a.out_lo[off + e] = f2bf_bits(v - __uint_as_float((uint32_t)hi << 16));
  }
}

// ===================================================================== acceptance
__global__ void __launch_bounds__(256) accept_stats_kernel(AcceptStatsArgs a) {
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
  const int nvec = n * a.hd / 8;
  for (int e = threadIdx.x; e < nvec; e += 128) {
    kd[e] = ks[e];
    vd[e] = vs[e];
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

cudaError_t norm_rows(const NormRowsArgs& a, int M, cudaStream_t st) {
  norm_rows_kernel<<<M, 256, 0, st>>>(a);
  return cudaGetLastError();
}
cudaError_t rope_store(const RopeStoreArgs& a, int M, cudaStream_t st) {
  rope_store_kernel<<<M, 128, 0, st>>>(a);
  return cudaGetLastError();
}
cudaError_t attn_rows(const AttnRowsArgs& a, int nseq, int hd, int splits, int row_blocks, cudaStream_t st) {
  dim3 grid(splits, a.KVr * row_blocks, nseq);
  const float scale = 1.0f / sqrtf((float)hd);
  if (hd == 128) attn_rows_kernel<128><<<grid, 128, 0, st>>>(a, scale);
  else if (hd == 64) attn_rows_kernel<64><<<grid, 128, 0, st>>>(a, scale);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}
cudaError_t accept_stats(const AcceptStatsArgs& a, int splits, cudaStream_t st) {
  accept_stats_kernel<<<dim3(a.M, splits), 256, 0, st>>>(a);
  return cudaGetLastError();
}
cudaError_t accept_finalize(const AcceptFinalArgs& a, int B, cudaStream_t st) {
  accept_finalize_kernel<<<B, 64, 0, st>>>(a);
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
