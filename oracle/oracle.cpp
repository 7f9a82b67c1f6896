// oracle.cpp — CPU ORACLE for the Sirius decode hot path.  TEST INFRASTRUCTURE ONLY.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
// legs may load this library.  It shares no code with the CUDA path
// (paper_2409_03856_b200/): no headers, no helpers, no constants.  Its inputs come from
// synth/ (seeded generators) only.
//
// What it computes: one Llama-style decoder row in fp64 with plain loops, following
//   * the Llama decoder the paper sparsifies (§2.1; §5.1),
//   * CATS / FSparse (§2.1; PAPER.md:121 footnote; §3.2):
//     the gate is dense, a = SiLU(x·W_gate) is thresholded per layer, |a| >= t_l, and only
//     the active columns of W_up / rows of W_down are used ("Up and Down linear layers only"),
//   * CSparse / Griffin (§2.1): a per-prompt neuron set fixed for the whole
//     generation, the MLP restricted to it (plan argument of oracle_forward_row / oracle_mlp),
//   * the shared KV cache of Algorithm 1 (PAPER.md:242 Require; "Enables Full to
//     directly rewrites KV Cache"; §4.2): a row is written at its position either
//     into the cache (sparse/dense decode, prefill) or into a staging area (full-model verify of a
//     kernel, whose K/V later overwrite the cache rows — kv_rewrite).
// The Sirius loop itself (Algorithm 1) is oracle/sirius_oracle.py.
//
// Numeric contract (reading D15, north_star "bf16 weights with fp32 accumulation"):
// weights are bf16; the KV cache stores K (after RoPE) and V rounded to bf16 (round-to-nearest-
// even, directly from the fp64 value) — the static bf16 KV cache of PAPER.md:496.  Every other
// activation (residual stream, RMSNorm outputs, q, attention output, g, a, u, m, scores, softmax,
// logits) is kept at full precision (fp64 here).  With round_kv = 0 nothing is rounded (the mode
// used to pin this file against HuggingFace LlamaForCausalLM in fp64).
//
// Each function below is one step of the definition; no blocking, fusion or reordering beyond
// the definition.  std::thread only splits independent output rows.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace {

struct Oracle {
  // shape
  int vocab, d, L, H, KV, hd, ffn, max_seq, max_gamma, threads, round_kv;
  double theta, eps;
  // weights (host, bf16 bit patterns, borrowed)
  const uint16_t *embed, *final_norm, *lm_head;
  std::vector<const uint16_t*> attn_norm, wqkv, wo, ffn_norm, wgate, wup, wdown;
  // shared KV cache C and verify staging; values are exactly the (bf16-rounded) stored K/V
  std::vector<double> kc, vc;  // [L][max_seq][KV][hd]
  std::vector<double> ks, vs;  // [L][max_gamma][KV][hd]
  // RoPE table: fp64 computation rounded to fp32 (reading D16)
  std::vector<float> rcos, rsin;  // [max_seq][hd/2]
};

inline double bf16_value(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return (double)f;
}

// Round-to-nearest-even to bf16 precision (8 significant bits), directly from fp64.
inline double round_bf16(double x) {
  if (x == 0.0 || !std::isfinite(x)) return x;
  int e;
  double m = std::frexp(x, &e);                       // x = m * 2^e, 0.5 <= |m| < 1
  return std::ldexp(std::nearbyint(std::ldexp(m, 8)), e - 8);  // nearbyint: default mode = RNE
}

inline double kv_store(const Oracle* o, double x) { return o->round_kv ? round_bf16(x) : x; }

template <class F>
void parallel_rows(int n, int threads, F fn) {
  if (threads <= 1 || n < 64) {
    for (int i = 0; i < n; ++i) fn(i);
    return;
  }
  std::vector<std::thread> ts;
  for (int t = 0; t < threads; ++t) {
    int b = (int)((long long)n * t / threads), e = (int)((long long)n * (t + 1) / threads);
    ts.emplace_back([=] { for (int i = b; i < e; ++i) fn(i); });
  }
  for (auto& th : ts) th.join();
}

// y[r] = sum_k W[r][k] * x[k] for rows r of a row-major bf16 matrix [n][k].
void matvec(const Oracle* o, const uint16_t* W, int n, int k, const double* x, double* y) {
  parallel_rows(n, o->threads, [&](int r) {
    const uint16_t* w = W + (size_t)r * k;
    double s = 0.0;
    for (int c = 0; c < k; ++c) s += bf16_value(w[c]) * x[c];
    y[r] = s;
  });
}

// RMSNorm: h = x / sqrt(mean(x^2) + eps) * w.
void rmsnorm(const Oracle* o, const double* x, const uint16_t* w, double* h) {
  double ss = 0.0;
  for (int k = 0; k < o->d; ++k) ss += x[k] * x[k];
  double r = 1.0 / std::sqrt(ss / o->d + o->eps);
  for (int k = 0; k < o->d; ++k) h[k] = x[k] * r * bf16_value(w[k]);
}

// RoPE, rotate-half convention: pairs (i, i + hd/2); angle = pos * theta^(-2i/hd).
void rope(const Oracle* o, double* v, int pos) {
  int half = o->hd / 2;
  for (int i = 0; i < half; ++i) {
    double c = o->rcos[(size_t)pos * half + i], s = o->rsin[(size_t)pos * half + i];
    double a = v[i], b = v[i + half];
    v[i] = a * c - b * s;
    v[i + half] = b * c + a * s;
  }
}

size_t kv_index(const Oracle* o, int l, int slot, int nslots, int kvh) {
  return (((size_t)l * nslots + slot) * o->KV + kvh) * o->hd;
}

// One decoder layer's attention block for a row at position pos.
// Visible keys: if stage_row < 0, cache slots [0, pos] (the row's own K/V were just written to
// slot pos); else cache slots [0, pos - stage_row) followed by staging rows [0, stage_row].
// Tree rows (tree_vis != 0): cache slots [0, n_cache) followed by
// the staging rows whose bit is set in tree_vis (the row's ancestor chain and itself), in index order.
// kv_only: stop after the row's K/V are stored (nothing downstream of them is wanted).
void attention_block(Oracle* o, int l, double* x, int pos, int stage_row, bool kv_only = false,
                     uint64_t tree_vis = 0, int tree_n_cache = 0) {
  const int d = o->d, H = o->H, KV = o->KV, hd = o->hd, rows = (H + 2 * KV) * hd;
  std::vector<double> h(d), qkv(rows), attn(H * hd), y(d);
  rmsnorm(o, x, o->attn_norm[l], h.data());
  matvec(o, o->wqkv[l], rows, d, h.data(), qkv.data());
  double* q = qkv.data();
  double* k = q + H * hd;
  double* v = k + KV * hd;
  for (int hh = 0; hh < H; ++hh) rope(o, q + hh * hd, pos);
  for (int kh = 0; kh < KV; ++kh) rope(o, k + kh * hd, pos);
  for (int i = H * hd; i < rows; ++i) qkv[i] = kv_store(o, qkv[i]);  // K (after RoPE), V as stored in the bf16 cache

  // store this row's K/V
  for (int kh = 0; kh < KV; ++kh)
    for (int i = 0; i < hd; ++i) {
      if (stage_row < 0) {
        o->kc[kv_index(o, l, pos, o->max_seq, kh) + i] = k[kh * hd + i];
        o->vc[kv_index(o, l, pos, o->max_seq, kh) + i] = v[kh * hd + i];
      } else {
        o->ks[kv_index(o, l, stage_row, o->max_gamma, kh) + i] = k[kh * hd + i];
        o->vs[kv_index(o, l, stage_row, o->max_gamma, kh) + i] = v[kh * hd + i];
      }
    }
  if (kv_only) return;
  int n_cache = stage_row < 0 ? pos + 1 : pos - stage_row;
  std::vector<int> srows;  // visible staging rows, ascending
  if (tree_vis) {
    n_cache = tree_n_cache;
    for (int r = 0; r < 64; ++r)
      if ((tree_vis >> r) & 1ull) srows.push_back(r);
  } else if (stage_row >= 0) {
    for (int r = 0; r <= stage_row; ++r) srows.push_back(r);
  }
  const int n_stage = (int)srows.size();
  const int n_vis = n_cache + n_stage;
  const double scale = 1.0 / std::sqrt((double)hd);
  std::vector<double> s(n_vis);
  for (int hh = 0; hh < H; ++hh) {
    const int kh = hh / (H / KV);  // GQA: kv head = q head // (H/KV)
    const double* qh = q + hh * hd;
    auto key = [&](int p) -> const double* {
      return p < n_cache ? &o->kc[kv_index(o, l, p, o->max_seq, kh)]
                         : &o->ks[kv_index(o, l, srows[p - n_cache], o->max_gamma, kh)];
    };
    auto val = [&](int p) -> const double* {
      return p < n_cache ? &o->vc[kv_index(o, l, p, o->max_seq, kh)]
                         : &o->vs[kv_index(o, l, srows[p - n_cache], o->max_gamma, kh)];
    };
    double mx = -INFINITY;
    for (int p = 0; p < n_vis; ++p) {
      const double* kp = key(p);
      double acc = 0.0;
      for (int i = 0; i < hd; ++i) acc += qh[i] * kp[i];
      s[p] = acc * scale;
      mx = std::max(mx, s[p]);
    }
    double den = 0.0;
    for (int p = 0; p < n_vis; ++p) den += std::exp(s[p] - mx);
    for (int p = 0; p < n_vis; ++p) s[p] = std::exp(s[p] - mx) / den;  // softmax probabilities
    for (int i = 0; i < hd; ++i) {
      double acc = 0.0;
      for (int p = 0; p < n_vis; ++p) acc += s[p] * val(p)[i];
      attn[hh * hd + i] = acc;
    }
  }
  matvec(o, o->wo[l], d, H * hd, attn.data(), y.data());
  for (int j = 0; j < d; ++j) x[j] += y[j];
}

// One decoder layer's MLP with CATS thresholding.
//   h2 = RMSNorm(x);  g = h2 . W_gate (dense, always);  a = SiLU(g) = g / (1 + e^-g)
//   active_i  <=>  dense  or  |a_i| >= t_l
//   u_i = h2 . W_up[i]  (active i only);  m_i = a_i * u_i;  x += sum_{active i, ascending} m_i W_down[i]
// CSparse (§2.1: "within the same input prompt, the sparsity pattern is fixed for all
// tokens generated"; Griffin): plan != NULL gives the prompt's fixed neuron set of this
// layer (plan[i] = 1 iff neuron i is kept) and active_i <=> plan[i]; the MLP is then the dense MLP of
// the kept neurons (gate, up and down restricted to them; a_i of the others is computed but unused).
void mlp_block(Oracle* o, int l, double* x, int sparse, double t, double* gate_out, uint8_t* mask_out,
               int* n_active, const uint8_t* plan = nullptr) {
  const int d = o->d, F = o->ffn;
  std::vector<double> h2(d), g(F), a(F), m(F, 0.0);
  std::vector<uint8_t> mask(F);
  rmsnorm(o, x, o->ffn_norm[l], h2.data());
  matvec(o, o->wgate[l], F, d, h2.data(), g.data());
  int cnt = 0;
  for (int i = 0; i < F; ++i) {
    a[i] = g[i] / (1.0 + std::exp(-g[i]));
    mask[i] = plan ? plan[i] : ((!sparse || std::fabs(a[i]) >= t) ? 1 : 0);
    cnt += mask[i];
  }
  if (sparse == 3) {  // top-k FSparse (PAPER.md:121 footnote "topk on the Gate Layer activations"): t is
                      // the keep fraction; the k = round(t * ffn) largest |a|, exact ties to the lower index
    const int k = (int)std::floor(t * F + 0.5);
    std::vector<int> order(F);
    for (int i = 0; i < F; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return std::fabs(a[x]) > std::fabs(a[y]); });
    std::fill(mask.begin(), mask.end(), 0);
    for (int r = 0; r < k; ++r) mask[order[r]] = 1;
    cnt = k;
  }
  const uint16_t* Wu = o->wup[l];
  parallel_rows(F, o->threads, [&](int i) {
    if (!mask[i]) return;
    const uint16_t* w = Wu + (size_t)i * d;
    double u = 0.0;
    for (int k = 0; k < d; ++k) u += bf16_value(w[k]) * h2[k];
    m[i] = a[i] * u;
  });
  // y_j = sum over active i (ascending) of m_i * W_down[i][j]; threads own column blocks and stream
  // the neuron rows (each y_j still sums over i in ascending order).
  const uint16_t* Wd = o->wdown[l];
  std::vector<double> y(d, 0.0);
  const int nblk = (d + 63) / 64;
  parallel_rows(nblk, o->threads, [&](int blk) {
    const int j0 = blk * 64, j1 = std::min(d, j0 + 64);
    for (int i = 0; i < F; ++i)
      if (mask[i])
        for (int j = j0; j < j1; ++j) y[j] += m[i] * bf16_value(Wd[(size_t)i * d + j]);
  });
  for (int j = 0; j < d; ++j) x[j] += y[j];
  if (gate_out)
    for (int i = 0; i < F; ++i) gate_out[i] = a[i];
  if (mask_out) std::memcpy(mask_out, mask.data(), F);
  if (n_active) *n_active = cnt;
}

}  // namespace

extern "C" {

void* oracle_create(int vocab, int d, int L, int H, int KV, int hd, int ffn, double theta, double eps, int max_seq,
                    int max_gamma, int threads, int round_kv) {
  Oracle* o = new Oracle();
  o->vocab = vocab; o->d = d; o->L = L; o->H = H; o->KV = KV; o->hd = hd; o->ffn = ffn;
  o->theta = theta; o->eps = eps; o->max_seq = max_seq; o->max_gamma = max_gamma;
  o->threads = threads; o->round_kv = round_kv;
  o->attn_norm.resize(L); o->wqkv.resize(L); o->wo.resize(L); o->ffn_norm.resize(L);
  o->wgate.resize(L); o->wup.resize(L); o->wdown.resize(L);
  o->kc.assign((size_t)L * max_seq * KV * hd, 0.0);
  o->vc.assign((size_t)L * max_seq * KV * hd, 0.0);
  o->ks.assign((size_t)L * max_gamma * KV * hd, 0.0);
  o->vs.assign((size_t)L * max_gamma * KV * hd, 0.0);
  const int half = hd / 2;
  o->rcos.resize((size_t)max_seq * half);
  o->rsin.resize((size_t)max_seq * half);
  for (int p = 0; p < max_seq; ++p)
    for (int i = 0; i < half; ++i) {
      double inv_freq = std::pow(theta, -2.0 * i / hd);
      double ang = (double)p * inv_freq;
      o->rcos[(size_t)p * half + i] = (float)std::cos(ang);
      o->rsin[(size_t)p * half + i] = (float)std::sin(ang);
    }
  return o;
}

void oracle_destroy(void* h) { delete (Oracle*)h; }

void oracle_set_global(void* h, const uint16_t* embed, const uint16_t* final_norm, const uint16_t* lm_head) {
  Oracle* o = (Oracle*)h;
  o->embed = embed; o->final_norm = final_norm; o->lm_head = lm_head;
}

void oracle_set_layer(void* h, int l, const uint16_t* attn_norm, const uint16_t* wqkv, const uint16_t* wo,
                      const uint16_t* ffn_norm, const uint16_t* wgate, const uint16_t* wup, const uint16_t* wdown) {
  Oracle* o = (Oracle*)h;
  o->attn_norm[l] = attn_norm; o->wqkv[l] = wqkv; o->wo[l] = wo; o->ffn_norm[l] = ffn_norm;
  o->wgate[l] = wgate; o->wup[l] = wup; o->wdown[l] = wdown;
}

// Full row forward.  sparse: 0 = dense model M_F, 1 = CATS sparse model M_S (thresholds[L], fp32),
// 2 = CSparse model M_S with the fixed neuron plan[L*ffn] (1 = kept), 3 = top-k FSparse model M_S
// (thresholds[L] = keep fraction per layer).
// stage_row < 0: write K/V to cache slot pos; >= 0: write to staging row stage_row (verify).
// logits: [vocab] fp64 or NULL.  gate_out: [L*ffn] a = SiLU(g) or NULL.  mask_out: [L*ffn] or NULL.
// n_active: [L] or NULL.  x_out: [d] final residual (pre final-norm) or NULL.
// tree_vis != 0 (tree rows, stage_row >= 0): the row sees cache [0, tree_n_cache) and the staging rows of
// its bits (ancestor chain + itself) instead of staging [0, stage_row].
void oracle_forward_row(void* h, int tok, int pos, int sparse, const float* thresholds, int stage_row,
                        double* logits, double* gate_out, uint8_t* mask_out, int* n_active, double* x_out,
                        const uint8_t* plan, uint64_t tree_vis, int tree_n_cache) {
  Oracle* o = (Oracle*)h;
  const int d = o->d;
  std::vector<double> x(d), hf(d);
  for (int k = 0; k < d; ++k) x[k] = bf16_value(o->embed[(size_t)tok * d + k]);  // x = E[tok]
  for (int l = 0; l < o->L; ++l) {
    attention_block(o, l, x.data(), pos, stage_row, false, tree_vis, tree_n_cache);
    mlp_block(o, l, x.data(), sparse, (sparse == 1 || sparse == 3) ? (double)thresholds[l] : 0.0,
              gate_out ? gate_out + (size_t)l * o->ffn : nullptr, mask_out ? mask_out + (size_t)l * o->ffn : nullptr,
              n_active ? n_active + l : nullptr, sparse == 2 ? plan + (size_t)l * o->ffn : nullptr);
  }
  if (x_out) std::memcpy(x_out, x.data(), sizeof(double) * d);
  if (logits) {
    rmsnorm(o, x.data(), o->final_norm, hf.data());
    matvec(o, o->lm_head, o->vocab, d, hf.data(), logits);
  }
}

// Prompt row whose only wanted output is its K/V cache rows (every prefill row but the last):
// the full row for layers [0, L-1), then the last layer's K/V store.  The stored values are those
// oracle_forward_row writes for the same row (the skipped work — last-layer attention, MLP and
// head — does not feed them).
void oracle_prefill_kv_row(void* h, int tok, int pos) {
  Oracle* o = (Oracle*)h;
  const int d = o->d;
  std::vector<double> x(d);
  for (int k = 0; k < d; ++k) x[k] = bf16_value(o->embed[(size_t)tok * d + k]);
  for (int l = 0; l + 1 < o->L; ++l) {
    attention_block(o, l, x.data(), pos, -1);
    mlp_block(o, l, x.data(), 0, 0.0, nullptr, nullptr, nullptr);
  }
  attention_block(o, o->L - 1, x.data(), pos, -1, true);
}

// Layer-isolated MLP (kernel-level parity at full shapes): x[d] in/out.  sparse 2: plan[ffn] (CSparse).
void oracle_mlp(void* h, int l, double* x, int sparse, float threshold, double* gate_out, uint8_t* mask_out,
                int* n_active, const uint8_t* plan) {
  mlp_block((Oracle*)h, l, x, sparse, (sparse == 1 || sparse == 3) ? (double)threshold : 0.0, gate_out, mask_out,
            n_active,
            sparse == 2 ? plan : nullptr);
}

// KV rewrite (Algorithm 1, §4.2): staging rows [0, n) -> cache slots [T, T+n).
void oracle_kv_rewrite(void* h, int T, int n) {
  Oracle* o = (Oracle*)h;
  for (int l = 0; l < o->L; ++l)
    for (int r = 0; r < n; ++r)
      for (int kh = 0; kh < o->KV; ++kh)
        for (int i = 0; i < o->hd; ++i) {
          o->kc[kv_index(o, l, T + r, o->max_seq, kh) + i] = o->ks[kv_index(o, l, r, o->max_gamma, kh) + i];
          o->vc[kv_index(o, l, T + r, o->max_seq, kh) + i] = o->vs[kv_index(o, l, r, o->max_gamma, kh) + i];
        }
}

// Tree commit ("select the one that reaches the longest advance length", with the KV rewrite
// of P:257): staging rows rows[0..n) -> cache slots [T, T+n).
void oracle_kv_rewrite_rows(void* h, int T, int n, const int* rows) {
  Oracle* o = (Oracle*)h;
  for (int l = 0; l < o->L; ++l)
    for (int r = 0; r < n; ++r)
      for (int kh = 0; kh < o->KV; ++kh)
        for (int i = 0; i < o->hd; ++i) {
          o->kc[kv_index(o, l, T + r, o->max_seq, kh) + i] = o->ks[kv_index(o, l, rows[r], o->max_gamma, kh) + i];
          o->vc[kv_index(o, l, T + r, o->max_seq, kh) + i] = o->vs[kv_index(o, l, rows[r], o->max_gamma, kh) + i];
        }
}

// Read back cache rows [0, n) of layer l: k/v out [n][KV][hd] (tests: rewrite equivalence).
void oracle_read_cache(void* h, int l, int n, double* k, double* v) {
  Oracle* o = (Oracle*)h;
  size_t per = (size_t)o->KV * o->hd;
  std::memcpy(k, &o->kc[kv_index(o, l, 0, o->max_seq, 0)], sizeof(double) * per * n);
  std::memcpy(v, &o->vc[kv_index(o, l, 0, o->max_seq, 0)], sizeof(double) * per * n);
}

double oracle_round_bf16(double x) { return round_bf16(x); }

}  // extern "C"
