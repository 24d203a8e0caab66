/*
 * oracle.c — CPU fp32 restatement of the Glinthawk two-tier decode step.
 *
 * TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs as the checker; never part of the product path.
 *
 * Parity status: the reference repository (/root/reference/proj, "tierplan") contains no
 * decode arithmetic, so there is no upstream decode code to pin against.
 * This file restates the paper's operations and is pinned (a) on the reference's accounting
 * goldens through oracle/ref_shim.cpp + the compiled reference sources, (b) on Hugging Face
 * transformers' LlamaForCausalLM (transformers 5.5.0, fp32) holding the same weights
 * (oracle/hf_llama.py, tests/test_oracle_hf.py, tests/golden/hf_llama_c1.npz: the 512 C1 greedy
 * tokens are identical), and (c) on committed golden vectors (tests/golden/).
 *
 * What it restates (P = /root/reference/PAPER.md):
 *   F1 (Table 8 rows P:875-877): RMSNorm -> x*[W_q|W_k|W_v] -> RoPE            or_pre
 *   F2 (rows P:889-891): append (k,v) at pos, softmax(q K^T / sqrt(d_h)) V     or_attend
 *       MHA with GQA support
 *   F3 (rows P:879-883): x' W_o + x -> RMSNorm -> SwiGLU(W_1, W_3) -> W_2 + h   or_post
 *   classifier: RMSNorm -> x W_cls^T -> greedy argmax (lowest index on ties)         or_classify
 *   numerics: "Kernel computations run at FP32, while kernel results are stored in the
 *   model's native data type" -> every stage output above is rounded to the storage dtype.
 *   shapes: TransformerSpec (proj/include/tierplan/model.hpp:14-28); KV bytes per prompt
 *   2*dtype*N*S*D_kv (proj/src/model.cpp:40-46); message layouts = PayloadModel byte counts
 *   (proj/src/netmodel.cpp:18-24): fwd [x|q|k|v], bwd [x|attn].
 *   Llama-2 pieces the paper leaves implicit: RMSNorm eps, RoPE on adjacent
 *   pairs (2i, 2i+1) with theta^(-2i/d_h), SiLU-gated FFN, 1/sqrt(d_h) scale.
 *
 * Synthetic weights: value(seed, tensor, idx) = Irwin-Hall(4) integer sum, centred, times
 * k = sqrt(3)*std/2^24 (one rounding).  Compiled with -ffp-contract=off so the restatement is
 * bit-identical to the device generator (paper_2501_11779_b200/csrc/common.cuh).
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  uint64_t n_layers, d_model, d_kv, d_hidden, n_heads, n_kv_heads, max_seq_len, dtype_bytes, vocab_size;
  float rope_theta, norm_eps;
} or_spec;

/* ------------------------------------------------------------------ storage dtype */
static inline float bf2f(uint16_t b) {
  union { uint32_t u; float f; } v;
  v.u = (uint32_t)b << 16;
  return v.f;
}
static inline uint16_t f2bf(float f) { /* round to nearest even, finite inputs */
  union { uint32_t u; float f; } v;
  v.f = f;
  uint32_t u = v.u;
  if ((u & 0x7f800000u) == 0x7f800000u) return (uint16_t)((u >> 16) | ((u & 0xffff) ? 0x40 : 0));
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
/* element i of a native-dtype array */
static inline float ld(const void* p, int db, size_t i) {
  return db == 4 ? ((const float*)p)[i] : bf2f(((const uint16_t*)p)[i]);
}
static inline void st(void* p, int db, size_t i, float v) {
  if (db == 4) ((float*)p)[i] = v;
  else ((uint16_t*)p)[i] = f2bf(v);
}
/* round a float to what the storage dtype can hold */
static inline float rnd(int db, float v) { return db == 4 ? v : bf2f(f2bf(v)); }

/* ------------------------------------------------------------------ synthetic generator */
static inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static inline uint64_t tensor_base(uint64_t seed, uint64_t tensor) {
  return mix64(seed ^ (tensor * 0xD1B54A32D192ED03ull));
}
static inline float randn_scaled(uint64_t base, uint64_t idx, float k) {
  uint64_t h0 = mix64(base + 2 * idx), h1 = mix64(base + 2 * idx + 1);
  int64_t s = (int64_t)(h0 >> 40) + (int64_t)((h0 >> 16) & 0xFFFFFF) + (int64_t)(h1 >> 40) +
              (int64_t)((h1 >> 16) & 0xFFFFFF);
  int64_t c = s - (int64_t)2 * (1 << 24);
  return (float)c * k;
}
static float ih_k(double std_) { return (float)(1.7320508075688772 * std_ / 16777216.0); }
enum { TID_EMBED = 1, TID_CLS = 2 };
static uint64_t tid_layer(uint64_t l, uint64_t w) { return 64 + l * 16 + w; }
enum { WQ = 0, WK = 1, WV = 2, WO = 3, W1 = 4, W3 = 5, W2 = 6 };
static uint64_t tid_kv(uint64_t l, uint64_t slot, uint64_t kv) { return (1ull << 40) | (l << 24) | (slot << 1) | kv; }

/* ------------------------------------------------------------------ model */
typedef struct {
  void *wq, *wk, *wv, *wo, *w1, *w3, *w2; /* [out][in], native dtype */
} or_layer;

typedef struct {
  or_spec s;
  int D, Dkv, Dh, H, Hkv, S, V, dh, db;
  uint32_t l0, l1;
  or_layer* layers;
  void *embed, *cls;
  float* rope; /* [S][dh/2][2] */
} or_model;

static void spec_derive(const or_spec* s, int* D, int* Dkv, int* Dh, int* H, int* Hkv, int* S, int* V, int* dh, int* db) {
  *D = (int)s->d_model; *Dkv = (int)s->d_kv; *Dh = (int)s->d_hidden; *H = (int)s->n_heads;
  *Hkv = (int)s->n_kv_heads; *S = (int)s->max_seq_len; *V = (int)s->vocab_size; *dh = *D / *H;
  *db = (int)s->dtype_bytes;
}

static void* gen_matrix(int db, uint64_t seed, uint64_t tid, size_t rows, size_t cols, double std_) {
  const size_t n = rows * cols;
  void* p = malloc(n * (size_t)db);
  const uint64_t base = tensor_base(seed, tid);
  const float k = ih_k(std_);
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < n; ++i) st(p, db, i, randn_scaled(base, i, k));
  return p;
}

or_model* or_model_create(const or_spec* s, uint64_t seed, uint32_t l0, uint32_t l1) {
  or_model* m = (or_model*)calloc(1, sizeof(or_model));
  m->s = *s;
  spec_derive(s, &m->D, &m->Dkv, &m->Dh, &m->H, &m->Hkv, &m->S, &m->V, &m->dh, &m->db);
  m->l0 = l0; m->l1 = l1;
  m->layers = (or_layer*)calloc(l1 - l0, sizeof(or_layer));
  const int D = m->D, Dkv = m->Dkv, Dh = m->Dh, db = m->db;
  const double sD = 1.0 / sqrt((double)D), sH = 1.0 / sqrt((double)Dh);
  for (uint32_t l = l0; l < l1; ++l) {
    or_layer* L = &m->layers[l - l0];
    L->wq = gen_matrix(db, seed, tid_layer(l, WQ), D, D, sD);
    L->wk = gen_matrix(db, seed, tid_layer(l, WK), Dkv, D, sD);
    L->wv = gen_matrix(db, seed, tid_layer(l, WV), Dkv, D, sD);
    L->wo = gen_matrix(db, seed, tid_layer(l, WO), D, D, sD);
    L->w1 = gen_matrix(db, seed, tid_layer(l, W1), Dh, D, sD);
    L->w3 = gen_matrix(db, seed, tid_layer(l, W3), Dh, D, sD);
    L->w2 = gen_matrix(db, seed, tid_layer(l, W2), D, Dh, sH);
  }
  if (l0 == 0) m->embed = gen_matrix(db, seed, TID_EMBED, m->V, D, 1.0);
  if (l1 == s->n_layers) m->cls = gen_matrix(db, seed, TID_CLS, m->V, D, sD);
  const int half = m->dh / 2;
  m->rope = (float*)malloc(sizeof(float) * 2 * (size_t)m->S * half);
  for (int p = 0; p < m->S; ++p)
    for (int i = 0; i < half; ++i) {
      const double freq = pow((double)s->rope_theta, -2.0 * i / (double)m->dh);
      const double a = (double)p * freq;
      m->rope[((size_t)p * half + i) * 2] = (float)cos(a);
      m->rope[((size_t)p * half + i) * 2 + 1] = (float)sin(a);
    }
  return m;
}

void or_model_destroy(or_model* m) {
  if (!m) return;
  for (uint32_t l = m->l0; l < m->l1; ++l) {
    or_layer* L = &m->layers[l - m->l0];
    free(L->wq); free(L->wk); free(L->wv); free(L->wo); free(L->w1); free(L->w3); free(L->w2);
  }
  free(m->layers); free(m->embed); free(m->cls); free(m->rope); free(m);
}

/* raw weight element access for tests: which = 0..6 (q,k,v,o,1,3,2), 7 = embed, 8 = cls */
float or_model_weight(const or_model* m, uint32_t layer, int which, uint64_t idx) {
  const void* p = NULL;
  if (which == 7) p = m->embed;
  else if (which == 8) p = m->cls;
  else {
    const or_layer* L = &m->layers[layer - m->l0];
    const void* t[7] = {L->wq, L->wk, L->wv, L->wo, L->w1, L->w3, L->w2};
    p = t[which];
  }
  return p ? ld(p, m->db, idx) : NAN;
}

/* ------------------------------------------------------------------ kernels (fp32 compute) */
/* Summation order (test calibration only).  0 = the restatement's order.  1 = every fp32 reduction
 * (GEMM dot products, attention scores, the softmax denominator and P.V, RMSNorm sums of squares)
 * runs in the reverse order: an equally valid P:514 implementation whose stored bf16 values differ
 * from order 0 only where a differently ordered fp32 sum rounds across a bf16 boundary.  Order 0 vs
 * order 1 measures the bf16-storage noise floor the GPU's (split-K / tensor-core) order is held to. */
static int g_order = 0;
void or_set_sum_order(int order) { g_order = order; }

/* Y[b][n] = sum_k X[b][k] W[n][k]; X fp32 [B][K] (already storage-rounded), W native dtype */
static void gemm(const float* X, int B, const void* W, int db, int N, int K, float* Y) {
#pragma omp parallel
  {
    float* wrow = (float*)malloc(sizeof(float) * (size_t)K);
#pragma omp for schedule(static)
    for (int n = 0; n < N; ++n) {
      for (int k = 0; k < K; ++k) wrow[k] = ld(W, db, (size_t)n * K + k);
      for (int b = 0; b < B; ++b) {
        const float* x = X + (size_t)b * K;
        float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        float s;
        if (g_order == 0) {
          int k = 0;
          for (; k + 8 <= K; k += 8)
            for (int j = 0; j < 8; ++j) acc[j] += wrow[k + j] * x[k + j];
          s = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
          for (; k < K; ++k) s += wrow[k] * x[k];
        } else {
          int k = K;
          for (; k >= 8; k -= 8)
            for (int j = 0; j < 8; ++j) acc[j] += wrow[k - 1 - j] * x[k - 1 - j];
          s = ((acc[7] + acc[6]) + (acc[5] + acc[4])) + ((acc[3] + acc[2]) + (acc[1] + acc[0]));
          for (; k > 0; --k) s += wrow[k - 1] * x[k - 1];
        }
        Y[(size_t)b * N + n] = s;
      }
    }
    free(wrow);
  }
}

/* y = x * 1/sqrt(mean(x^2)+eps) * g  (g = 1, norms are unit-initialised) */
static void rmsnorm_row(const float* x, int D, float eps, float* y, int db) {
  float ss = 0.f;
  if (g_order == 0)
    for (int i = 0; i < D; ++i) ss += x[i] * x[i];
  else
    for (int i = D - 1; i >= 0; --i) ss += x[i] * x[i];
  const float inv = 1.0f / sqrtf(ss / (float)D + eps);
  for (int i = 0; i < D; ++i) y[i] = rnd(db, x[i] * inv);
}

static float* load_rows(const void* src, int db, int B, int cols, long ld_src, long off) {
  float* out = (float*)malloc(sizeof(float) * (size_t)B * cols);
  for (int b = 0; b < B; ++b)
    for (int i = 0; i < cols; ++i) out[(size_t)b * cols + i] = ld(src, db, (size_t)b * ld_src + off + i);
  return out;
}

int or_embed(const or_model* m, int B, const int32_t* tok, void* x) {
  if (!m->embed) return 2;
  for (int b = 0; b < B; ++b) {
    int t = tok[b] < 0 ? 0 : (tok[b] >= m->V ? m->V - 1 : tok[b]);
    for (int i = 0; i < m->D; ++i) st(x, m->db, (size_t)b * m->D + i, ld(m->embed, m->db, (size_t)t * m->D + i));
  }
  return 0;
}

/* F1: msg_fwd[b] = [x | rope(q) | rope(k) | v] */
int or_pre(const or_model* m, uint32_t layer, int B, const void* x, const int32_t* pos, void* fwd) {
  if (layer < m->l0 || layer >= m->l1) return 2;
  const or_layer* L = &m->layers[layer - m->l0];
  const int D = m->D, Dkv = m->Dkv, db = m->db, dh = m->dh, half = dh / 2;
  const long ldf = 2L * D + 2L * Dkv;
  float* xf = load_rows(x, db, B, D, D, 0);
  float* xn = (float*)malloc(sizeof(float) * (size_t)B * D);
  for (int b = 0; b < B; ++b) rmsnorm_row(xf + (size_t)b * D, D, m->s.norm_eps, xn + (size_t)b * D, db);
  float* q = (float*)malloc(sizeof(float) * (size_t)B * D);
  float* k = (float*)malloc(sizeof(float) * (size_t)B * Dkv);
  float* v = (float*)malloc(sizeof(float) * (size_t)B * Dkv);
  gemm(xn, B, L->wq, db, D, D, q);
  gemm(xn, B, L->wk, db, Dkv, D, k);
  gemm(xn, B, L->wv, db, Dkv, D, v);
  for (int b = 0; b < B; ++b) {
    const float* cs = m->rope + (size_t)pos[b] * half * 2;
    for (int pass = 0; pass < 2; ++pass) {
      float* r = pass == 0 ? q + (size_t)b * D : k + (size_t)b * Dkv;
      const int n = pass == 0 ? D : Dkv;
      for (int i = 0; i < n; i += 2) {
        const int pi = (i % dh) / 2;
        const float c = cs[pi * 2], sn = cs[pi * 2 + 1];
        const float a = r[i], e = r[i + 1];
        r[i] = a * c - e * sn;
        r[i + 1] = a * sn + e * c;
      }
    }
    for (int i = 0; i < D; ++i) st(fwd, db, (size_t)b * ldf + i, xf[(size_t)b * D + i]);
    for (int i = 0; i < D; ++i) st(fwd, db, (size_t)b * ldf + D + i, q[(size_t)b * D + i]);
    for (int i = 0; i < Dkv; ++i) st(fwd, db, (size_t)b * ldf + 2 * D + i, k[(size_t)b * Dkv + i]);
    for (int i = 0; i < Dkv; ++i) st(fwd, db, (size_t)b * ldf + 2 * D + Dkv + i, v[(size_t)b * Dkv + i]);
  }
  free(xf); free(xn); free(q); free(k); free(v);
  return 0;
}

/* ------------------------------------------------------------------ KV context (Tier-2) */
typedef struct {
  or_spec s;
  int D, Dkv, Dh, H, Hkv, S, V, dh, db;
  uint32_t l0, l1, n_slots;
  void* arena; /* [layer][slot][kv][h][S][dh] native dtype (same layout as the device arena) */
} or_kv;

static size_t kv_index(const or_kv* c, uint32_t layer, uint32_t slot, int kv, int h, int p) {
  return (((((size_t)(layer - c->l0) * c->n_slots + slot) * 2 + kv) * c->Hkv + h) * (size_t)c->S + p) * c->dh;
}

or_kv* or_kv_create(const or_spec* s, uint32_t l0, uint32_t l1, uint32_t n_slots) {
  or_kv* c = (or_kv*)calloc(1, sizeof(or_kv));
  c->s = *s;
  spec_derive(s, &c->D, &c->Dkv, &c->Dh, &c->H, &c->Hkv, &c->S, &c->V, &c->dh, &c->db);
  c->l0 = l0; c->l1 = l1; c->n_slots = n_slots;
  const size_t n = (size_t)(l1 - l0) * n_slots * 2 * c->Hkv * (size_t)c->S * c->dh;
  c->arena = calloc(n, (size_t)c->db);
  return c->arena ? c : (free(c), (or_kv*)NULL);
}
void or_kv_destroy(or_kv* c) { if (c) { free(c->arena); free(c); } }

/* same values as the device pre-fill (gh_tier2_fill_synthetic) */
void or_kv_fill_synthetic(or_kv* c, uint64_t seed, uint32_t n_fill, uint32_t npos) {
  const float k = ih_k(1.0);
  for (uint32_t l = c->l0; l < c->l1; ++l)
    for (uint32_t slot = 0; slot < n_fill; ++slot)
      for (int kv = 0; kv < 2; ++kv) {
        const uint64_t base = tensor_base(seed, tid_kv(l, slot, kv));
#pragma omp parallel for schedule(static)
        for (int h = 0; h < c->Hkv; ++h)
          for (uint32_t p = 0; p < npos; ++p)
            for (int d = 0; d < c->dh; ++d) {
              const uint64_t logical = ((uint64_t)h * c->S + p) * c->dh + d;
              st(c->arena, c->db, kv_index(c, l, slot, kv, h, (int)p) + d, randn_scaled(base, logical, k));
            }
      }
}

void or_kv_read(const or_kv* c, uint32_t layer, uint32_t slot, int kv, int h, int n, float* out) {
  for (int p = 0; p < n; ++p)
    for (int d = 0; d < c->dh; ++d) out[(size_t)p * c->dh + d] = ld(c->arena, c->db, kv_index(c, layer, slot, kv, h, p) + d);
}

/* F2: append k,v at pos[b]; attn = softmax(q K^T / sqrt(d_h)) V over positions 0..pos[b] */
int or_attend(or_kv* c, uint32_t layer, int B, const uint32_t* slot, const int32_t* pos, const void* fwd, void* bwd) {
  if (layer < c->l0 || layer >= c->l1) return 2;
  const int D = c->D, Dkv = c->Dkv, db = c->db, dh = c->dh, H = c->H, Hkv = c->Hkv, grp = H / Hkv;
  const long ldf = 2L * D + 2L * Dkv, ldb = 2L * D;
  for (int b = 0; b < B; ++b) {
    if (slot[b] >= c->n_slots || pos[b] < 0 || pos[b] >= c->S) return 3;
    for (int h = 0; h < Hkv; ++h)
      for (int d = 0; d < dh; ++d) {
        const size_t i = kv_index(c, layer, slot[b], 0, h, pos[b]) + d;
        const size_t j = kv_index(c, layer, slot[b], 1, h, pos[b]) + d;
        st(c->arena, db, i, ld(fwd, db, (size_t)b * ldf + 2 * D + h * dh + d));
        st(c->arena, db, j, ld(fwd, db, (size_t)b * ldf + 2 * D + Dkv + h * dh + d));
      }
  }
  const float scale = 1.0f / sqrtf((float)dh);
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int b = 0; b < B; ++b)
    for (int h = 0; h < H; ++h) {
      const int n = pos[b] + 1, kvh = h / grp;
      float* sc = (float*)malloc(sizeof(float) * (size_t)n);
      float q[256], o[256];
      for (int d = 0; d < dh; ++d) { q[d] = ld(fwd, db, (size_t)b * ldf + D + h * dh + d); o[d] = 0.f; }
      float mx = -INFINITY;
      for (int p = 0; p < n; ++p) {
        const size_t kb = kv_index(c, layer, slot[b], 0, kvh, p);
        float s = 0.f;
        if (g_order == 0)
          for (int d = 0; d < dh; ++d) s += q[d] * ld(c->arena, db, kb + d);
        else
          for (int d = dh - 1; d >= 0; --d) s += q[d] * ld(c->arena, db, kb + d);
        sc[p] = s * scale;
        if (sc[p] > mx) mx = sc[p];
      }
      float den = 0.f;
      for (int p = 0; p < n; ++p) sc[p] = expf(sc[p] - mx);
      for (int i = 0; i < n; ++i) {
        const int p = g_order == 0 ? i : n - 1 - i;
        den += sc[p];
        const size_t vb = kv_index(c, layer, slot[b], 1, kvh, p);
        for (int d = 0; d < dh; ++d) o[d] += sc[p] * ld(c->arena, db, vb + d);
      }
      for (int d = 0; d < dh; ++d) st(bwd, db, (size_t)b * ldb + D + h * dh + d, o[d] / den);
      free(sc);
    }
  for (int b = 0; b < B; ++b)
    for (int i = 0; i < D; ++i) st(bwd, db, (size_t)b * ldb + i, ld(fwd, db, (size_t)b * ldf + i));
  return 0;
}

/* F3: h = attn W_o^T + x; x' = h + W_2(silu(W_1 rms(h)) * W_3 rms(h)) */
int or_post(const or_model* m, uint32_t layer, int B, const void* bwd, void* x_next) {
  if (layer < m->l0 || layer >= m->l1) return 2;
  const or_layer* L = &m->layers[layer - m->l0];
  const int D = m->D, Dh = m->Dh, db = m->db;
  const long ldb = 2L * D;
  float* xr = load_rows(bwd, db, B, D, ldb, 0);
  float* at = load_rows(bwd, db, B, D, ldb, D);
  float* h = (float*)malloc(sizeof(float) * (size_t)B * D);
  gemm(at, B, L->wo, db, D, D, h);
  for (size_t i = 0; i < (size_t)B * D; ++i) h[i] = rnd(db, h[i] + xr[i]);
  float* hn = (float*)malloc(sizeof(float) * (size_t)B * D);
  for (int b = 0; b < B; ++b) rmsnorm_row(h + (size_t)b * D, D, m->s.norm_eps, hn + (size_t)b * D, db);
  float* a = (float*)malloc(sizeof(float) * (size_t)B * Dh);
  float* u = (float*)malloc(sizeof(float) * (size_t)B * Dh);
  gemm(hn, B, L->w1, db, Dh, D, a);
  gemm(hn, B, L->w3, db, Dh, D, u);
  for (size_t i = 0; i < (size_t)B * Dh; ++i) a[i] = rnd(db, a[i] / (1.0f + expf(-a[i])) * u[i]);
  float* y = (float*)malloc(sizeof(float) * (size_t)B * D);
  gemm(a, B, L->w2, db, D, Dh, y);
  for (size_t i = 0; i < (size_t)B * D; ++i) st(x_next, db, i, y[i] + h[i]);
  free(xr); free(at); free(h); free(hn); free(a); free(u); free(y);
  return 0;
}

int or_classify(const or_model* m, int B, const void* x, float* logits, int32_t* next) {
  if (!m->cls) return 2;
  const int D = m->D, V = m->V, db = m->db;
  float* xf = load_rows(x, db, B, D, D, 0);
  float* xn = (float*)malloc(sizeof(float) * (size_t)B * D);
  for (int b = 0; b < B; ++b) rmsnorm_row(xf + (size_t)b * D, D, m->s.norm_eps, xn + (size_t)b * D, db);
  float* lg = logits ? logits : (float*)malloc(sizeof(float) * (size_t)B * V);
  gemm(xn, B, m->cls, db, V, D, lg);
  for (int b = 0; b < B; ++b) {
    int best = 0;
    for (int i = 1; i < V; ++i)
      if (lg[(size_t)b * V + i] > lg[(size_t)b * V + best]) best = i;
    next[b] = best;
  }
  if (!logits) free(lg);
  free(xf); free(xn);
  return 0;
}

/* One decode step over layers [m->l0, m->l1) (the model must own embedding and classifier). */
int or_decode_step(const or_model* m, or_kv* c, int B, const int32_t* tok, const int32_t* pos,
                   const uint32_t* slot, int32_t* next, float* logits) {
  const int D = m->D, Dkv = m->Dkv, db = m->db;
  void* x = malloc((size_t)B * D * db);
  void* x2 = malloc((size_t)B * D * db);
  void* fwd = malloc((size_t)B * (2 * D + 2 * Dkv) * db);
  void* bwd = malloc((size_t)B * 2 * D * db);
  int rc = or_embed(m, B, tok, x);
  for (uint32_t l = m->l0; rc == 0 && l < m->l1; ++l) {
    rc = or_pre(m, l, B, x, pos, fwd);
    if (!rc) rc = or_attend(c, l, B, slot, pos, fwd, bwd);
    if (!rc) rc = or_post(m, l, B, bwd, x2);
    void* t = x; x = x2; x2 = t;
  }
  if (!rc) rc = or_classify(m, B, x, logits, next);
  free(x); free(x2); free(fwd); free(bwd);
  return rc;
}

void or_set_threads(int n) { if (n > 0) omp_set_num_threads(n); }
int or_max_threads(void) { return omp_get_max_threads(); }

/* generator check for tests: n values of tensor `tid` at std `std_` */
void or_randn(uint64_t seed, uint64_t tid, uint64_t start, uint64_t n, double std_, float* out) {
  const uint64_t base = tensor_base(seed, tid);
  const float k = ih_k(std_);
  for (uint64_t i = 0; i < n; ++i) out[i] = randn_scaled(base, start + i, k);
}
