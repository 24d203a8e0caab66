// runtime.cpp — Tier-1 / Tier-2 stage objects, the NCCL transport and the decode engine
// behind the C ABI (include/gh/gh.h).
//
// Stage taxonomy follows the reference (proj/include/tierplan/profiles.hpp:13):
//   nonattention = gh_tier1_pre (F1) + gh_tier1_post (F3)      on the weight-holding GPU
//   attention    = gh_tier2_attend (F2)                         on the KV-holding GPU
//   classifier   = gh_tier1_classify
// Messages between the stages use the PayloadModel byte layout (netmodel.cpp:18-24).
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "params.hpp"
#include "common.cuh"
#include "gemm_tc.cuh"
#include "gh/gh.h"
#include "internal.hpp"
#include "kernels.hpp"
#include "sched.hpp"

namespace gh {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

// ---------------------------------------------------------------- derived shape
struct Shape {
  gh_model_spec s{};
  int N = 0, D = 0, Dkv = 0, Dh = 0, H = 0, Hkv = 0, S = 0, V = 0, dh = 0, db = 0;
  static gh_status from(const gh_model_spec* spec, Shape* out) {
    GH_TRY(gh_spec_validate(spec));
    Shape x;
    x.s = *spec;
    x.N = (int)spec->n_layers; x.D = (int)spec->d_model; x.Dkv = (int)spec->d_kv;
    x.Dh = (int)spec->d_hidden; x.H = (int)spec->n_heads; x.Hkv = (int)spec->n_kv_heads;
    x.S = (int)spec->max_seq_len; x.V = (int)spec->vocab_size; x.db = (int)spec->dtype_bytes;
    x.dh = x.D / x.H;
    if (x.db != 2 && x.db != 4) return fail(GH_EUNSUPPORTED, "kernels implement dtype_bytes 2 (bf16) and 4 (fp32)");
    if (x.Dkv / x.Hkv != x.dh) return fail(GH_EUNSUPPORTED, "query and kv head dims differ (d_model/n_heads != d_kv/n_kv_heads)");
    if (x.H % x.Hkv != 0) return fail(GH_EUNSUPPORTED, "n_heads must be a multiple of n_kv_heads");
    if (!attention_supported(x.db, x.dh)) return fail(GH_EUNSUPPORTED, "head dim must be 48, 64 or 128");
    if (x.dh % 2) return fail(GH_EUNSUPPORTED, "RoPE needs an even head dim");
    if ((x.D * x.db) % 16 || (x.Dkv * x.db) % 16) return fail(GH_EUNSUPPORTED, "rows must be 16-byte multiples");
    *out = x;
    return GH_OK;
  }
  long ld_fwd() const { return 2L * D + 2L * Dkv; }
  long ld_bwd() const { return 2L * D; }
};

struct DevMem {
  void* p = nullptr;
  ~DevMem() { if (p) cudaFree(p); }
};

static gh_status dev_alloc(std::vector<std::unique_ptr<DevMem>>& pool, size_t bytes, void** out) {
  auto m = std::make_unique<DevMem>();
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMalloc(&m->p, bytes);
  if (e != cudaSuccess)
    return fail(e == cudaErrorMemoryAllocation ? GH_EINFEASIBLE : GH_ECUDA,
                "cudaMalloc(" + std::to_string(bytes) + "): " + cudaGetErrorString(e));
  *out = m->p;
  pool.push_back(std::move(m));
  return GH_OK;
}

// cache of tensor maps over activation buffers: key (ptr, rows, cols, ld, box)
struct TmapCache {
  std::map<std::tuple<const void*, uint64_t, uint64_t, uint64_t, uint32_t>, CUtensorMap> m;
  gh_status get(const void* p, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box, CUtensorMap** out) {
    auto key = std::make_tuple(p, rows, cols, ld, box);
    auto it = m.find(key);
    if (it == m.end()) {
      CUtensorMap t;
      cudaError_t e = make_tmap_bf16(&t, p, rows, cols, ld, box);
      if (e != cudaSuccess) return fail(GH_ECUDA, "cuTensorMapEncodeTiled failed (activation)");
      it = m.emplace(key, t).first;
    }
    *out = &it->second;
    return GH_OK;
  }
};

}  // namespace gh

using namespace gh;

// ================================================================== GEMM profiler (diagnostics)
// gh_debug_gemm_profile(1): every Tier-1 GEMM launch of this process is bracketed by CUDA events
// (which serialises it against its neighbours: no PDL overlap), and gh_debug_gemm_profile_dump
// reports the mean time per (N, K, B, all-reduce) shape.  Off by default.
namespace gh {
struct GemmProfiler {
  bool on = false;
  struct Rec { int N, K, B; bool tp; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  std::mutex mu;
  // GH_GEMM_TRACE=NxK: per-CTA timelines of the profiled GEMMs of that shape (gemm_tc.cuh trace
  // stamps), summarised as medians over CTAs and launches
  int trace_n = 0, trace_k = 0;
  std::vector<std::vector<double>> phases;  // per launch: median per phase
  // gh_debug_gemm_profile(2): timeline mode -- no events (PDL overlap kept); every GEMM launch gets
  // its own slice of trace stamps, summarised per launch by the dump (first CTA start, median
  // griddepcontrol.wait return, last CTA exit)
  bool timeline = false;
  unsigned long long* tl_buf = nullptr;
  int tl_cap = 0, tl_next = 0, tl_dev = -1;
  struct TlRec { int N, K, B; bool pair; };
  std::vector<TlRec> tl_recs;
} g_prof;
}  // namespace gh

// ================================================================== Tier-1
// Rows of a GEMM's activation operand delivered by peer copies: flag words [n] that reach
// sequence number v once their copy has landed (GemmShape::xwait; the split's F3 input)
struct PeerWait {
  const unsigned int* f;
  int n;
  unsigned int v;
};

struct gh_tier1 {
  Shape sh;
  int device = 0;
  uint32_t l0 = 0, l1 = 0, max_batch = 0;
  // Tier-1 tensor parallelism: this object holds rank tp_rank's slice of every layer
  // (heads [r H/T, (r+1) H/T) of W_q / W_k / W_v and the matching input columns of W_o; hidden
  // units [r Dh/T, (r+1) Dh/T) of W_1 / W_3 and the matching input columns of W_2), the embedding
  // and classifier whole.  W_o and W_2 are all-reduced inside their GEMM epilogue (tp_allreduce).
  int tp = 1, tp_rank = 0;
  struct TpCtx {
    // receive buffers [tp][slice][row][BN] of {fp32 value, sequence number} (two parities)
    float* buf[2] = {nullptr, nullptr};
    float* peer_buf[2][kMaxTp] = {};     // rank p's receive buffers (p == tp_rank: local)
    unsigned int seq = 0;                // all-reduces issued (identical on every rank)
    bool ready = false;                  // peer mappings in place (engine peer setup)
  } tpc;
  std::vector<std::unique_ptr<DevMem>> mem;
  struct Layer {
    Weight qkv, o, w13, w2;
    CUtensorMap tm_qkv, tm_o, tm_13, tm_2;
    void* attn_norm = nullptr;
    void* ffn_norm = nullptr;
  };
  std::vector<Layer> layers;
  bool has_embed = false, has_cls = false;
  Weight embed, cls;
  CUtensorMap tm_cls;
  void* final_norm = nullptr;
  float2* rope = nullptr;
  void *xn = nullptr, *h = nullptr, *hn = nullptr, *g = nullptr;
  float* ss_h = nullptr;  // per-slice sums of squares of h (fused FFN RMSNorm)
  float2* part = nullptr;
  GemmScratch gsc;
  unsigned long long* trace_buf = nullptr;  // GEMM profiler timelines (diagnostics)
  TmapCache tmaps;
  std::map<std::tuple<int, int, int, bool>, GemmPlan> plans;

  // tp: a GEMM whose epilogue all-reduces across the TP ranks (plan_gemm_tp)
  const GemmPlan& plan(int N, int K, int B, bool tp_reduce = false) {
    auto key = std::make_tuple(N, K, B, tp_reduce);
    auto it = plans.find(key);
    if (it == plans.end()) it = plans.emplace(key, tp_reduce ? plan_gemm_tp(N, K, B) : plan_gemm(N, K, B)).first;
    return it->second;
  }
  // X: [B, K] with row stride ldx
  // `next`: the weight the following Tier-1 kernel streams; its leading bytes are prefetched into
  // L2 during this GEMM's tail (gemm_tc.cuh, GemmShape::pf)
  gh_status gemm(const Weight& W, const CUtensorMap* tmW, const void* X, long ldx, int B,
                 const EpiParams& ep, cudaStream_t st, const Weight* next = nullptr, const PeerWait* pw = nullptr) {
    const GemmPlan& p = plan(W.N, W.K, B, ep.tp_n > 1);
    if (ep.tp_n > 1 && (p.pair || p.BN > 128)) return fail(GH_EINTERNAL, "tp all-reduce needs the split-K plan");
    CUtensorMap* tmX = nullptr;
    if (sh.db == 2) GH_TRY(tmaps.get(X, (uint64_t)B, (uint64_t)W.K, (uint64_t)ldx, (uint32_t)p.x_box_rows(), &tmX));
    GemmProfiler::Rec rec{};
    GemmScratch sc = gsc;
    if (pw) { sc.xwait = pw->f; sc.xwait_n = pw->n; sc.xwait_val = pw->v; }
    const bool traced = g_prof.on && W.N == g_prof.trace_n && W.K == g_prof.trace_k && !p.pair;
    if (g_prof.on) {
      rec = {W.N, W.K, B, ep.tp_n > 1, nullptr, nullptr};
      GH_CUDA(cudaEventCreate(&rec.a));
      GH_CUDA(cudaEventCreate(&rec.b));
      GH_CUDA(cudaEventRecord(rec.a, st));
      if (traced) {
        if (!trace_buf) {
          void* q;
          GH_TRY(dev_alloc(mem, (size_t)kNumSMs * 16 * 8, &q));
          trace_buf = (unsigned long long*)q;
        }
        GH_CUDA(cudaMemsetAsync(trace_buf, 0, (size_t)kNumSMs * 16 * 8, st));
        sc.trace = trace_buf;
      }
    }
    if (g_prof.timeline && g_prof.tl_next < g_prof.tl_cap) {
      std::lock_guard<std::mutex> lk(g_prof.mu);
      sc.trace = g_prof.tl_buf + (size_t)g_prof.tl_next++ * kNumSMs * 16;
      g_prof.tl_recs.push_back({W.N, W.K, B, p.pair});
    }
    GH_CUDA(launch_gemm(W, tmW, X, ldx, tmX, B, p, ep, sc, st, next ? next->ptr : nullptr, prefetch_bytes(next)));
    if (g_prof.on) {
      GH_CUDA(cudaEventRecord(rec.b, st));
      if (traced) {  // phases relative to the earliest CTA start: median over CTAs of the last tile
        std::vector<unsigned long long> h((size_t)kNumSMs * 16);
        GH_CUDA(cudaMemcpyAsync(h.data(), trace_buf, h.size() * 8, cudaMemcpyDeviceToHost, st));
        GH_CUDA(cudaStreamSynchronize(st));
        unsigned long long t0 = ~0ull;
        for (int c = 0; c < kNumSMs; ++c) if (h[c * 16 + 6]) t0 = std::min(t0, h[c * 16]);
        std::vector<double> med(16, 0.0);
        for (int i = 0; i < 16; ++i) {
          std::vector<double> v;
          for (int c = 0; c < kNumSMs; ++c)
            if (h[c * 16 + 6] && h[c * 16 + i]) v.push_back((double)(h[c * 16 + i] - t0) / 1e3);
          if (!v.empty()) { std::nth_element(v.begin(), v.begin() + v.size() / 2, v.end()); med[i] = v[v.size() / 2]; }
        }
        std::lock_guard<std::mutex> lk(g_prof.mu);
        g_prof.phases.push_back(med);
      }
      std::lock_guard<std::mutex> lk(g_prof.mu);
      g_prof.recs.push_back(rec);
    }
    return GH_OK;
  }
  static size_t prefetch_bytes(const Weight* w) {
    static const size_t cap = (size_t)(getenv("GH_PF_MB") ? atof(getenv("GH_PF_MB")) : 16.0) * (1 << 20);
    if (!w || !w->ptr || w->dtype_bytes != 2) return 0;
    return std::min(cap, w->elems() * 2);
  }
};

static EpiParams epi_default() {
  EpiParams e;
  memset(&e, 0, sizeof(e));
  return e;
}

// Tensor-parallel all-reduce parameters of the next reducing GEMM (W_o or W_2) of a TP Tier-1:
// a fresh sequence number, the receive buffers of its parity, the flag words of every rank.
static gh_status epi_tp(gh_tier1* t, int B, EpiParams& ep) {
  if (t->tp <= 1) return GH_OK;
  auto& c = t->tpc;
  if (!c.ready) return fail(GH_EINVAL, "tensor-parallel Tier-1 used before its peers were mapped (engine only)");
  if ((uint32_t)B > t->max_batch) return fail(GH_EINVAL, "B exceeds max_batch");
  const unsigned int seq = ++c.seq;
  ep.tp_n = t->tp;
  ep.tp_rank = t->tp_rank;
  ep.tp_seq = seq;
  for (int p = 0; p < t->tp; ++p) {
    ep.tp_dst[p] = c.peer_buf[seq & 1][p];
  }
  static const int dbg = getenv("GH_TP_DBG") ? atoi(getenv("GH_TP_DBG")) : 0;  // diagnostics (wrong results)
  ep.tp_dbg = dbg;
  return GH_OK;
}

// tm != nullptr: a tcgen05 GEMM operand -> tile-contiguous layout for bf16 (kernels.hpp Weight)
static gh_status init_weight(gh_tier1* t, Weight* w, int N, int K, CUtensorMap* tm, const RowSegs& segs) {
  w->N = N; w->K = K; w->dtype_bytes = t->sh.db;
  w->tiled = tm != nullptr && t->sh.db == 2;
  GH_TRY(dev_alloc(t->mem, w->elems() * t->sh.db, &w->ptr));
  if (w->tiled) {
    const uint64_t rows = (uint64_t)w->n_pad() * w->kb();
    cudaError_t e = make_tmap_bf16(tm, w->ptr, rows, 64, 64, 128);
    if (e != cudaSuccess) return fail(GH_ECUDA, "cuTensorMapEncodeTiled failed (weights)");
  }
  GH_CUDA(launch_init_weight(*w, segs, 0));
  return GH_OK;
}

extern "C" {

int gh_abi_version(void) { return GH_ABI_VERSION; }
const char* gh_last_error(void) { return g_last_error.c_str(); }
const char* gh_status_name(gh_status s) {
  switch (s) {
    case GH_OK: return "GH_OK";
    case GH_EINTERNAL: return "GH_EINTERNAL";
    case GH_EINVAL: return "GH_EINVAL";
    case GH_EINFEASIBLE: return "GH_EINFEASIBLE";
    case GH_ECUDA: return "GH_ECUDA";
    case GH_ENCCL: return "GH_ENCCL";
    case GH_EUNSUPPORTED: return "GH_EUNSUPPORTED";
  }
  return "GH_UNKNOWN";
}
int gh_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) { cudaGetLastError(); return 0; }
  return n;
}
uint64_t gh_kernel_launches(int reset) {
  uint64_t v = launch_counter();
  if (reset) launch_counter() = 0;
  return v;
}

}  // extern "C"

// tp > 1: tensor-parallel slice tp_rank of every layer (gh_tier1::tp); tp = 1: whole layers.
static gh_status tier1_create(const gh_model_spec* spec, int device, uint32_t layer_begin, uint32_t layer_end,
                              uint64_t seed, uint32_t max_batch, int tp, int tp_rank, gh_tier1** out) {
  if (!out) return fail(GH_EINVAL, "out is null");
  *out = nullptr;
  Shape sh;
  GH_TRY(Shape::from(spec, &sh));
  if (layer_begin >= layer_end || layer_end > (uint32_t)sh.N) return fail(GH_EINVAL, "bad layer range");
  if (max_batch == 0) return fail(GH_EINVAL, "max_batch must be >= 1");
  if (sh.V == 0) return fail(GH_EINVAL, "vocab_size required for Tier-1");
  if (tp < 1 || tp > kMaxTp || tp_rank < 0 || tp_rank >= tp) return fail(GH_EINVAL, "bad tensor-parallel rank");
  if (tp > 1) {
    if (sh.db != 2) return fail(GH_EUNSUPPORTED, "tensor parallelism: bf16 storage (tcgen05 path) only");
    if (sh.H % tp || sh.Hkv % tp) return fail(GH_EINVAL, "tensor parallelism: heads and kv heads must divide by tp");
    if ((sh.D / tp) % 64 || (sh.Dh / tp) % 64 || (sh.Dkv / tp) % 64)
      return fail(GH_EUNSUPPORTED, "tensor parallelism: D/tp, D_kv/tp and D_h/tp must be multiples of 64");
    if (max_batch > (uint32_t)kFusedNormMaxBatch) return fail(GH_EUNSUPPORTED, "tensor parallelism: batch <= 1024");
  }
  if (gh_device_count() <= device) return fail(GH_ECUDA, "no CUDA device " + std::to_string(device));
  GH_CUDA(cudaSetDevice(device));
  GH_CUDA(configure_kernels());
  auto t = std::make_unique<gh_tier1>();
  t->sh = sh; t->device = device; t->l0 = layer_begin; t->l1 = layer_end; t->max_batch = max_batch;
  t->tp = tp; t->tp_rank = tp_rank;
  const int D = sh.D, Dkv = sh.Dkv, Dh = sh.Dh, V = sh.V, db = sh.db;
  const int Dt = D / tp, Dkvt = Dkv / tp, Dht = Dh / tp;  // this rank's heads / hidden units
  cudaStream_t st = 0;
  t->layers.resize(layer_end - layer_begin);
  for (uint32_t l = layer_begin; l < layer_end; ++l) {
    auto& L = t->layers[l - layer_begin];
    const double sD = 1.0 / std::sqrt((double)D), sH = 1.0 / std::sqrt((double)Dh);
    {  // rows [q_r | k_r | v_r]
      const uint64_t tq[3] = {tid_layer(l, kWq), tid_layer(l, kWk), tid_layer(l, kWv)};
      const int rq[3] = {Dt, Dkvt, Dkvt};
      const double sq[3] = {sD, sD, sD};
      RowSegs sg = make_segs(seed, 3, tq, rq, sq, false);
      sg.row0[0] = tp_rank * Dt; sg.row0[1] = sg.row0[2] = tp_rank * Dkvt;
      GH_TRY(init_weight(t.get(), &L.qkv, Dt + 2 * Dkvt, D, &L.tm_qkv, sg));
    }
    {  // all D output rows, input columns of this rank's heads
      const uint64_t to = tid_layer(l, kWo); const int ro = D; const double so = sD;
      RowSegs sg = make_segs(seed, 1, &to, &ro, &so, false);
      sg.k0 = tp_rank * Dt; sg.ldk = D;
      GH_TRY(init_weight(t.get(), &L.o, D, Dt, &L.tm_o, sg));
    }
    {  // hidden units [r Dh/T, (r+1) Dh/T), gate / up interleaved
      const uint64_t t13[2] = {tid_layer(l, kW1), tid_layer(l, kW3)};
      const int r13[2] = {Dht, Dht};
      const double s13[2] = {sD, sD};
      RowSegs sg = make_segs(seed, 2, t13, r13, s13, true);
      sg.row0[0] = sg.row0[1] = tp_rank * Dht;
      GH_TRY(init_weight(t.get(), &L.w13, 2 * Dht, D, &L.tm_13, sg));
    }
    {  // all D output rows, input columns of this rank's hidden units
      const uint64_t t2 = tid_layer(l, kW2); const int r2 = D; const double s2 = sH;
      RowSegs sg = make_segs(seed, 1, &t2, &r2, &s2, false);
      sg.k0 = tp_rank * Dht; sg.ldk = Dh;
      GH_TRY(init_weight(t.get(), &L.w2, D, Dht, &L.tm_2, sg));
    }
    GH_TRY(dev_alloc(t->mem, (size_t)D * db, &L.attn_norm));
    GH_TRY(dev_alloc(t->mem, (size_t)D * db, &L.ffn_norm));
    GH_CUDA(launch_fill_const(db, L.attn_norm, D, 1.0f, st));
    GH_CUDA(launch_fill_const(db, L.ffn_norm, D, 1.0f, st));
  }
  t->has_embed = layer_begin == 0;
  t->has_cls = layer_end == (uint32_t)sh.N;
  if (t->has_embed) {
    const uint64_t te = kTidEmbed; const int re = V; const double se = 1.0;
    GH_TRY(init_weight(t.get(), &t->embed, V, D, nullptr, make_segs(seed, 1, &te, &re, &se, false)));
  }
  if (t->has_cls) {
    const uint64_t tc = kTidCls; const int rc = V; const double sc = 1.0 / std::sqrt((double)D);
    GH_TRY(init_weight(t.get(), &t->cls, V, D, &t->tm_cls, make_segs(seed, 1, &tc, &rc, &sc, false)));
    GH_TRY(dev_alloc(t->mem, (size_t)D * db, &t->final_norm));
    GH_CUDA(launch_fill_const(db, t->final_norm, D, 1.0f, st));
  }
  // RoPE table (cos, sin) computed in double on the host: [S][dh/2]
  {
    const int half = sh.dh / 2;
    std::vector<float2> tab((size_t)sh.S * half);
    for (int p = 0; p < sh.S; ++p)
      for (int i = 0; i < half; ++i) {
        const double freq = std::pow((double)spec->rope_theta, -2.0 * i / (double)sh.dh);
        const double a = (double)p * freq;
        tab[(size_t)p * half + i] = make_float2((float)std::cos(a), (float)std::sin(a));
      }
    void* r;
    GH_TRY(dev_alloc(t->mem, tab.size() * sizeof(float2), &r));
    GH_CUDA(cudaMemcpy(r, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice));
    t->rope = (float2*)r;
  }
  // scratch
  const size_t B = max_batch;
  GH_TRY(dev_alloc(t->mem, B * D * db, &t->xn));
  GH_TRY(dev_alloc(t->mem, B * D * db, &t->h));
  GH_TRY(dev_alloc(t->mem, B * D * db, &t->hn));
  GH_TRY(dev_alloc(t->mem, B * Dh * db, &t->g));
  {
    void* p;
    GH_TRY(dev_alloc(t->mem, (size_t)(D + 127) / 128 * 8 * B * sizeof(float), &p));  // tiles x max C
    t->ss_h = (float*)p;
  }
  {
    void* p;
    const size_t n_slices = (size_t)(V + 127) / 128 * 8;  // tiles x max cluster size
    GH_TRY(dev_alloc(t->mem, n_slices * B * sizeof(float2), &p));
    t->part = (float2*)p;
  }
  if (getenv("GH_GEMM_DBG")) t->gsc.debug_flags = atoi(getenv("GH_GEMM_DBG"));  // diagnostics (wrong results)
  if (db == 2) {  // the CTA-pair kernel's stream-K workspace (batches > 128, or GH_GEMM_PAIR=2)
    void* p;
    GH_TRY(dev_alloc(t->mem, kSkWsBytes, &p));
    t->gsc.sk_ws = (float*)p;
    GH_TRY(dev_alloc(t->mem, kNumSMs * sizeof(unsigned int), &p));
    t->gsc.sk_flags = (unsigned int*)p;
    GH_CUDA(cudaMemset(p, 0, kNumSMs * sizeof(unsigned int)));
  }
  if (db == 4) {
    void* p;
    const size_t n = B * (size_t)std::max({D + 2 * Dkv, 2 * Dh, V, D});
    GH_TRY(dev_alloc(t->mem, n * sizeof(float), &p));
    t->gsc.stage = (float*)p;
    t->gsc.stage_floats = n;
  }
  if (tp > 1) {  // all-reduce receive buffers (mapped by the peers in the engine's setup)
    void* p;
    for (int par = 0; par < 2; ++par) {  // [tp][slices][rows][BN] x 8 B: batch and rows padded to tiles
      const size_t bytes = (size_t)tp * ((B + 127) / 128 * 128) * ((D + 127) / 128 * 128) * 8;
      GH_TRY(dev_alloc(t->mem, bytes, &p));
      GH_CUDA(cudaMemset(p, 0, bytes));  // sequence numbers start at 1
      t->tpc.buf[par] = (float*)p;
    }
  }
  GH_CUDA(cudaDeviceSynchronize());
  *out = t.release();
  return GH_OK;
}

extern "C" {

gh_status gh_tier1_create(const gh_model_spec* spec, int device, uint32_t layer_begin,
                          uint32_t layer_end, uint64_t seed, uint32_t max_batch, gh_tier1** out) {
  return tier1_create(spec, device, layer_begin, layer_end, seed, max_batch, 1, 0, out);
}

gh_status gh_tier1_destroy(gh_tier1* t) {
  if (t) { cudaSetDevice(t->device); cudaDeviceSynchronize(); delete t; }
  return GH_OK;
}

}  // extern "C"

static gh_status t2_attend(gh_tier2* t, uint32_t layer, uint32_t B, const uint32_t* slot, const int32_t* pos,
                           const void* msg_fwd, void* msg_bwd, void* stream, const void* pf, size_t pf_bytes,
                           int kv_early = 0, int tp = 1);

// ---- Tier-1 stage implementations.  `SsRef` describes per-slice sums of squares of an
// activation buffer emitted by its producer (embedding / W2 epilogue) so that the consumer GEMM
// applies RMSNorm in its epilogue (bf16 path) instead of a separate normalisation kernel.  The
// public ABI entry points pass none (they normalise explicitly and are correct for any input);
// the engine, which owns the activation buffers, threads the sums of squares through.
namespace gh {
struct SsRef {
  const float* ss = nullptr;
  int slices = 0;
};
}  // namespace gh

static gh_status t1_embed(gh_tier1* t, uint32_t B, const int32_t* tok, void* x, float* ss_out, cudaStream_t st) {
  if (!t || !tok || !x) return fail(GH_EINVAL, "null argument");
  if (!t->has_embed) return fail(GH_EINVAL, "this Tier-1 span does not own the embedding");
  if (B > t->max_batch) return fail(GH_EINVAL, "B exceeds max_batch");
  GH_CUDA(launch_embed(t->sh.db, t->embed.ptr, tok, x, (int)B, t->sh.D, t->sh.V, t->sh.db == 2 ? ss_out : nullptr, st));
  return GH_OK;
}

static gh_status t1_pre(gh_tier1* t, uint32_t layer, uint32_t B, const void* x, SsRef ss, const int32_t* pos,
                        void* msg_fwd, cudaStream_t st) {
  if (!t || !x || !pos || !msg_fwd) return fail(GH_EINVAL, "null argument");
  if (layer < t->l0 || layer >= t->l1) return fail(GH_EINVAL, "layer not owned by this Tier-1");
  if (B > t->max_batch) return fail(GH_EINVAL, "B exceeds max_batch");
  if (B == 0) return GH_OK;
  const Shape& s = t->sh;
  auto& L = t->layers[layer - t->l0];
  EpiParams ep = epi_default();
  ep.kind = EPI_QKV_ROPE;
  ep.out = (char*)msg_fwd + (size_t)s.D * s.db;
  ep.ldo = s.ld_fwd();
  ep.rope = t->rope;
  ep.pos = pos;
  ep.d_head = s.dh;
  ep.rope_rows = s.D + s.Dkv;
  if (t->tp > 1) {
    // this rank's head block of the message, [x_r | q_r | k_r | v_r] (AttnArgs::tp layout)
    const int Dt = s.D / t->tp;
    if (!(ss.ss && B <= (uint32_t)kFusedNormMaxBatch))
      return fail(GH_EINVAL, "tensor-parallel F1 needs the fused RMSNorm statistics (engine path)");
    ep.out = (char*)msg_fwd + (size_t)Dt * s.db;
    ep.ldo = s.ld_fwd() / t->tp;
    ep.rope_rows = (s.D + s.Dkv) / t->tp;
    ep.ss_in = ss.ss; ep.ss_in_slices = ss.slices; ep.ss_dim = s.D; ep.ss_eps = s.s.norm_eps;
    ep.xcopy_src = (const char*)x + (size_t)t->tp_rank * Dt * s.db; ep.xcopy_ld = s.D; ep.xcopy_rows = Dt;
    return t->gemm(L.qkv, &L.tm_qkv, x, s.D, (int)B, ep, st);
  }
  if (s.db == 2 && ss.ss && B <= (uint32_t)kFusedNormMaxBatch) {
    // fused: QKV on the raw x, RMSNorm scale in the epilogue, x copied into the message there
    ep.ss_in = ss.ss; ep.ss_in_slices = ss.slices; ep.ss_dim = s.D; ep.ss_eps = s.s.norm_eps;
    ep.xcopy_src = x; ep.xcopy_ld = s.D; ep.xcopy_rows = s.D;
    return t->gemm(L.qkv, &L.tm_qkv, x, s.D, (int)B, ep, st);
  }
  // RMSNorm(x) -> xn ; x copied into the message's x slot
  GH_CUDA(launch_rmsnorm(s.db, x, s.D, L.attn_norm, t->xn, s.D, msg_fwd, s.ld_fwd(), (int)B, s.D,
                         s.s.norm_eps, st));
  return t->gemm(L.qkv, &L.tm_qkv, t->xn, s.D, (int)B, ep, st);
}

// x_resid: the layer's input activation [B][D] (tensor-parallel Tier-1: the residual is the local
// replica of x, the message block carries only this rank's columns); nullptr = the bwd message's x.
static gh_status t1_post_tp(gh_tier1* t, uint32_t layer, uint32_t B, const void* msg_bwd, const void* x_resid,
                            void* x_next, float* ss_next, int* ss_next_slices, cudaStream_t st,
                            const PeerWait* pw) {
  const Shape& s = t->sh;
  auto& L = t->layers[layer - t->l0];
  const int Dt = s.D / t->tp, Dht = s.Dh / t->tp;
  if (!x_resid || !ss_next) return fail(GH_EINVAL, "tensor-parallel F3 runs in the engine (residual + statistics)");
  // h = x + sum_r attn_r Wo_r^T   (all-reduced in the epilogue; + sums of squares of h)
  EpiParams ep = epi_default();
  ep.kind = EPI_STORE_RESID;
  ep.out = t->h; ep.ldo = s.D;
  ep.resid = x_resid; ep.ldr = s.D;
  ep.ss_out = t->ss_h;
  GH_TRY(epi_tp(t, (int)B, ep));
  GH_TRY(t->gemm(L.o, &L.tm_o, (const char*)msg_bwd + (size_t)Dt * s.db, s.ld_bwd() / t->tp, (int)B, ep, st,
                 &L.w13, pw));
  // g_r = silu(rms(h) W1_r^T) * (rms(h) W3_r^T): this rank's hidden units
  ep = epi_default();
  ep.kind = EPI_SWIGLU;
  ep.out = t->g; ep.ldo = Dht;
  ep.ss_in = t->ss_h; ep.ss_in_slices = t->plan(s.D, Dt, (int)B, true).slices(); ep.ss_dim = s.D;
  ep.ss_eps = s.s.norm_eps;
  GH_TRY(t->gemm(L.w13, &L.tm_13, t->h, s.D, (int)B, ep, st, &L.w2));
  // x_next = h + sum_r g_r W2_r^T   (all-reduced; + sums of squares of x_next)
  ep = epi_default();
  ep.kind = EPI_STORE_RESID;
  ep.out = x_next; ep.ldo = s.D;
  ep.resid = t->h; ep.ldr = s.D;
  ep.ss_out = ss_next;
  if (ss_next_slices) *ss_next_slices = t->plan(s.D, Dht, (int)B, true).slices();
  GH_TRY(epi_tp(t, (int)B, ep));
  const Weight* next = layer + 1 < t->l1 ? &t->layers[layer + 1 - t->l0].qkv : (t->has_cls ? &t->cls : nullptr);
  return t->gemm(L.w2, &L.tm_2, t->g, Dht, (int)B, ep, st, next);
}

static gh_status t1_post(gh_tier1* t, uint32_t layer, uint32_t B, const void* msg_bwd, void* x_next, float* ss_next,
                         int* ss_next_slices, cudaStream_t st, const void* x_resid = nullptr,
                         const PeerWait* pw = nullptr) {
  if (!t || !msg_bwd || !x_next) return fail(GH_EINVAL, "null argument");
  if (layer < t->l0 || layer >= t->l1) return fail(GH_EINVAL, "layer not owned by this Tier-1");
  if (B > t->max_batch) return fail(GH_EINVAL, "B exceeds max_batch");
  if (B == 0) return GH_OK;
  if (t->tp > 1) return t1_post_tp(t, layer, B, msg_bwd, x_resid, x_next, ss_next, ss_next_slices, st, pw);
  const Shape& s = t->sh;
  auto& L = t->layers[layer - t->l0];
  const bool fused = s.db == 2 && B <= (uint32_t)kFusedNormMaxBatch;
  // h = attn Wo^T + x   (+ per-slice sums of squares of h for the fused FFN norm)
  EpiParams ep = epi_default();
  ep.kind = EPI_STORE_RESID;
  ep.out = t->h; ep.ldo = s.D;
  ep.resid = msg_bwd; ep.ldr = s.ld_bwd();
  if (fused) ep.ss_out = t->ss_h;
  GH_TRY(t->gemm(L.o, &L.tm_o, (const char*)msg_bwd + (size_t)s.D * s.db, s.ld_bwd(), (int)B, ep, st, &L.w13, pw));
  // g = silu(rms(h) W1^T) * (rms(h) W3^T)
  const void* ffn_in = t->h;
  ep = epi_default();
  ep.kind = EPI_SWIGLU;
  ep.out = t->g; ep.ldo = s.Dh;
  if (fused) {
    ep.ss_in = t->ss_h; ep.ss_in_slices = t->plan(s.D, s.D, (int)B).slices(); ep.ss_dim = s.D;
    ep.ss_eps = s.s.norm_eps;
  } else {
    GH_CUDA(launch_rmsnorm(s.db, t->h, s.D, L.ffn_norm, t->hn, s.D, nullptr, 0, (int)B, s.D, s.s.norm_eps, st));
    ffn_in = t->hn;
  }
  GH_TRY(t->gemm(L.w13, &L.tm_13, ffn_in, s.D, (int)B, ep, st, &L.w2));
  // x_next = g W2^T + h   (+ sums of squares of x_next for the next fused norm)
  ep = epi_default();
  ep.kind = EPI_STORE_RESID;
  ep.out = x_next; ep.ldo = s.D;
  ep.resid = t->h; ep.ldr = s.D;
  if (fused && ss_next) {
    ep.ss_out = ss_next;
    if (ss_next_slices) *ss_next_slices = t->plan(s.D, s.Dh, (int)B).slices();
  }
  const Weight* next = layer + 1 < t->l1 ? &t->layers[layer + 1 - t->l0].qkv : (t->has_cls ? &t->cls : nullptr);
  return t->gemm(L.w2, &L.tm_2, t->g, s.Dh, (int)B, ep, st, next);
}

// Sampling (all three may be null = greedy): inv_temp [B] (0 = greedy row), seed [B], pos [B].
static gh_status t1_classify(gh_tier1* t, uint32_t B, const void* x, SsRef ss, float* logits, int32_t* next,
                             cudaStream_t st, const float* inv_temp = nullptr, const uint32_t* seed = nullptr,
                             const int32_t* pos = nullptr) {
  if (inv_temp && (!seed || !pos || !logits)) return fail(GH_EINVAL, "sampling needs seed, pos and a logits buffer");
  if (!t || !x || !next) return fail(GH_EINVAL, "null argument");
  if (!t->has_cls) return fail(GH_EINVAL, "this Tier-1 span does not own the classifier");
  if (B > t->max_batch) return fail(GH_EINVAL, "B exceeds max_batch");
  if (B == 0) return GH_OK;
  const Shape& s = t->sh;
  EpiParams ep = epi_default();
  ep.kind = EPI_LOGITS_ARGMAX;
  ep.logits = logits; ep.ldl = s.V;
  ep.part = t->part;
  const void* in = x;
  if (s.db == 2 && ss.ss && B <= (uint32_t)kFusedNormMaxBatch) {
    ep.ss_in = ss.ss; ep.ss_in_slices = ss.slices; ep.ss_dim = s.D; ep.ss_eps = s.s.norm_eps;
  } else {
    GH_CUDA(launch_rmsnorm(s.db, x, s.D, t->final_norm, t->xn, s.D, nullptr, 0, (int)B, s.D, s.s.norm_eps, st));
    in = t->xn;
  }
  GH_TRY(t->gemm(t->cls, &t->tm_cls, in, s.D, (int)B, ep, st, t->l1 > t->l0 ? &t->layers[0].qkv : nullptr));
  if (inv_temp) {  // temperature sampling over the written logits (keeps the GEMM epilogue lean)
    GH_CUDA(launch_argmax_rows(logits, (int)B, s.V, next, st, inv_temp, seed, pos));
  } else if (s.db == 2) {
    GH_CUDA(launch_argmax_final(t->part, t->plan(s.V, s.D, (int)B).slices(), (int)B, next, st));
  } else {
    GH_CUDA(launch_argmax_rows(logits ? logits : t->gsc.stage, (int)B, s.V, next, st, inv_temp, seed, pos));
  }
  return GH_OK;
}

extern "C" {

gh_status gh_tier1_classify_sample(gh_tier1* t, uint32_t B, const void* x, const int32_t* pos,
                                   const float* inv_temperature, const uint32_t* seed, float* logits,
                                   int32_t* next_tok, void* stream) {
  return t1_classify(t, B, x, SsRef{}, logits, next_tok, (cudaStream_t)stream, inv_temperature, seed, pos);
}

gh_status gh_tier1_embed(gh_tier1* t, uint32_t B, const int32_t* tok, void* x, void* stream) {
  return t1_embed(t, B, tok, x, nullptr, (cudaStream_t)stream);
}
gh_status gh_tier1_pre(gh_tier1* t, uint32_t layer, uint32_t B, const void* x, const int32_t* pos,
                       void* msg_fwd, void* stream) {
  return t1_pre(t, layer, B, x, SsRef{}, pos, msg_fwd, (cudaStream_t)stream);
}
gh_status gh_tier1_post(gh_tier1* t, uint32_t layer, uint32_t B, const void* msg_bwd, void* x_next,
                        void* stream) {
  return t1_post(t, layer, B, msg_bwd, x_next, nullptr, nullptr, (cudaStream_t)stream);
}
gh_status gh_tier1_classify(gh_tier1* t, uint32_t B, const void* x, float* logits, int32_t* next,
                            void* stream) {
  return t1_classify(t, B, x, SsRef{}, logits, next, (cudaStream_t)stream);
}

}  // extern "C"

// ================================================================== Tier-2
static_assert(kKvPagePositions == GH_KV_PAGE_POSITIONS, "page size of the ABI");

struct gh_tier2 {
  Shape sh;
  int device = 0;
  uint32_t l0 = 0, l1 = 0, n_slots = 0;
  std::vector<std::unique_ptr<DevMem>> mem;
  void* arena = nullptr;
  size_t arena_bytes = 0;
  bool has_tmap = false;
  CUtensorMap kv_tmap;  // whole arena, 3-D (tensor-core GQA attention)
  // paged arena: a pool of n_pages pages of kKvPagePositions positions (all layers of the span use
  // the same page ids); page_table[slot][p] maps a slot's positions [64p, 64p + 64) to a page
  bool paged = false;
  uint32_t n_pages = 0, max_pages = 0;
  int* d_pt = nullptr;              // device [n_slots][max_pages]
  int* d_limit = nullptr;           // device [n_slots] (synthetic fill of ragged contexts)
  // attention work counters (dynamic unit schedule), one pair per launch from a ring so that
  // launches in flight at the same time (in-flight batches) never share one
  static constexpr int kWorkRing = 64;
  unsigned int* work = nullptr;
  int work_next = 0;
  std::vector<int> h_pt;            // host mirror
  std::vector<uint32_t> mapped;     // pages mapped per slot
  std::vector<int> free_pages;      // LIFO pool
  // stream-ordered page-table updates (the dispatcher maps without synchronising): pinned
  // mirrors of the table, one per step of a small ring, each guarded by the event of its copies
  static constexpr int kPtRing = 4;
  int* pt_stage[kPtRing] = {};
  cudaEvent_t pt_ev[kPtRing] = {};
  int pt_cur = -1;
  ~gh_tier2() {
    for (int i = 0; i < kPtRing; ++i) {
      if (pt_stage[i]) cudaFreeHost(pt_stage[i]);
      if (pt_ev[i]) cudaEventDestroy(pt_ev[i]);
    }
  }
  long span() const { return paged ? kKvPagePositions : sh.S; }   // positions per block
  long slot_stride() const { return 2L * sh.Hkv * span() * sh.dh; }  // per slot (contiguous) or page
  long kv_stride() const { return (long)sh.Hkv * span() * sh.dh; }
  long head_stride() const { return span() * sh.dh; }
  long layer_stride() const { return (long)(paged ? n_pages : n_slots) * slot_stride(); }
  void layout(AttnArgs& a) const {
    a.slot_stride = slot_stride();
    a.kv_stride = kv_stride();
    a.head_stride = head_stride();
    a.n_slots = (int)(paged ? n_pages : n_slots);
    a.page_table = paged ? d_pt : nullptr;
    a.max_pages = (int)max_pages;
  }
};

static gh_status tier2_create(const gh_model_spec* spec, int device, uint32_t layer_begin, uint32_t layer_end,
                              uint32_t n_slots, uint32_t n_pages, gh_tier2** out) {
  if (!out) return fail(GH_EINVAL, "out is null");
  *out = nullptr;
  Shape sh;
  GH_TRY(Shape::from(spec, &sh));
  if (layer_begin >= layer_end || layer_end > (uint32_t)sh.N) return fail(GH_EINVAL, "bad layer range");
  if (n_slots == 0) return fail(GH_EINVAL, "n_slots must be >= 1");
  if (gh_device_count() <= device) return fail(GH_ECUDA, "no CUDA device " + std::to_string(device));
  GH_CUDA(cudaSetDevice(device));
  GH_CUDA(configure_kernels());
  auto t = std::make_unique<gh_tier2>();
  t->sh = sh; t->device = device; t->l0 = layer_begin; t->l1 = layer_end; t->n_slots = n_slots;
  t->paged = n_pages > 0;
  t->n_pages = n_pages;
  t->max_pages = (uint32_t)((sh.S + kKvPagePositions - 1) / kKvPagePositions);
  t->arena_bytes = (size_t)(layer_end - layer_begin) * (size_t)t->layer_stride() * sh.db;
  size_t free_b = 0, total_b = 0;
  GH_CUDA(cudaMemGetInfo(&free_b, &total_b));
  if (t->arena_bytes > free_b)
    return fail(GH_EINFEASIBLE, "KV arena of " + std::to_string(t->arena_bytes) +
                                    " bytes exceeds free device memory (binding constraint: memory)");
  GH_TRY(dev_alloc(t->mem, t->arena_bytes, &t->arena));
  // zeroed once: never-written positions are finite (tile loads past a prompt's length are masked,
  // and 0 x NaN would not be)
  GH_CUDA(cudaMemset(t->arena, 0, t->arena_bytes));
  {
    void* p;
    GH_TRY(dev_alloc(t->mem, gh_tier2::kWorkRing * 2 * sizeof(unsigned int), &p));
    GH_CUDA(cudaMemset(p, 0, gh_tier2::kWorkRing * 2 * sizeof(unsigned int)));
    t->work = (unsigned int*)p;
  }
  if (t->paged) {
    void* p;
    const size_t n = (size_t)n_slots * t->max_pages;
    GH_TRY(dev_alloc(t->mem, n * sizeof(int), &p));
    t->d_pt = (int*)p;
    GH_TRY(dev_alloc(t->mem, (size_t)n_slots * sizeof(int), &p));
    t->d_limit = (int*)p;
    t->h_pt.assign(n, 0);  // unmapped entries point at page 0 (a valid address; never attended)
    GH_CUDA(cudaMemcpy(t->d_pt, t->h_pt.data(), n * sizeof(int), cudaMemcpyHostToDevice));
    t->mapped.assign(n_slots, 0);
    for (uint32_t i = 0; i < n_pages; ++i) t->free_pages.push_back((int)(n_pages - 1 - i));
  }
  if (sh.db == 2 && sh.dh == 128) {
    const uint64_t rows = (uint64_t)(layer_end - layer_begin) * (t->paged ? n_pages : n_slots) * 2 * sh.Hkv;
    t->has_tmap = make_tmap_kv(&t->kv_tmap, t->arena, rows, (uint64_t)t->span(), 128) == cudaSuccess;
  }
  *out = t.release();
  return GH_OK;
}

extern "C" {

gh_status gh_tier2_create(const gh_model_spec* spec, int device, uint32_t layer_begin,
                          uint32_t layer_end, uint32_t n_slots, gh_tier2** out) {
  return tier2_create(spec, device, layer_begin, layer_end, n_slots, 0, out);
}

gh_status gh_tier2_create_paged(const gh_model_spec* spec, int device, uint32_t layer_begin, uint32_t layer_end,
                                uint32_t n_slots, uint32_t n_pages, gh_tier2** out) {
  if (n_pages == 0) return fail(GH_EINVAL, "n_pages must be >= 1");
  return tier2_create(spec, device, layer_begin, layer_end, n_slots, n_pages, out);
}

gh_status gh_tier2_map(gh_tier2* t, uint32_t slot, uint32_t n_positions, void* stream) {
  if (!t) return fail(GH_EINVAL, "null argument");
  if (slot >= t->n_slots) return fail(GH_EINVAL, "slot " + std::to_string(slot) + " >= n_slots");
  if (n_positions > (uint32_t)t->sh.S)
    return fail(GH_EINFEASIBLE, std::to_string(n_positions) + " positions exceed max_seq_len");
  if (!t->paged) return GH_OK;  // contiguous slots hold max_seq_len positions
  const uint32_t need = (n_positions + kKvPagePositions - 1) / kKvPagePositions;
  const uint32_t have = t->mapped[slot];
  if (need <= have) return GH_OK;
  if (need - have > t->free_pages.size())
    return fail(GH_EINFEASIBLE, "KV page pool exhausted: " + std::to_string(need - have) + " pages needed, " +
                                    std::to_string(t->free_pages.size()) + " free (binding constraint: memory)");
  GH_CUDA(cudaSetDevice(t->device));
  cudaStream_t st = (cudaStream_t)stream;
  GH_CUDA(cudaStreamSynchronize(st));  // steps already queued on `stream` see the old table
  int* row = t->h_pt.data() + (size_t)slot * t->max_pages;
  for (uint32_t p = have; p < need; ++p) {
    row[p] = t->free_pages.back();
    t->free_pages.pop_back();
  }
  t->mapped[slot] = need;
  GH_CUDA(cudaMemcpyAsync(t->d_pt + (size_t)slot * t->max_pages + have, row + have, (size_t)(need - have) * sizeof(int),
                          cudaMemcpyHostToDevice, st));
  GH_CUDA(cudaStreamSynchronize(st));
  return GH_OK;
}

}  // extern "C"

// ---- stream-ordered page-table updates (dispatcher).  Steps already queued on the stream keep
// reading the old entries; the copy lands before the next step, so no host synchronisation.
static gh_status t2_updates_begin(gh_tier2* t) {
  if (!t->paged) return GH_OK;
  t->pt_cur = (t->pt_cur + 1) % gh_tier2::kPtRing;
  const int c = t->pt_cur;
  const size_t n = (size_t)t->n_slots * t->max_pages;
  if (!t->pt_stage[c]) {
    GH_CUDA(cudaMallocHost((void**)&t->pt_stage[c], n * sizeof(int)));
    GH_CUDA(cudaEventCreateWithFlags(&t->pt_ev[c], cudaEventDisableTiming));
  } else {
    GH_CUDA(cudaEventSynchronize(t->pt_ev[c]));  // its copies of kPtRing steps ago are done
  }
  return GH_OK;
}
static gh_status t2_map_async(gh_tier2* t, uint32_t slot, uint32_t n_positions, cudaStream_t st) {
  if (slot >= t->n_slots) return fail(GH_EINVAL, "slot " + std::to_string(slot) + " >= n_slots");
  if (n_positions > (uint32_t)t->sh.S)
    return fail(GH_EINFEASIBLE, std::to_string(n_positions) + " positions exceed max_seq_len");
  if (!t->paged) return GH_OK;
  const uint32_t need = (n_positions + kKvPagePositions - 1) / kKvPagePositions;
  const uint32_t have = t->mapped[slot];
  if (need <= have) return GH_OK;
  if (need - have > t->free_pages.size())
    return fail(GH_EINFEASIBLE, "KV page pool exhausted (binding constraint: memory)");
  const size_t base = (size_t)slot * t->max_pages;
  int* row = t->h_pt.data() + base;
  int* stage = t->pt_stage[t->pt_cur] + base;
  for (uint32_t p = have; p < need; ++p) {
    row[p] = t->free_pages.back();
    t->free_pages.pop_back();
    stage[p] = row[p];
  }
  t->mapped[slot] = need;
  GH_CUDA(cudaMemcpyAsync(t->d_pt + base + have, stage + have, (size_t)(need - have) * sizeof(int),
                          cudaMemcpyHostToDevice, st));
  return GH_OK;
}
static gh_status t2_updates_end(gh_tier2* t, cudaStream_t st) {
  if (t->paged) GH_CUDA(cudaEventRecord(t->pt_ev[t->pt_cur], st));
  return GH_OK;
}

extern "C" {

gh_status gh_tier2_unmap(gh_tier2* t, uint32_t slot) {
  if (!t) return fail(GH_EINVAL, "null argument");
  if (slot >= t->n_slots) return fail(GH_EINVAL, "slot " + std::to_string(slot) + " >= n_slots");
  if (!t->paged) return GH_OK;
  int* row = t->h_pt.data() + (size_t)slot * t->max_pages;
  for (uint32_t p = t->mapped[slot]; p-- > 0;) t->free_pages.push_back(row[p]);
  t->mapped[slot] = 0;
  return GH_OK;
}

uint32_t gh_tier2_pages_free(const gh_tier2* t) { return t && t->paged ? (uint32_t)t->free_pages.size() : 0; }

gh_status gh_tier2_destroy(gh_tier2* t) {
  if (t) { cudaSetDevice(t->device); cudaDeviceSynchronize(); delete t; }
  return GH_OK;
}

uint64_t gh_tier2_arena_bytes(const gh_tier2* t) { return t ? t->arena_bytes : 0; }

gh_status gh_tier2_check(const gh_tier2* t, uint32_t B, const uint32_t* slot, const int32_t* pos) {
  if (!t || (B && (!slot || !pos))) return fail(GH_EINVAL, "null argument");
  for (uint32_t b = 0; b < B; ++b) {
    if (slot[b] >= t->n_slots)
      return fail(GH_EINFEASIBLE, "slot " + std::to_string(slot[b]) + " >= n_slots " + std::to_string(t->n_slots) +
                                      " (binding constraint: memory)");
    if (pos[b] < 0 || pos[b] >= t->sh.S)
      return fail(GH_EINFEASIBLE, "position " + std::to_string(pos[b]) + " outside [0, max_seq_len)");
    if (t->paged && (uint32_t)pos[b] / kKvPagePositions >= t->mapped[slot[b]])
      return fail(GH_EINFEASIBLE, "position " + std::to_string(pos[b]) + " of slot " + std::to_string(slot[b]) +
                                      " is not mapped to a KV page (gh_tier2_map)");
  }
  return GH_OK;
}

gh_status gh_tier2_attend(gh_tier2* t, uint32_t layer, uint32_t B, const uint32_t* slot, const int32_t* pos,
                          const void* msg_fwd, void* msg_bwd, void* stream) {
  return t2_attend(t, layer, B, slot, pos, msg_fwd, msg_bwd, stream, nullptr, 0);
}
}  // extern "C"

// `pf`: leading bytes of the weight Tier-1 streams next on this GPU (colocated engine), prefetched
// into L2 during the attention kernel's tail
// `kv_early`: the caller guarantees the kernel's predecessor writes neither the arena nor pos / slot
static gh_status t2_attend(gh_tier2* t, uint32_t layer, uint32_t B, const uint32_t* slot, const int32_t* pos,
                           const void* msg_fwd, void* msg_bwd, void* stream, const void* pf, size_t pf_bytes,
                           int kv_early, int tp) {
  if (!t || !slot || !pos || !msg_fwd || !msg_bwd) return fail(GH_EINVAL, "null argument");
  if (layer < t->l0 || layer >= t->l1) return fail(GH_EINVAL, "layer not owned by this Tier-2");
  if (B == 0) return GH_OK;
  const Shape& s = t->sh;
  if (tp > 1 && !(t->has_tmap && s.Hkv % tp == 0))
    return fail(GH_EUNSUPPORTED, "head-blocked (tensor-parallel) messages need the tensor-core attention kernel");
  AttnArgs a;
  a.tp = tp;
  a.msg_fwd = msg_fwd;
  a.msg_bwd = msg_bwd;
  a.arena = (char*)t->arena + (size_t)(layer - t->l0) * t->layer_stride() * s.db;
  a.slot = slot;
  a.pos = pos;
  t->layout(a);
  a.B = (int)B; a.H = s.H; a.Hkv = s.Hkv; a.D = s.D; a.Dkv = s.Dkv;
  a.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)s.dh));
  static const int attn_flags = getenv("GH_ATTN_FLAGS") ? atoi(getenv("GH_ATTN_FLAGS")) : 0;  // diagnostics
  a.flags = attn_flags;
  a.pf = pf;
  a.pf_bytes = pf ? pf_bytes : 0;
  a.layer_local = (int)(layer - t->l0);
  static const bool static_units = getenv("GH_ATTN_STATIC") != nullptr;  // diagnostics
  a.work = static_units ? nullptr : t->work + 2 * (t->work_next++ % gh_tier2::kWorkRing);
  a.kv_tmap = t->has_tmap ? &t->kv_tmap : nullptr;
  static const bool no_early = getenv("GH_ATTN_NO_EARLY") != nullptr;  // diagnostics
  a.kv_early = kv_early && !no_early;
  GH_CUDA(launch_attention(s.db, s.dh, a, (cudaStream_t)stream));
  return GH_OK;
}

static gh_status t2_append(gh_tier2* t, uint32_t layer, uint32_t B, const uint32_t* slot, const int32_t* pos,
                           const void* msg_fwd, void* stream) {
  if (!t || !slot || !pos || !msg_fwd) return fail(GH_EINVAL, "null argument");
  if (layer < t->l0 || layer >= t->l1) return fail(GH_EINVAL, "layer not owned by this Tier-2");
  if (B == 0) return GH_OK;
  const Shape& s = t->sh;
  AttnArgs a{};
  a.msg_fwd = msg_fwd;
  a.arena = (char*)t->arena + (size_t)(layer - t->l0) * t->layer_stride() * s.db;
  a.slot = slot;
  a.pos = pos;
  t->layout(a);
  a.B = (int)B; a.H = s.H; a.Hkv = s.Hkv; a.D = s.D; a.Dkv = s.Dkv;
  GH_CUDA(launch_append_kv(s.db, s.dh, a, (cudaStream_t)stream));
  return GH_OK;
}

extern "C" {

gh_status gh_tier2_append(gh_tier2* t, uint32_t layer, uint32_t B, const uint32_t* slot, const int32_t* pos,
                          const void* msg_fwd, void* stream) {
  return t2_append(t, layer, B, slot, pos, msg_fwd, stream);
}

gh_status gh_tier2_fill_synthetic(gh_tier2* t, uint64_t seed, uint32_t n_fill, uint32_t npos, void* stream) {
  if (!t) return fail(GH_EINVAL, "null argument");
  if (n_fill > t->n_slots || npos > (uint32_t)t->sh.S) return fail(GH_EINVAL, "fill exceeds arena");
  const int* limit = nullptr;
  if (t->paged) {  // each slot is filled up to its mapping (ragged contexts), at least one page
    std::vector<int> lim(n_fill);
    for (uint32_t i = 0; i < n_fill; ++i) {
      if (t->mapped[i] == 0)
        return fail(GH_EINVAL, "fill: slot " + std::to_string(i) + " has no KV pages (gh_tier2_map)");
      lim[i] = (int)std::min<uint32_t>(npos, t->mapped[i] * (uint32_t)kKvPagePositions);
    }
    if (n_fill) {
      GH_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
      GH_CUDA(cudaMemcpy(t->d_limit, lim.data(), n_fill * sizeof(int), cudaMemcpyHostToDevice));
    }
    limit = t->d_limit;
  }
  AttnArgs lay{};
  t->layout(lay);
  GH_CUDA(launch_fill_kv(t->sh.db, t->arena, seed, (int)t->l0, (int)t->l1, (int)n_fill, t->layer_stride(), lay,
                         limit, t->sh.Hkv, t->sh.S, t->sh.dh, (int)npos, (cudaStream_t)stream));
  return GH_OK;
}

// host layout: paged [layer][page][2][Hkv][64][dh] (whole pages); contiguous [layer][2 Hkv][n][dh]
uint64_t gh_tier2_kv_swap_bytes(const gh_tier2* t, uint32_t n) {
  if (!t) return 0;
  const uint64_t P = t->paged ? (uint64_t)((n + kKvPagePositions - 1) / kKvPagePositions) * kKvPagePositions : n;
  return (uint64_t)(t->l1 - t->l0) * 2 * t->sh.Hkv * P * t->sh.dh * t->sh.db;
}

}  // extern "C"

// The swap copies of one slot, queued on `stream` (ordered after the steps already queued there,
// before the ones queued later); gh_tier2_kv_swap waits for them, the dispatcher does not.
static gh_status t2_kv_swap_async(gh_tier2* t, uint32_t slot, uint32_t n, void* host, int to_host, cudaStream_t st) {
  if (!t || !host) return fail(GH_EINVAL, "null argument");
  if (slot >= t->n_slots || n > (uint32_t)t->sh.S) return fail(GH_EINVAL, "kv_swap out of range");
  if (t->paged && t->mapped[slot] * (uint32_t)kKvPagePositions < n)
    return fail(GH_EINVAL, "kv_swap: positions are not mapped");
  if (n == 0) return GH_OK;
  const Shape& s = t->sh;
  GH_CUDA(cudaSetDevice(t->device));
  const cudaMemcpyKind kind = to_host ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice;
  char* h = (char*)host;
  char* arena = (char*)t->arena;
  for (int l = 0; l < (int)(t->l1 - t->l0); ++l) {
    const size_t lbase = (size_t)l * t->layer_stride() * s.db;
    if (t->paged) {  // one block of 2 x Hkv x 64 positions per page
      const uint32_t np = (n + kKvPagePositions - 1) / kKvPagePositions;
      const size_t blk = (size_t)t->slot_stride() * s.db;
      for (uint32_t p = 0; p < np; ++p) {
        char* d = arena + lbase + (size_t)t->h_pt[(size_t)slot * t->max_pages + p] * blk;
        if (to_host) GH_CUDA(cudaMemcpyAsync(h, d, blk, kind, st));
        else GH_CUDA(cudaMemcpyAsync(d, h, blk, kind, st));
        h += blk;
      }
    } else {  // 2 x Hkv rows of n positions at a pitch of max_seq_len positions
      const size_t row = (size_t)n * s.dh * s.db, pitch = (size_t)t->span() * s.dh * s.db;
      char* d = arena + lbase + (size_t)slot * t->slot_stride() * s.db;
      if (to_host) GH_CUDA(cudaMemcpy2DAsync(h, row, d, pitch, row, 2 * s.Hkv, kind, st));
      else GH_CUDA(cudaMemcpy2DAsync(d, pitch, h, row, row, 2 * s.Hkv, kind, st));
      h += row * 2 * s.Hkv;
    }
  }
  return GH_OK;
}

extern "C" {

gh_status gh_tier2_kv_swap(gh_tier2* t, uint32_t slot, uint32_t n, void* host, int to_host, void* stream) {
  GH_TRY(t2_kv_swap_async(t, slot, n, host, to_host, (cudaStream_t)stream));
  if (t && host && n) GH_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  return GH_OK;
}

gh_status gh_tier2_read_kv(gh_tier2* t, uint32_t layer, uint32_t slot, uint32_t kv, uint32_t head,
                           uint32_t n, void* host_out) {
  if (!t || !host_out) return fail(GH_EINVAL, "null argument");
  if (layer < t->l0 || layer >= t->l1 || slot >= t->n_slots || kv > 1 || head >= (uint32_t)t->sh.Hkv ||
      n > (uint32_t)t->sh.S)
    return fail(GH_EINVAL, "read_kv out of range");
  if (t->paged && t->mapped[slot] * (uint32_t)kKvPagePositions < n)
    return fail(GH_EINVAL, "read_kv: positions are not mapped");
  const Shape& s = t->sh;
  GH_CUDA(cudaSetDevice(t->device));
  GH_CUDA(cudaDeviceSynchronize());
  AttnArgs lay{};
  t->layout(lay);
  lay.page_table = t->paged ? t->h_pt.data() : nullptr;  // host mirror for the offsets
  const size_t lbase = (size_t)(layer - t->l0) * t->layer_stride();
  for (uint32_t q = 0; q < n;) {  // contiguous runs (one page at most when paged)
    const uint32_t m = t->paged ? std::min<uint32_t>(n - q, kKvPagePositions - q % kKvPagePositions) : n - q;
    const size_t off = lbase + kv_offset(lay, (int)slot, (int)head, (int)q, s.dh) + (size_t)kv * t->kv_stride();
    GH_CUDA(cudaMemcpy((char*)host_out + (size_t)q * s.dh * s.db, (char*)t->arena + off * s.db,
                       (size_t)m * s.dh * s.db, cudaMemcpyDeviceToHost));
    q += m;
  }
  return GH_OK;
}

}  // extern "C"

// ================================================================== NCCL transport (dlopen)
namespace {
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) { api.why = std::string("dlopen libnccl.so.2 failed: ") + dlerror(); return; }
#define GH_SYM(name) api.name = (decltype(api.name))dlsym(h, "nccl" #name); if (!api.name) { api.why = "missing nccl" #name; return; }
    GH_SYM(GetUniqueId) GH_SYM(CommInitRank) GH_SYM(CommDestroy) GH_SYM(Send) GH_SYM(Recv)
    GH_SYM(GroupStart) GH_SYM(GroupEnd) GH_SYM(AllGather) GH_SYM(AllReduce) GH_SYM(GetErrorString)
#undef GH_SYM
    api.ok = true;
  });
  return api;
}
}  // namespace

#define GH_NCCL(call)                                                                          \
  do {                                                                                         \
    ncclResult_t r_ = (call);                                                                  \
    if (r_ != ncclSuccess) return fail(GH_ENCCL, std::string(#call) + ": " + nccl().GetErrorString(r_)); \
  } while (0)

struct gh_comm {
  int nranks = 0, rank = 0, device = 0;
  std::vector<ncclComm_t> comms;  // one communicator per in-flight batch
};

extern "C" {

gh_status gh_comm_unique_id(uint8_t out[128]) {
  if (!out) return fail(GH_EINVAL, "null argument");
  if (!nccl().ok) return fail(GH_ENCCL, nccl().why);
  ncclUniqueId id;
  GH_NCCL(nccl().GetUniqueId(&id));
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  memcpy(out, &id, 128);
  return GH_OK;
}

gh_status gh_comm_create_n(const uint8_t* ids, int n_comms, int nranks, int rank, int device, gh_comm** out) {
  if (!ids || !out || n_comms < 1) return fail(GH_EINVAL, "bad argument");
  if (!nccl().ok) return fail(GH_ENCCL, nccl().why);
  GH_CUDA(cudaSetDevice(device));
  auto c = std::make_unique<gh_comm>();
  c->nranks = nranks; c->rank = rank; c->device = device;
  for (int i = 0; i < n_comms; ++i) {
    ncclUniqueId id;
    memcpy(&id, ids + 128 * i, 128);
    ncclComm_t comm;
    GH_NCCL(nccl().CommInitRank(&comm, nranks, id, rank));
    c->comms.push_back(comm);
  }
  *out = c.release();
  return GH_OK;
}

gh_status gh_comm_create(const uint8_t unique_id[128], int nranks, int rank, int device, gh_comm** out) {
  return gh_comm_create_n(unique_id, 1, nranks, rank, device, out);
}

gh_status gh_comm_destroy(gh_comm* c) {
  if (c) {
    for (auto cm : c->comms) nccl().CommDestroy(cm);
    delete c;
  }
  return GH_OK;
}

}  // extern "C"

// ================================================================== Engine
// colocated: Tier-1 + Tier-2 on this GPU.  Tier split: rank 0 = Tier-1, ranks 1.. = Tier-2.
struct gh_engine {
  gh_engine_config cfg{};
  Shape sh;
  int role = 0;  // 0 colocated, 1 tier1, 2 tier2
  gh_comm* comm = nullptr;
  int kp = 0;    // K' = number of Tier-2 ranks per Tier-1 span (split mode)
  int n1 = 1;    // Tier-1 pipeline stages (layer spans)
  int span = 0;  // this rank's span (tier1 / tier2)
  int shard = 0; // tier2: this rank's prompt shard within its span
  int l0 = 0, l1 = 0;  // this rank's layers
  int tp = 1;    // Tier-1 tensor-parallel ranks: ranks 0..tp-1 share every layer
  int t1n() const { return tp > 1 ? tp : n1; }  // Tier-1 ranks (TP ranks or pipeline spans)
  int t2_rank(int sp, int j) const { return t1n() + sp * kp + j; }
  // message rows of this rank: a TP Tier-1 rank holds its head block [x_r|q_r|k_r|v_r] / [x_r|attn_r]
  long fwd_w() const { return sh.ld_fwd() / (role == 1 ? tp : 1); }
  long bwd_w() const { return sh.ld_bwd() / (role == 1 ? tp : 1); }
  gh_tier1* t1 = nullptr;
  gh_tier2* t2 = nullptr;
  std::vector<std::unique_ptr<DevMem>> mem;
  struct Batch {
    int32_t *tok = nullptr, *pos = nullptr, *next = nullptr;
    uint32_t* slot = nullptr;
    std::vector<uint32_t> slot_host;       // host copy of `slot` (admission checks)
    float* inv_temp = nullptr;             // [R] 1 / temperature per row (0 = greedy), sampling
    uint32_t* seed = nullptr;              // [R] sampling seed per row
    bool sampling = false;                 // some row has T > 0 (classifier path; graph recaptured on change)
    void *x0 = nullptr, *x1 = nullptr, *fwd = nullptr, *bwd = nullptr;
    float *ss0 = nullptr, *ss1 = nullptr;  // per-slice sums of squares of x0 / x1 (fused RMSNorm)
    int ss_slices[2] = {0, 0};
    int cur = 0;                           // which of x0 / x1 holds the current activation
    void* x(int i) const { return i ? x1 : x0; }
    float* ss(int i) const { return i ? ss1 : ss0; }
    float* logits = nullptr;
    cudaStream_t stream = nullptr;
    cudaEvent_t done = nullptr;
    cudaGraphExec_t graph = nullptr;
    // first span of Tier-1 pipeline spans: gh_engine_advance is applied when the batch's next step
    // starts (after its tokens came back from the last span), not at the end of this step
    bool adv_pending = false;
    int adv_inc = 0;
  };
  std::vector<Batch> batches;
  bool keep_logits = false;               // classifier runs also store the logits (gh_engine_keep_logits)
  std::vector<int> shard_off, shard_cnt;  // split mode: per Tier-2 rank
  int my_cnt = 0;                         // tier2: prompts of my shard per batch
  cudaEvent_t fork = nullptr;
  // Peer transport (split mode, pipelined step): messages are written straight into the
  // receiving GPU's buffers over NVLink by copy engines (CUDA IPC mappings of the peer's
  // cudaMalloc buffers), and completion is a sequence number written into the receiver's flag
  // word after the copy (cuStreamWriteValue32) and awaited by the receiver's compute stream
  // (cuStreamWaitValue32) -- no SM time and no NCCL kernel on either side.
  struct Peer {
    bool on = false;
    // my flag words, IF x (K' + 3): [ib*K' + j] bwd of Tier-2 shard j arrived (tier1),
    // [IF*K' + ib] fwd arrived (tier2), [IF*(K'+1) + ib] activation from the previous span
    // arrived (tier1, span > 0), [IF*(K'+2) + ib] next tokens from the last span arrived (span 0)
    uint32_t* flags = nullptr;
    std::vector<std::vector<void*>> fwd, pos; // tier1: [j][ib] its Tier-2 rank j's fwd / pos buffers
    std::vector<uint32_t*> rflags;            // tier1: [j] its Tier-2 rank j's flags; tier2: [r] Tier-1 rank r's
    std::vector<std::vector<void*>> bwd;      // tier2: [r][ib] Tier-1 rank r's bwd buffers (r < tp)
    uint32_t* nflags = nullptr;               // tier1 span s < n1-1: span s+1's flags
    std::vector<void*> nx, nss, npos;         // [ib] span s+1's x0 / ss0 / pos buffers
    uint32_t* fflags = nullptr;               // last span (n1 > 1): span 0's flags
    std::vector<void*> fnext;                 // [ib] span 0's next-token buffers
    std::vector<cudaStream_t> cs;             // copy streams (one per Tier-2 rank, + one to the next span)
    std::vector<cudaEvent_t> ev;              // per batch: message produced on the compute stream
    std::vector<uint32_t> seq;                // per batch: layer messages exchanged so far (both directions)
    std::vector<uint32_t> seqxo, seqxi;       // per batch: activations handed to / from the neighbour spans
    std::vector<uint32_t> seqt;               // per batch: token hand-backs sent (last span) / awaited (span 0)
    std::vector<void*> opened;                // IPC mappings
  } peer;
  ~gh_engine() {
    for (void* p : peer.opened) cudaIpcCloseMemHandle(p);
    for (auto s : peer.cs) cudaStreamDestroy(s);
    for (auto v : peer.ev) cudaEventDestroy(v);
    for (auto& b : batches) {
      if (b.graph) cudaGraphExecDestroy(b.graph);
      if (b.stream) cudaStreamDestroy(b.stream);
      if (b.done) cudaEventDestroy(b.done);
    }
    if (fork) cudaEventDestroy(fork);
    gh_tier1_destroy(t1);
    gh_tier2_destroy(t2);
  }
  int rows() const { return role == 2 ? my_cnt : (int)cfg.batch; }
  bool use_graph_any() const {
    for (auto& b : batches) if (b.graph) return true;
    return false;
  }
};

// Tier-1 stage calls on an in-flight batch's activation ping-pong (x0 / x1) with the sums of
// squares of the current activation threaded from its producer to its consumer (fused RMSNorm).
static gh_status act_embed(gh_engine* e, gh_engine::Batch& b, cudaStream_t st) {
  b.cur = 0;
  b.ss_slices[0] = 1;
  return t1_embed(e->t1, e->cfg.batch, b.tok, b.x0, b.ss0, st);
}
static gh_status act_pre(gh_engine* e, gh_engine::Batch& b, int l, cudaStream_t st) {
  return t1_pre(e->t1, l, e->cfg.batch, b.x(b.cur), SsRef{b.ss(b.cur), b.ss_slices[b.cur]}, b.pos, b.fwd, st);
}
static gh_status act_post(gh_engine* e, gh_engine::Batch& b, int l, cudaStream_t st, const PeerWait* pw = nullptr) {
  const int nx = b.cur ^ 1;
  GH_TRY(t1_post(e->t1, l, e->cfg.batch, b.bwd, b.x(nx), b.ss(nx), &b.ss_slices[nx], st, b.x(b.cur), pw));
  b.cur = nx;
  return GH_OK;
}
static gh_status act_classify(gh_engine* e, gh_engine::Batch& b, float* logits, cudaStream_t st) {
  if (!logits && e->keep_logits) logits = b.logits;
  if (b.sampling)  // logits are always written (the sampler reads them)
    return t1_classify(e->t1, e->cfg.batch, b.x(b.cur), SsRef{b.ss(b.cur), b.ss_slices[b.cur]},
                       logits ? logits : b.logits, b.next, st, b.inv_temp, b.seed, b.pos);
  return t1_classify(e->t1, e->cfg.batch, b.x(b.cur), SsRef{b.ss(b.cur), b.ss_slices[b.cur]}, logits, b.next, st);
}

extern "C" {
static gh_status peer_setup(gh_engine* e);
static gh_status peer_wait_tokens(gh_engine* e, int ib, cudaStream_t st);
}

static gh_status engine_layer_loop_colocated(gh_engine* e, gh_engine::Batch& b, bool want_logits, cudaStream_t st) {
  const Shape& s = e->sh;
  const uint32_t B = e->cfg.batch;
  GH_TRY(act_embed(e, b, st));
  for (int l = 0; l < s.N; ++l) {
    GH_TRY(act_pre(e, b, l, st));
    const Weight& wo = e->t1->layers[l].o;
    if (e->cfg.prefill) GH_TRY(t2_append(e->t2, l, B, b.slot, b.pos, b.fwd, st));  // rows may share a prompt
    // predecessor: the QKV GEMM (or the append kernel with prefill rows, which writes the arena)
    GH_TRY(t2_attend(e->t2, l, B, b.slot, b.pos, b.fwd, b.bwd, st, wo.ptr, gh_tier1::prefetch_bytes(&wo),
                     e->cfg.prefill ? 0 : 1));
    GH_TRY(act_post(e, b, l, st));
  }
  return act_classify(e, b, want_logits ? b.logits : nullptr, st);
}

extern "C" {

gh_status gh_engine_create(const gh_engine_config* cfg, gh_comm* comm, gh_engine** out) {
  if (!cfg || !out) return fail(GH_EINVAL, "null argument");
  *out = nullptr;
  auto e = std::make_unique<gh_engine>();
  e->cfg = *cfg;
  GH_TRY(Shape::from(&cfg->spec, &e->sh));
  if (cfg->batch == 0 || cfg->inflight == 0) return fail(GH_EINVAL, "batch and inflight must be >= 1");
  if (gh_device_count() <= cfg->device) return fail(GH_ECUDA, "no CUDA device " + std::to_string(cfg->device));
  GH_CUDA(cudaSetDevice(cfg->device));
  const Shape& s = e->sh;
  e->comm = comm;
  const int world = comm ? comm->nranks : 1;
  const int rank = comm ? comm->rank : 0;
  e->l0 = 0;
  e->l1 = s.N;
  e->tp = cfg->tier1_tp > 1 ? (int)cfg->tier1_tp : 1;
  if (world == 1) {
    if (e->tp > 1) return fail(GH_EINVAL, "tier1_tp > 1 needs a tier split (world >= tier1_tp + 1)");
    e->role = 0;
  } else if (e->tp > 1) {
    // Tier-1 tensor parallelism: ranks 0..tp-1 hold a head / hidden-unit slice of every layer,
    // ranks tp.. are the K' Tier-2 ranks (each holds all heads of its prompt shard)
    if (cfg->tier1_ranks > 1) return fail(GH_EUNSUPPORTED, "tier1_tp and tier1_ranks (pipeline spans) together");
    if (world <= e->tp) return fail(GH_EINVAL, "world size must be tier1_tp + K' with K' >= 1");
    if (cfg->transport == GH_TRANSPORT_NCCL) return fail(GH_EUNSUPPORTED, "tensor parallelism needs the peer transport");
    if (cfg->prefill) return fail(GH_EUNSUPPORTED, "chunked prefill rows: no tensor parallelism");
    if (e->tp > kMaxTp) return fail(GH_EUNSUPPORTED, "tier1_tp <= 4");
    if (s.db != 2 || s.dh != 128 || s.Hkv % e->tp)
      return fail(GH_EUNSUPPORTED, "tensor parallelism: bf16, head dim 128, kv heads divisible by tier1_tp");
    e->kp = world - e->tp;
    e->role = rank < e->tp ? 1 : 2;
    e->shard = rank < e->tp ? 0 : rank - e->tp;
    if ((int)cfg->batch < e->kp) return fail(GH_EINVAL, "batch smaller than the number of Tier-2 ranks");
    std::vector<uint64_t> off(e->kp), cnt(e->kp);  // balanced shards (analytic.cpp:119)
    GH_TRY(gh_shard_plan(cfg->batch, e->kp, off.data(), cnt.data()));
    for (int j = 0; j < e->kp; ++j) {
      e->shard_off.push_back((int)off[j]);
      e->shard_cnt.push_back((int)cnt[j]);
    }
    if (e->role == 2) e->my_cnt = e->shard_cnt[e->shard];
  } else {
    e->n1 = cfg->tier1_ranks > 1 ? (int)cfg->tier1_ranks : 1;
    if (world <= e->n1 || (world - e->n1) % e->n1)
      return fail(GH_EINVAL, "world size must be tier1_ranks * (1 + K') with K' >= 1");
    if (e->n1 > s.N) return fail(GH_EINVAL, "more Tier-1 spans than layers");
    if (e->n1 > 1 && cfg->transport == GH_TRANSPORT_NCCL)
      return fail(GH_EUNSUPPORTED, "Tier-1 pipeline stages need the peer transport");
    if (cfg->prefill && cfg->tier1_ranks > 1)
      return fail(GH_EUNSUPPORTED, "chunked prefill rows: one Tier-1 rank");
    e->kp = (world - e->n1) / e->n1;
    e->role = rank < e->n1 ? 1 : 2;
    e->span = rank < e->n1 ? rank : (rank - e->n1) / e->kp;
    e->shard = rank < e->n1 ? 0 : (rank - e->n1) % e->kp;
    std::vector<uint64_t> spans(e->n1);  // contiguous layer blocks, remainder to low ranks (optimizer.cpp:116-123)
    GH_TRY(gh_layer_spans((uint64_t)s.N, (uint64_t)e->n1, spans.data()));
    for (int sp = 0; sp < e->span; ++sp) e->l0 += (int)spans[sp];
    e->l1 = e->l0 + (int)spans[e->span];
    if ((int)cfg->batch < e->kp) return fail(GH_EINVAL, "batch smaller than the number of Tier-2 ranks");
    std::vector<uint64_t> off(e->kp), cnt(e->kp);  // balanced shards (analytic.cpp:119)
    GH_TRY(gh_shard_plan(cfg->batch, e->kp, off.data(), cnt.data()));
    for (int j = 0; j < e->kp; ++j) {
      e->shard_off.push_back((int)off[j]);
      e->shard_cnt.push_back((int)cnt[j]);
    }
    if (e->role == 2) e->my_cnt = e->shard_cnt[e->shard];
  }
  {  // the decomposition is exactly the host-side gh_engine_layout (tested on CPU at world 8)
    gh_rank_layout lay;
    GH_TRY(gh_engine_layout((uint32_t)world, (uint32_t)rank, cfg->tier1_ranks, cfg->tier1_tp, (uint64_t)s.N,
                            cfg->batch, &lay));
    const bool same = lay.role == e->role && (e->role == 0 || (lay.span == e->span && (int)lay.kp == e->kp &&
                      (int)lay.layer_begin == e->l0 && (int)lay.layer_end == e->l1 &&
                      (e->role != 2 || (lay.shard == e->shard && (int)lay.row_off == e->shard_off[e->shard] &&
                                        (int)lay.row_cnt == e->my_cnt))));
    if (!same) return fail(GH_EINTERNAL, "engine layout disagrees with gh_engine_layout");
  }
  const int R = e->rows();
  if (e->role != 2)
    GH_TRY(tier1_create(&cfg->spec, cfg->device, (uint32_t)e->l0, (uint32_t)e->l1, cfg->weight_seed, cfg->batch,
                        e->tp, e->tp > 1 ? rank : 0, &e->t1));
  if (e->role != 1) {
    uint32_t need = (uint32_t)R * cfg->inflight;
    uint32_t n_slots = cfg->n_slots ? cfg->n_slots : need;
    if (n_slots < need && !cfg->prefill)  // prefill rows share slots: any n_slots >= 1
      return fail(GH_EINFEASIBLE, "n_slots smaller than batch * inflight (binding constraint: memory)");
    GH_TRY(tier2_create(&cfg->spec, cfg->device, (uint32_t)e->l0, (uint32_t)e->l1, n_slots, cfg->kv_pages, &e->t2));
  }
  GH_CUDA(cudaEventCreateWithFlags(&e->fork, cudaEventDisableTiming));
  e->batches.resize(cfg->inflight);
  for (uint32_t ib = 0; ib < cfg->inflight; ++ib) {
    auto& b = e->batches[ib];
    void* p;
    GH_TRY(dev_alloc(e->mem, (size_t)R * 4, &p)); b.tok = (int32_t*)p;
    GH_TRY(dev_alloc(e->mem, (size_t)R * 4, &p)); b.pos = (int32_t*)p;
    GH_TRY(dev_alloc(e->mem, (size_t)R * 4, &p)); b.next = (int32_t*)p;
    GH_TRY(dev_alloc(e->mem, (size_t)R * 4, &p)); b.slot = (uint32_t*)p;
    GH_TRY(dev_alloc(e->mem, (size_t)R * 4, &p)); b.inv_temp = (float*)p;
    GH_CUDA(cudaMemset(p, 0, (size_t)R * 4));  // greedy until gh_engine_set_sampling
    GH_TRY(dev_alloc(e->mem, (size_t)R * 4, &p)); b.seed = (uint32_t*)p;
    GH_CUDA(cudaMemset(p, 0, (size_t)R * 4));
    GH_TRY(dev_alloc(e->mem, (size_t)R * s.D * s.db, &b.x0));
    GH_TRY(dev_alloc(e->mem, (size_t)R * s.D * s.db, &b.x1));
    GH_TRY(dev_alloc(e->mem, (size_t)R * e->fwd_w() * s.db, &b.fwd));
    GH_TRY(dev_alloc(e->mem, (size_t)R * e->bwd_w() * s.db, &b.bwd));
    {
      const size_t nss = (size_t)(s.D + 127) / 128 * 8 * R;  // W2 output tiles x max cluster size
      GH_TRY(dev_alloc(e->mem, nss * sizeof(float), &p)); b.ss0 = (float*)p;
      GH_TRY(dev_alloc(e->mem, nss * sizeof(float), &p)); b.ss1 = (float*)p;
    }
    if (e->role != 2) { GH_TRY(dev_alloc(e->mem, (size_t)R * s.V * 4, &p)); b.logits = (float*)p; }
    std::vector<uint32_t> slots(R);
    for (int i = 0; i < R; ++i) slots[i] = e->t2 ? (ib * R + i) % e->t2->n_slots : ib * R + i;
    GH_CUDA(cudaMemcpy(b.slot, slots.data(), R * 4, cudaMemcpyHostToDevice));
    b.slot_host = slots;
    GH_CUDA(cudaMemset(b.tok, 0, R * 4));
    GH_CUDA(cudaMemset(b.pos, 0, R * 4));
    GH_CUDA(cudaMemset(b.next, 0, R * 4));
    GH_CUDA(cudaStreamCreateWithFlags(&b.stream, cudaStreamNonBlocking));
    GH_CUDA(cudaEventCreateWithFlags(&b.done, cudaEventDisableTiming));
  }
  GH_CUDA(cudaDeviceSynchronize());
  if (e->role != 0 && cfg->transport != GH_TRANSPORT_NCCL) GH_TRY(peer_setup(e.get()));
  if ((cfg->transport == GH_TRANSPORT_PEER || e->n1 > 1 || e->tp > 1) && e->role != 0 && !e->peer.on)
    return fail(GH_EUNSUPPORTED, "peer transport requested but not available on every rank");
  *out = e.release();
  return GH_OK;
}

int gh_engine_transport(const gh_engine* e) {
  if (!e || e->role == 0) return -1;
  return e->peer.on ? GH_TRANSPORT_PEER : GH_TRANSPORT_NCCL;
}

gh_status gh_engine_destroy(gh_engine* e) {
  delete e;
  return GH_OK;
}

int gh_engine_role(const gh_engine* e) { return e ? e->role : -1; }
gh_tier1* gh_engine_tier1(gh_engine* e) { return e ? e->t1 : nullptr; }

gh_status gh_engine_read_next(gh_engine* e, uint32_t ib, int32_t* next_host) {
  if (!e || ib >= e->batches.size() || !next_host) return fail(GH_EINVAL, "bad argument");
  if (e->role == 2) return fail(GH_EINVAL, "Tier-2 ranks hold no token state");
  GH_CUDA(cudaSetDevice(e->cfg.device));
  GH_CUDA(cudaDeviceSynchronize());
  GH_CUDA(cudaMemcpy(next_host, e->batches[ib].next, (size_t)e->cfg.batch * 4, cudaMemcpyDeviceToHost));
  return GH_OK;
}

gh_status gh_engine_keep_logits(gh_engine* e, int keep) {
  if (!e) return fail(GH_EINVAL, "null engine");
  if (e->role == 2) return fail(GH_EINVAL, "Tier-2 ranks run no classifier");
  if (e->use_graph_any()) return fail(GH_EUNSUPPORTED, "set before the first step (the CUDA graph is captured then)");
  e->keep_logits = keep != 0;
  return GH_OK;
}

gh_status gh_engine_read_logits(gh_engine* e, uint32_t ib, float* logits_host) {
  if (!e || ib >= e->batches.size() || !logits_host) return fail(GH_EINVAL, "bad argument");
  if (e->role == 2 || !e->batches[ib].logits) return fail(GH_EINVAL, "this rank holds no logits");
  GH_CUDA(cudaSetDevice(e->cfg.device));
  GH_CUDA(cudaDeviceSynchronize());
  GH_CUDA(cudaMemcpy(logits_host, e->batches[ib].logits, (size_t)e->cfg.batch * e->sh.V * 4, cudaMemcpyDeviceToHost));
  return GH_OK;
}

gh_status gh_engine_advance(gh_engine* e, uint32_t ib, int inc, void* stream) {
  if (!e || ib >= e->batches.size()) return fail(GH_EINVAL, "bad engine / batch index");
  if (e->role == 2) return fail(GH_EINVAL, "Tier-2 ranks hold no token state");
  auto& b = e->batches[ib];
  if (e->role == 1 && e->span > 0) return GH_OK;  // later spans take tokens / positions from the hand-off
  if (e->role == 1 && e->n1 > 1 && e->peer.on) {  // deferred to the batch's next step (split_step_peer)
    b.adv_pending = true;
    b.adv_inc += inc;
    return GH_OK;
  }
  GH_CUDA(cudaSetDevice(e->cfg.device));
  GH_TRY(peer_wait_tokens(e, (int)ib, (cudaStream_t)stream));  // first span: the last span's next tokens
  GH_CUDA(launch_advance(b.tok, b.next, b.pos, (int)e->cfg.batch, inc, (cudaStream_t)stream));
  return GH_OK;
}
gh_tier2* gh_engine_tier2(gh_engine* e) { return e ? e->t2 : nullptr; }

gh_status gh_engine_kv_map(gh_engine* e, uint32_t slot, uint32_t n_positions) {
  if (!e) return fail(GH_EINVAL, "null engine");
  if (!e->t2) return fail(GH_EUNSUPPORTED, "this rank holds no KV (Tier-1 role)");
  return gh_tier2_map(e->t2, slot, n_positions, nullptr);
}

gh_status gh_engine_kv_swap(gh_engine* e, uint32_t slot, uint32_t n_positions, void* host, int to_host) {
  if (!e) return fail(GH_EINVAL, "null engine");
  if (!e->t2) return fail(GH_EUNSUPPORTED, "this rank holds no KV (Tier-1 role)");
  GH_CUDA(cudaSetDevice(e->t2->device));
  GH_CUDA(cudaDeviceSynchronize());  // the engine's queued steps read / write the arena
  return gh_tier2_kv_swap(e->t2, slot, n_positions, host, to_host, nullptr);
}

uint64_t gh_engine_kv_swap_bytes(const gh_engine* e, uint32_t n_positions) {
  return e && e->t2 ? gh_tier2_kv_swap_bytes(e->t2, n_positions) : 0;
}

gh_status gh_engine_set_sampling(gh_engine* e, uint32_t ib, const float* temperature_host, const uint32_t* seed_host) {
  if (!e || ib >= e->batches.size()) return fail(GH_EINVAL, "bad engine / batch index");
  if (e->role == 2) return GH_OK;  // Tier-2 ranks do not classify
  if (!temperature_host || !seed_host) return fail(GH_EINVAL, "null temperature / seed");
  auto& b = e->batches[ib];
  const int R = e->rows();
  std::vector<float> inv(R);
  for (int i = 0; i < R; ++i) {
    if (!(temperature_host[i] >= 0.f)) return fail(GH_EINVAL, "temperature must be >= 0");
    inv[i] = temperature_host[i] > 0.f ? 1.0f / temperature_host[i] : 0.f;
  }
  GH_CUDA(cudaSetDevice(e->cfg.device));
  GH_CUDA(cudaDeviceSynchronize());  // no step in flight reads the old values
  GH_CUDA(cudaMemcpy(b.inv_temp, inv.data(), (size_t)R * 4, cudaMemcpyHostToDevice));
  GH_CUDA(cudaMemcpy(b.seed, seed_host, (size_t)R * 4, cudaMemcpyHostToDevice));
  bool any = false;
  for (float v : inv) any = any || v > 0.f;
  if (any != b.sampling) {
    b.sampling = any;
    if (b.graph) { cudaGraphExecDestroy(b.graph); b.graph = nullptr; }  // recaptured on the next step
  }
  return GH_OK;
}

gh_status gh_engine_shard(const gh_engine* e, int* index, uint32_t* off, uint32_t* cnt, uint32_t* kp) {
  if (!e) return fail(GH_EINVAL, "null engine");
  const bool t2 = e->role == 2;
  if (index) *index = t2 ? e->shard : -1;
  if (off) *off = t2 ? (uint32_t)e->shard_off[e->shard] : 0u;
  if (cnt) *cnt = t2 ? (uint32_t)e->my_cnt : e->cfg.batch;
  if (kp) *kp = (uint32_t)e->kp;
  return GH_OK;
}

gh_status gh_engine_set_slots(gh_engine* e, uint32_t ib, const uint32_t* slot_host) {
  if (!e || !slot_host || ib >= e->batches.size()) return fail(GH_EINVAL, "bad engine / batch index / slots");
  if (e->role == 1) return GH_OK;  // Tier-1 holds no KV: the Tier-2 ranks take their rows' slots
  auto& b = e->batches[ib];
  const int R = e->rows();          // Tier-2: the rows of this rank's shard (gh_engine_shard)
  for (int i = 0; i < R; ++i)
    if (slot_host[i] >= e->t2->n_slots)
      return fail(GH_EINVAL, "slot " + std::to_string(slot_host[i]) + " >= n_slots " + std::to_string(e->t2->n_slots));
  GH_CUDA(cudaSetDevice(e->cfg.device));
  GH_CUDA(cudaDeviceSynchronize());  // no step in flight reads the old slots
  GH_CUDA(cudaMemcpy(b.slot, slot_host, (size_t)R * 4, cudaMemcpyHostToDevice));
  b.slot_host.assign(slot_host, slot_host + R);
  return GH_OK;
}

gh_status gh_engine_kv_unmap(gh_engine* e, uint32_t slot) {
  if (!e) return fail(GH_EINVAL, "null engine");
  if (!e->t2) return fail(GH_EUNSUPPORTED, "this rank holds no KV (Tier-1 role)");
  return gh_tier2_unmap(e->t2, slot);
}

gh_status gh_engine_io(gh_engine* e, uint32_t ib, int32_t** tok, int32_t** pos, uint32_t** slot, int32_t** next) {
  if (!e || ib >= e->batches.size()) return fail(GH_EINVAL, "bad engine / batch index");
  auto& b = e->batches[ib];
  if (tok) *tok = b.tok;
  if (pos) *pos = b.pos;
  if (slot) *slot = b.slot;
  if (next) *next = b.next;
  return GH_OK;
}

// --- tier-split body for one in-flight batch, issued on the batch stream.
// Tier-1:  for each layer: F1 -> send shards [x|q|k|v] -> recv shards [x|attn] -> F3
// Tier-2:  for each layer: recv shard -> F2 -> send shard
static gh_status split_begin(gh_engine* e, gh_engine::Batch& b, ncclComm_t comm, cudaStream_t st) {
  auto& api = nccl();
  if (e->role == 1) {
    // step header: positions of each shard (Dispatcher batch state)
    GH_NCCL(api.GroupStart());
    for (int j = 0; j < e->kp; ++j)
      GH_NCCL(api.Send(b.pos + e->shard_off[j], e->shard_cnt[j], ncclInt32, j + 1, comm, st));
    GH_NCCL(api.GroupEnd());
    GH_TRY(act_embed(e, b, st));
  } else {
    GH_NCCL(api.Recv(b.pos, e->my_cnt, ncclInt32, 0, comm, st));
  }
  return GH_OK;
}

static gh_status split_layer(gh_engine* e, gh_engine::Batch& b, ncclComm_t comm, int l, cudaStream_t st) {
  auto& api = nccl();
  const Shape& s = e->sh;
  const size_t fwd_row = (size_t)s.ld_fwd() * s.db, bwd_row = (size_t)s.ld_bwd() * s.db;
  if (e->role == 1) {
    GH_TRY(act_pre(e, b, l, st));
    GH_NCCL(api.GroupStart());
    for (int j = 0; j < e->kp; ++j)
      GH_NCCL(api.Send((char*)b.fwd + e->shard_off[j] * fwd_row, e->shard_cnt[j] * fwd_row, ncclUint8, j + 1, comm, st));
    GH_NCCL(api.GroupEnd());
    GH_NCCL(api.GroupStart());
    for (int j = 0; j < e->kp; ++j)
      GH_NCCL(api.Recv((char*)b.bwd + e->shard_off[j] * bwd_row, e->shard_cnt[j] * bwd_row, ncclUint8, j + 1, comm, st));
    GH_NCCL(api.GroupEnd());
    GH_TRY(act_post(e, b, l, st));
  } else {
    GH_NCCL(api.Recv(b.fwd, e->my_cnt * fwd_row, ncclUint8, 0, comm, st));
    if (e->cfg.prefill) GH_TRY(t2_append(e->t2, l, e->my_cnt, b.slot, b.pos, b.fwd, st));
    GH_TRY(gh_tier2_attend(e->t2, l, e->my_cnt, b.slot, b.pos, b.fwd, b.bwd, st));
    GH_NCCL(api.Send(b.bwd, e->my_cnt * bwd_row, ncclUint8, 0, comm, st));
  }
  return GH_OK;
}

gh_status gh_engine_step_device(gh_engine* e, uint32_t ib, void* stream) {
  if (!e || ib >= e->batches.size()) return fail(GH_EINVAL, "bad engine / batch index");
  auto& b = e->batches[ib];
  cudaStream_t st = (cudaStream_t)stream;
  GH_CUDA(cudaSetDevice(e->cfg.device));
  if (e->role == 0) {
    if (e->cfg.use_graph) {
      if (!b.graph) {
        cudaStream_t cs;
        GH_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        GH_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        gh_status r = engine_layer_loop_colocated(e, b, false, cs);
        cudaGraph_t g = nullptr;
        cudaError_t ce = cudaStreamEndCapture(cs, &g);
        cudaStreamDestroy(cs);
        if (r != GH_OK) { if (g) cudaGraphDestroy(g); return r; }
        GH_CUDA(ce);
        cudaError_t ie = cudaGraphInstantiate(&b.graph, g, 0);
        cudaGraphDestroy(g);
        GH_CUDA(ie);
      }
      GH_CUDA(cudaGraphLaunch(b.graph, st));
      return GH_OK;
    }
    return engine_layer_loop_colocated(e, b, false, st);
  }
  if (e->n1 > 1 || e->tp > 1)
    return fail(GH_EUNSUPPORTED, "Tier-1 pipeline stages / tensor parallelism: use gh_engine_step_all / step_all_host");
  ncclComm_t comm = e->comm->comms[0];
  GH_TRY(split_begin(e, b, comm, st));
  for (int l = 0; l < e->sh.N; ++l) GH_TRY(split_layer(e, b, comm, l, st));
  if (e->role == 1) GH_TRY(act_classify(e, b, nullptr, st));
  return GH_OK;
}

// All in-flight batches; in split mode the batches are interleaved layer by layer on their own
// streams so that Tier-1 compute of one batch overlaps Tier-2 attention of another.
// ---- tier split, all in-flight batches, one stream per rank, software-pipelined.
// Tier-1 issue order: embed_b, pre_b(0) for every batch b, then for each layer l and batch b:
//   [group: pending sends + recv_b(l)] -> post_b(l) -> pre_b(l+1) (its send becomes pending)
// Tier-2: [group: positions + recv_0(0)] -> for each (l, b): attend_b(l) -> [group: send_b(l) +
// recv of the next (batch, layer)].  Every send is grouped with the recv the issuing rank needs
// next, so the rendezvous of both directions progresses together (no deadlock), and while
// Tier-2 attends batch b Tier-1 runs F3 / F1 of the other batches.  A single stream means no
// NCCL kernel ever spins next to a persistent GEMM / attention grid on the same GPU.
static gh_status t1_group(gh_engine* e, ncclComm_t comm, cudaStream_t st, std::vector<int>& pending_send,
                          int recv_ib, bool pos_header) {
  auto& api = nccl();
  const Shape& s = e->sh;
  const size_t fwd_row = (size_t)s.ld_fwd() * s.db, bwd_row = (size_t)s.ld_bwd() * s.db;
  GH_NCCL(api.GroupStart());
  if (pos_header)
    for (auto& b : e->batches)
      for (int j = 0; j < e->kp; ++j)
        GH_NCCL(api.Send(b.pos + e->shard_off[j], e->shard_cnt[j], ncclInt32, j + 1, comm, st));
  for (int ib : pending_send) {
    auto& b = e->batches[ib];
    for (int j = 0; j < e->kp; ++j)
      GH_NCCL(api.Send((char*)b.fwd + e->shard_off[j] * fwd_row, e->shard_cnt[j] * fwd_row, ncclUint8, j + 1,
                       comm, st));
  }
  if (recv_ib >= 0) {
    auto& b = e->batches[recv_ib];
    for (int j = 0; j < e->kp; ++j)
      GH_NCCL(api.Recv((char*)b.bwd + e->shard_off[j] * bwd_row, e->shard_cnt[j] * bwd_row, ncclUint8, j + 1,
                       comm, st));
  }
  GH_NCCL(api.GroupEnd());
  pending_send.clear();
  return GH_OK;
}

static gh_status t2_group(gh_engine* e, ncclComm_t comm, cudaStream_t st, int send_ib, int recv_ib,
                          bool pos_header) {
  auto& api = nccl();
  const Shape& s = e->sh;
  const size_t fwd_row = (size_t)s.ld_fwd() * s.db, bwd_row = (size_t)s.ld_bwd() * s.db;
  GH_NCCL(api.GroupStart());
  if (pos_header)
    for (auto& b : e->batches) GH_NCCL(api.Recv(b.pos, e->my_cnt, ncclInt32, 0, comm, st));
  if (send_ib >= 0) GH_NCCL(api.Send(e->batches[send_ib].bwd, e->my_cnt * bwd_row, ncclUint8, 0, comm, st));
  if (recv_ib >= 0) GH_NCCL(api.Recv(e->batches[recv_ib].fwd, e->my_cnt * fwd_row, ncclUint8, 0, comm, st));
  GH_NCCL(api.GroupEnd());
  return GH_OK;
}

// ---- peer transport (see gh_engine::Peer)
namespace {
typedef CUresult (*PFN_streamValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
struct MemOps {
  PFN_streamValue32 wait = nullptr, write = nullptr;
};
MemOps& memops() {
  static MemOps m;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      m.wait = (PFN_streamValue32)p;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      m.write = (PFN_streamValue32)p;
  });
  return m;
}
}  // namespace

#define GH_CU(call)                                                                           \
  do {                                                                                        \
    CUresult r_ = (call);                                                                     \
    if (r_ != CUDA_SUCCESS) return fail(GH_ECUDA, std::string(#call) + " failed: " + std::to_string((int)r_)); \
  } while (0)

// Collective over all ranks of the engine's communicator: export this rank's receive buffers as
// CUDA IPC handles, all-gather them, map the peers' buffers.  The transport is enabled only if
// every rank mapped every buffer it needs (all-reduce min of the outcome), so all ranks agree.
// Exported slots per rank: [flags, fwd x IF, pos x IF, bwd x IF, x0 x IF, ss0 x IF, next x IF].
static gh_status peer_setup(gh_engine* e) {
  auto& api = nccl();
  auto& P = e->peer;
  const int IF = (int)e->batches.size(), kp = e->kp, world = e->comm->nranks, rank = e->comm->rank;
  const int n1 = e->n1, tp = e->tp;
  const int nslot = 3 + 6 * IF;
  auto slot_fwd = [&](int ib) { return 1 + ib; };
  auto slot_pos = [&](int ib) { return 1 + IF + ib; };
  auto slot_bwd = [&](int ib) { return 1 + 2 * IF + ib; };
  auto slot_x0 = [&](int ib) { return 1 + 3 * IF + ib; };
  auto slot_ss0 = [&](int ib) { return 1 + 4 * IF + ib; };
  auto slot_next = [&](int ib) { return 1 + 5 * IF + ib; };
  const int slot_tpb = 1 + 6 * IF;  // TP all-reduce receive buffers (2 parities)
  ncclComm_t comm = e->comm->comms[0];
  void* p;
  const size_t nflags = (size_t)IF * (kp + tp + 2);
  GH_TRY(dev_alloc(e->mem, nflags * 4, &p));
  P.flags = (uint32_t*)p;
  GH_CUDA(cudaMemset(P.flags, 0, nflags * 4));
  std::vector<cudaIpcMemHandle_t> mine(nslot);
  memset(mine.data(), 0, nslot * sizeof(cudaIpcMemHandle_t));
  int ok = memops().wait && memops().write;
  auto get = [&](int i, void* ptr) {
    if (ptr && cudaIpcGetMemHandle(&mine[i], ptr) != cudaSuccess) { cudaGetLastError(); ok = 0; }
  };
  get(0, P.flags);
  for (int ib = 0; ib < IF; ++ib) {
    auto& b = e->batches[ib];
    get(slot_fwd(ib), b.fwd);
    get(slot_pos(ib), b.pos);
    get(slot_bwd(ib), b.bwd);
    if (e->role == 1) {
      get(slot_x0(ib), b.x0);
      if (b.ss0) get(slot_ss0(ib), b.ss0);
      get(slot_next(ib), b.next);
    }
  }
  if (e->role == 1 && tp > 1) {
    get(slot_tpb, e->t1->tpc.buf[0]);
    get(slot_tpb + 1, e->t1->tpc.buf[1]);
  }
  const size_t rec = nslot * sizeof(cudaIpcMemHandle_t);
  void *dmine, *dall, *dok;
  GH_TRY(dev_alloc(e->mem, rec, &dmine));
  GH_TRY(dev_alloc(e->mem, rec * world, &dall));
  GH_TRY(dev_alloc(e->mem, 4, &dok));
  cudaStream_t st;
  GH_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  GH_CUDA(cudaMemcpy(dmine, mine.data(), rec, cudaMemcpyHostToDevice));
  GH_NCCL(api.AllGather(dmine, dall, rec, ncclUint8, comm, st));
  GH_CUDA(cudaStreamSynchronize(st));
  std::vector<cudaIpcMemHandle_t> all((size_t)nslot * world);
  GH_CUDA(cudaMemcpy(all.data(), dall, rec * world, cudaMemcpyDeviceToHost));
  auto open = [&](int r, int i) -> void* {
    void* q = nullptr;
    if (!ok) return nullptr;
    if (cudaIpcOpenMemHandle(&q, all[(size_t)r * nslot + i], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      ok = 0;
      return nullptr;
    }
    P.opened.push_back(q);
    return q;
  };
  if (e->role == 1) {
    P.fwd.assign(kp, std::vector<void*>(IF, nullptr));
    P.pos.assign(kp, std::vector<void*>(IF, nullptr));
    for (int j = 0; j < kp; ++j) {
      const int r = e->t2_rank(e->span, j);
      P.rflags.push_back((uint32_t*)open(r, 0));
      for (int ib = 0; ib < IF; ++ib) { P.fwd[j][ib] = open(r, slot_fwd(ib)); P.pos[j][ib] = open(r, slot_pos(ib)); }
    }
    if (e->span + 1 < n1) {  // activation hand-off to the next span (the PP message is [x], netmodel.cpp:22)
      const int r = e->span + 1;
      P.nflags = (uint32_t*)open(r, 0);
      for (int ib = 0; ib < IF; ++ib) {
        P.nx.push_back(open(r, slot_x0(ib)));
        P.nss.push_back(e->batches[ib].ss0 ? open(r, slot_ss0(ib)) : nullptr);
        P.npos.push_back(open(r, slot_pos(ib)));
      }
    }
    if (n1 > 1 && e->span == n1 - 1) {  // next tokens back to the first span (it owns the embedding)
      P.fflags = (uint32_t*)open(0, 0);
      for (int ib = 0; ib < IF; ++ib) P.fnext.push_back(open(0, slot_next(ib)));
    }
    if (tp > 1) {  // the other TP ranks' all-reduce receive buffers
      auto& c = e->t1->tpc;
      for (int q = 0; q < tp; ++q) {
        if (q == rank) {
          c.peer_buf[0][q] = c.buf[0];
          c.peer_buf[1][q] = c.buf[1];
        } else {
          c.peer_buf[0][q] = (float*)open(q, slot_tpb);
          c.peer_buf[1][q] = (float*)open(q, slot_tpb + 1);
        }
      }
    }
  } else if (tp > 1) {  // every TP Tier-1 rank receives its head block of the attention output
    P.bwd.assign(tp, std::vector<void*>(IF, nullptr));
    for (int r = 0; r < tp; ++r) {
      P.rflags.push_back((uint32_t*)open(r, 0));
      for (int ib = 0; ib < IF; ++ib) P.bwd[r][ib] = open(r, slot_bwd(ib));
    }
  } else {
    P.rflags.push_back((uint32_t*)open(e->span, 0));
    P.bwd.assign(1, std::vector<void*>());
    for (int ib = 0; ib < IF; ++ib) P.bwd[0].push_back(open(e->span, slot_bwd(ib)));
  }
  (void)rank;
  GH_CUDA(cudaMemcpy(dok, &ok, 4, cudaMemcpyHostToDevice));
  GH_NCCL(api.AllReduce(dok, dok, 1, ncclInt32, ncclMin, comm, st));
  GH_CUDA(cudaStreamSynchronize(st));
  GH_CUDA(cudaMemcpy(&ok, dok, 4, cudaMemcpyDeviceToHost));
  cudaStreamDestroy(st);
  if (!ok) {
    for (void* q : P.opened) cudaIpcCloseMemHandle(q);
    P.opened.clear();
    return GH_OK;  // NCCL send/recv transport
  }
  const int ncs = e->role == 1 ? kp + 1 : std::max(1, tp);
  for (int j = 0; j < ncs; ++j) {
    cudaStream_t c;
    GH_CUDA(cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking));
    P.cs.push_back(c);
  }
  for (int ib = 0; ib < IF; ++ib) {
    cudaEvent_t v;
    GH_CUDA(cudaEventCreateWithFlags(&v, cudaEventDisableTiming));
    P.ev.push_back(v);
  }
  P.seq.assign(IF, 0);
  P.seqxo.assign(IF, 0);
  P.seqxi.assign(IF, 0);
  P.seqt.assign(IF, 0);
  P.on = true;
  if (e->role == 1 && tp > 1) e->t1->tpc.ready = true;
  return GH_OK;
}

// flag word offsets (gh_engine::Peer::flags)
//   [ib*K' + j]                   tier1: the attention output of Tier-2 shard j arrived
//   [IF*K' + ib*tp + r]           tier2: the fwd head block of Tier-1 rank r arrived (tp = 1: r = 0)
//   [IF*(K'+tp) + ib]             tier1 span > 0: the previous span's activation arrived
//   [IF*(K'+tp+1) + ib]           tier1 span 0: the last span's next tokens arrived
static uint32_t f_bwd(const gh_engine* e, int ib, int j) { return (uint32_t)(ib * e->kp + j); }
static uint32_t f_fwd(const gh_engine* e, int ib, int r) {
  return (uint32_t)(e->batches.size() * e->kp + ib * e->tp + r);
}
static uint32_t f_x(const gh_engine* e, int ib) { return (uint32_t)(e->batches.size() * (e->kp + e->tp) + ib); }
static uint32_t f_tok(const gh_engine* e, int ib) { return (uint32_t)(e->batches.size() * (e->kp + e->tp + 1) + ib); }

// Tier-1: copy batch ib's fwd message shards (and, at the first layer of a step, its positions)
// into every Tier-2 rank of this span, then publish the sequence number in that rank's flag word.
static gh_status peer_send_fwd(gh_engine* e, int ib, bool with_pos, cudaStream_t st) {
  auto& P = e->peer;
  auto& b = e->batches[ib];
  const size_t fwd_row = (size_t)e->fwd_w() * e->sh.db;  // this rank's (head block of the) row
  const int me = e->tp > 1 ? e->comm->rank : 0;           // TP rank: block index at the Tier-2
  const uint32_t sq = ++P.seq[ib];
  GH_CUDA(cudaEventRecord(P.ev[ib], st));
  for (int j = 0; j < e->kp; ++j) {
    cudaStream_t c = P.cs[j];
    GH_CUDA(cudaStreamWaitEvent(c, P.ev[ib], 0));
    if (with_pos && me == 0)
      GH_CUDA(cudaMemcpyAsync(P.pos[j][ib], b.pos + e->shard_off[j], (size_t)e->shard_cnt[j] * 4, cudaMemcpyDeviceToDevice, c));
    // head block `me` of the Tier-2's [tp][cnt][row/tp] buffer (tp = 1: the plain rows)
    GH_CUDA(cudaMemcpyAsync((char*)P.fwd[j][ib] + (size_t)me * e->shard_cnt[j] * fwd_row,
                            (char*)b.fwd + e->shard_off[j] * fwd_row, e->shard_cnt[j] * fwd_row,
                            cudaMemcpyDeviceToDevice, c));
    GH_CU(memops().write((CUstream)c, (CUdeviceptr)(P.rflags[j] + f_fwd(e, ib, me)), sq, CU_STREAM_WRITE_VALUE_DEFAULT));
  }
  return GH_OK;
}

// Sums-of-squares slices the last W2 epilogue of a span wrote (the next span's first QKV applies
// its RMSNorm from them, exactly as inside one span); 0 = the unfused path.
static int handoff_ss_slices(gh_engine* e) {
  const Shape& s = e->sh;
  const int B = (int)e->cfg.batch;
  if (s.db != 2 || B > kFusedNormMaxBatch) return 0;
  return e->t1->plan(s.D, s.Dh, B).slices();
}

// Tier-1 span s -> s+1: the activation x (+ its sums of squares and the positions) of batch ib.
static gh_status peer_send_next_span(gh_engine* e, int ib, cudaStream_t st) {
  auto& P = e->peer;
  auto& b = e->batches[ib];
  const Shape& s = e->sh;
  const size_t R = e->cfg.batch;
  const uint32_t sq = ++P.seqxo[ib];
  cudaStream_t c = P.cs[e->kp];
  GH_CUDA(cudaEventRecord(P.ev[ib], st));
  GH_CUDA(cudaStreamWaitEvent(c, P.ev[ib], 0));
  GH_CUDA(cudaMemcpyAsync(P.nx[ib], b.x(b.cur), R * s.D * s.db, cudaMemcpyDeviceToDevice, c));
  const int sl = b.ss_slices[b.cur];
  if (P.nss[ib] && sl > 0)
    GH_CUDA(cudaMemcpyAsync(P.nss[ib], b.ss(b.cur), (size_t)sl * R * sizeof(float), cudaMemcpyDeviceToDevice, c));
  GH_CUDA(cudaMemcpyAsync(P.npos[ib], b.pos, R * 4, cudaMemcpyDeviceToDevice, c));
  GH_CU(memops().write((CUstream)c, (CUdeviceptr)(P.nflags + f_x(e, ib)), sq, CU_STREAM_WRITE_VALUE_DEFAULT));
  return GH_OK;
}

// Last span -> first span: the greedy next tokens of batch ib (the first span owns the embedding).
static gh_status peer_send_tokens(gh_engine* e, int ib, cudaStream_t st) {
  auto& P = e->peer;
  auto& b = e->batches[ib];
  const uint32_t sq = ++P.seqt[ib];
  cudaStream_t c = P.cs[e->kp];
  GH_CUDA(cudaEventRecord(P.ev[ib], st));
  GH_CUDA(cudaStreamWaitEvent(c, P.ev[ib], 0));
  GH_CUDA(cudaMemcpyAsync(P.fnext[ib], b.next, e->cfg.batch * 4, cudaMemcpyDeviceToDevice, c));
  GH_CU(memops().write((CUstream)c, (CUdeviceptr)(P.fflags + f_tok(e, ib)), sq, CU_STREAM_WRITE_VALUE_DEFAULT));
  return GH_OK;
}

// First span with n1 > 1: the next tokens of the previous step of batch ib have landed in b.next.
static gh_status peer_wait_tokens(gh_engine* e, int ib, cudaStream_t st) {
  auto& P = e->peer;
  if (!P.on || e->n1 == 1 || e->role != 1 || e->span != 0) return GH_OK;
  if (P.seqt[ib] >= P.seqxo[ib]) return GH_OK;  // already awaited (or no step run yet)
  P.seqt[ib] = P.seqxo[ib];                     // one hand-back per step this span ran
  GH_CU(memops().wait((CUstream)st, (CUdeviceptr)(P.flags + f_tok(e, ib)), P.seqt[ib], CU_STREAM_WAIT_VALUE_GEQ));
  return GH_OK;
}

// One pipelined step of every in-flight batch over the peer transport.  Per Tier-1 span:
//   span 0:  embed_b -> F1_b(l0) -> fwd;   span s > 0: wait x_b from span s-1 -> F1_b(l0) -> fwd
//   for each (layer l, batch b): wait attention of every shard -> F3_b(l) -> F1_b(l+1) -> fwd,
//   after the span's last layer: classifier (last span, tokens back to span 0) or x -> span s+1.
// Tier-2 rank: for each (layer, batch): wait fwd -> F2 (+ KV append) -> bwd back.
static gh_status split_step_peer(gh_engine* e, cudaStream_t st) {
  auto& P = e->peer;
  const int nb = (int)e->batches.size();
  // diagnostics: GH_SPLIT_NOWAIT=1 drops the flag waits (wrong results; isolates compute time)
  static const bool nowait = getenv("GH_SPLIT_NOWAIT") != nullptr;
  static const bool nosend = nowait && getenv("GH_SPLIT_NOSEND") != nullptr;  // + no fwd copies
  static const bool memop_wait = getenv("GH_SPLIT_MEMOP_WAIT") != nullptr;
  // Tier-1 pipeline spans: the in-flight batches are cut into min(IF, spans) groups processed one
  // after another (each group's batches interleaved per layer, so the Tier-2 round trips overlap),
  // so that span s works on group g while span s+1 works on group g-1 -- with every batch's
  // layers interleaved across all IF batches, span s+1 could only start at the end of span s's
  // step and the spans would run one at a time.  One span: a single group (unchanged order).
  const int ng = e->n1 > 1 ? std::min(nb, e->n1) : 1;
  if (e->role == 1) {
    const bool first = e->span == 0, last = e->span == e->n1 - 1;
    for (int gi = 0; gi < ng; ++gi) {
    const int gb0 = gi * nb / ng, gb1 = (gi + 1) * nb / ng;
    for (int ib = gb0; ib < gb1; ++ib) {
      auto& b = e->batches[ib];
      if (first && b.adv_pending) {  // the tokens of this batch's previous step (gh_engine_advance)
        GH_TRY(peer_wait_tokens(e, ib, st));
        GH_CUDA(launch_advance(b.tok, b.next, b.pos, (int)e->cfg.batch, b.adv_inc, st));
        b.adv_pending = false;
        b.adv_inc = 0;
      }
      if (first) {
        GH_TRY(act_embed(e, b, st));
      } else {
        // the previous span's activation (x, its sums of squares, the positions) has landed
        ++P.seqxi[ib];
        if (!nowait)
          GH_CU(memops().wait((CUstream)st, (CUdeviceptr)(P.flags + f_x(e, ib)), P.seqxi[ib],
                              CU_STREAM_WAIT_VALUE_GEQ));
        b.cur = 0;
        b.ss_slices[0] = handoff_ss_slices(e);
      }
      GH_TRY(act_pre(e, b, e->l0, st));
      GH_TRY(peer_send_fwd(e, ib, true, st));
    }
    for (int l = e->l0; l < e->l1; ++l)
      for (int ib = gb0; ib < gb1; ++ib) {
        auto& b = e->batches[ib];
        // every shard of the attention output has landed: the W_o GEMM's producers poll the flag
        // words themselves (weights stream meanwhile, and the launch keeps its programmatic overlap
        // with the previous kernel); GH_SPLIT_MEMOP_WAIT=1 waits in the stream instead (diagnostics)
        const PeerWait pw{P.flags + f_bwd(e, ib, 0), e->kp, P.seq[ib]};
        for (int j = 0; j < e->kp && !nowait && memop_wait; ++j)
          GH_CU(memops().wait((CUstream)st, (CUdeviceptr)(P.flags + f_bwd(e, ib, j)), P.seq[ib],
                              CU_STREAM_WAIT_VALUE_GEQ));
        GH_TRY(act_post(e, b, l, st, nowait || memop_wait ? nullptr : &pw));
        if (l + 1 < e->l1) {
          GH_TRY(act_pre(e, b, l + 1, st));
          if (!nosend) GH_TRY(peer_send_fwd(e, ib, false, st));
        } else if (last) {
          GH_TRY(act_classify(e, b, nullptr, st));
          if (e->n1 > 1) GH_TRY(peer_send_tokens(e, ib, st));
        } else {
          GH_TRY(peer_send_next_span(e, ib, st));
        }
      }
    }
  } else {
    const int tp = e->tp;
    const size_t bwd_row = (size_t)e->sh.ld_bwd() / tp * e->sh.db;  // one head block of a row
    const int me = e->shard;
    for (int gi = 0; gi < ng; ++gi)
    for (int l = e->l0; l < e->l1; ++l)
      for (int ib = gi * nb / ng; ib < (gi + 1) * nb / ng; ++ib) {
        auto& b = e->batches[ib];
        const uint32_t sq = ++P.seq[ib];
        for (int r = 0; r < tp && !nowait; ++r)  // every Tier-1 rank's head block has landed
          GH_CU(memops().wait((CUstream)st, (CUdeviceptr)(P.flags + f_fwd(e, ib, r)), sq, CU_STREAM_WAIT_VALUE_GEQ));
        if (e->cfg.prefill) GH_TRY(t2_append(e->t2, l, e->my_cnt, b.slot, b.pos, b.fwd, st));
        GH_TRY(t2_attend(e->t2, l, e->my_cnt, b.slot, b.pos, b.fwd, b.bwd, st, nullptr, 0, 0, tp));
        GH_CUDA(cudaEventRecord(P.ev[ib], st));
        for (int r = 0; r < tp; ++r) {  // head block r of every row to Tier-1 rank r
          cudaStream_t c = P.cs[r];
          GH_CUDA(cudaStreamWaitEvent(c, P.ev[ib], 0));
          GH_CUDA(cudaMemcpyAsync((char*)P.bwd[r][ib] + e->shard_off[me] * bwd_row,
                                  (char*)b.bwd + (size_t)r * e->my_cnt * bwd_row, e->my_cnt * bwd_row,
                                  cudaMemcpyDeviceToDevice, c));
          GH_CU(memops().write((CUstream)c, (CUdeviceptr)(P.rflags[r] + f_bwd(e, ib, me)), sq,
                               CU_STREAM_WRITE_VALUE_DEFAULT));
        }
      }
  }
  return GH_OK;
}

static gh_status split_step_pipelined(gh_engine* e, cudaStream_t st) {
  if (e->peer.on) return split_step_peer(e, st);
  if (e->n1 > 1 || e->tp > 1) return fail(GH_EUNSUPPORTED, "Tier-1 pipeline stages / tensor parallelism need the peer transport");
  const int nb = (int)e->batches.size();
  const int N = e->sh.N;
  ncclComm_t comm = e->comm->comms[0];
  if (e->role == 1) {
    std::vector<int> pending;
    bool header = true;
    for (int ib = 0; ib < nb; ++ib) {
      auto& b = e->batches[ib];
      GH_TRY(act_embed(e, b, st));
      GH_TRY(act_pre(e, b, 0, st));
      pending.push_back(ib);
      if (ib < nb - 1) {  // let Tier-2 start on batch ib while batch ib+1 is prepared
        GH_TRY(t1_group(e, comm, st, pending, -1, header));
        header = false;
      }
    }
    for (int l = 0; l < N; ++l)
      for (int ib = 0; ib < nb; ++ib) {
        auto& b = e->batches[ib];
        GH_TRY(t1_group(e, comm, st, pending, ib, header));
        header = false;
        GH_TRY(act_post(e, b, l, st));
        if (l + 1 < N) {
          GH_TRY(act_pre(e, b, l + 1, st));
          pending.push_back(ib);
        } else {
          GH_TRY(act_classify(e, b, nullptr, st));
        }
      }
    if (!pending.empty()) GH_TRY(t1_group(e, comm, st, pending, -1, false));
  } else {
    GH_TRY(t2_group(e, comm, st, -1, 0, true));
    for (int l = 0; l < N; ++l)
      for (int ib = 0; ib < nb; ++ib) {
        auto& b = e->batches[ib];
        if (e->cfg.prefill) GH_TRY(t2_append(e->t2, l, e->my_cnt, b.slot, b.pos, b.fwd, st));
    GH_TRY(gh_tier2_attend(e->t2, l, e->my_cnt, b.slot, b.pos, b.fwd, b.bwd, st));
        const bool last = (l == N - 1 && ib == nb - 1);
        GH_TRY(t2_group(e, comm, st, ib, last ? -1 : (ib + 1) % nb, false));
      }
  }
  return GH_OK;
}

gh_status gh_engine_step_all(gh_engine* e, void* stream) {
  if (!e) return fail(GH_EINVAL, "null engine");
  cudaStream_t st = (cudaStream_t)stream;
  GH_CUDA(cudaSetDevice(e->cfg.device));
  const int nb = (int)e->batches.size();
  if (e->role == 0) {
    for (int ib = 0; ib < nb; ++ib) GH_TRY(gh_engine_step_device(e, ib, stream));
    return GH_OK;
  }
  return split_step_pipelined(e, st);
}

gh_status gh_engine_step_all_host(gh_engine* e, const int32_t* tok_host, const int32_t* pos_host,
                                  int32_t* next_host, void* stream) {
  if (!e) return fail(GH_EINVAL, "null engine");
  cudaStream_t st = (cudaStream_t)stream;
  GH_CUDA(cudaSetDevice(e->cfg.device));
  const size_t R = e->cfg.batch;
  if (e->role != 2 && !next_host) return fail(GH_EINVAL, "host next-token buffer required");
  if (e->role != 2 && e->span == 0) {
    if (!tok_host || !pos_host) return fail(GH_EINVAL, "host token/pos buffers required");
    for (size_t ib = 0; ib < e->batches.size(); ++ib) {
      e->batches[ib].adv_pending = false;  // host inputs replace a deferred advance
      e->batches[ib].adv_inc = 0;
      GH_CUDA(cudaMemcpyAsync(e->batches[ib].tok, tok_host + ib * R, R * 4, cudaMemcpyHostToDevice, st));
      GH_CUDA(cudaMemcpyAsync(e->batches[ib].pos, pos_host + ib * R, R * 4, cudaMemcpyHostToDevice, st));
    }
  }
  GH_TRY(gh_engine_step_all(e, stream));
  if (e->role != 2)
    for (size_t ib = 0; ib < e->batches.size(); ++ib)
      GH_CUDA(cudaMemcpyAsync(next_host + ib * R, e->batches[ib].next, R * 4, cudaMemcpyDeviceToHost, st));
  GH_CUDA(cudaStreamSynchronize(st));
  return GH_OK;
}

gh_status gh_engine_step_host(gh_engine* e, uint32_t ib, const int32_t* tok_host, const int32_t* pos_host,
                              int32_t* next_host, float* logits_host, void* stream) {
  if (!e || ib >= e->batches.size()) return fail(GH_EINVAL, "bad engine / batch index");
  auto& b = e->batches[ib];
  cudaStream_t st = (cudaStream_t)stream;
  GH_CUDA(cudaSetDevice(e->cfg.device));
  const int R = e->rows();
  if (e->role != 2) {
    if (!tok_host || !pos_host || !next_host) return fail(GH_EINVAL, "host token/pos/next buffers required");
    if (e->role == 0 && e->t2->paged)  // paged KV: every attended position must be mapped
      GH_TRY(gh_tier2_check(e->t2, (uint32_t)R, b.slot_host.data(), pos_host));
    GH_CUDA(cudaMemcpyAsync(b.tok, tok_host, (size_t)R * 4, cudaMemcpyHostToDevice, st));
    GH_CUDA(cudaMemcpyAsync(b.pos, pos_host, (size_t)R * 4, cudaMemcpyHostToDevice, st));
  }
  if (logits_host && e->role == 0) {
    GH_TRY(engine_layer_loop_colocated(e, b, true, st));
  } else if (logits_host && e->role == 1) {
    if (e->n1 > 1 || e->tp > 1)
      return fail(GH_EUNSUPPORTED, "Tier-1 pipeline stages / tensor parallelism: use gh_engine_step_all / step_all_host");
    ncclComm_t comm = e->comm->comms[0];
    GH_TRY(split_begin(e, b, comm, st));
    for (int l = 0; l < e->sh.N; ++l) GH_TRY(split_layer(e, b, comm, l, st));
    GH_TRY(act_classify(e, b, b.logits, st));
  } else {
    GH_TRY(gh_engine_step_device(e, ib, stream));
  }
  if (e->role != 2) {
    GH_CUDA(cudaMemcpyAsync(next_host, b.next, (size_t)R * 4, cudaMemcpyDeviceToHost, st));
    if (logits_host)
      GH_CUDA(cudaMemcpyAsync(logits_host, b.logits, (size_t)R * e->sh.V * 4, cudaMemcpyDeviceToHost, st));
  }
  GH_CUDA(cudaStreamSynchronize(st));
  return GH_OK;
}

}  // extern "C"

// ================================================================== batch-state dispatcher
// The host scheduler (sched.hpp) driving the engine: IF in-flight batches x B lanes, each lane
// bound to its context slot (colocated: ib * B + row; Tier-2 rank: ib * cnt + row - off, the
// engine's default slots), continuous refill from the queue, per-shard page accounting.  Every
// step: KV actions of the lanes this rank holds (stream-ordered page-table updates, no host
// synchronisation), the lane inputs uploaded from a pinned ring and selected on the device
// (prompt token from the host or the lane's own previous token), the engine step over all
// in-flight batches (gh_engine_step_all: pipelined tier split, or the colocated CUDA graphs),
// and the next tokens copied back into the ring; the host reads a step's tokens one step later,
// so it never waits for the step it just queued.  Every rank of a tier split runs the same
// dispatcher over the same requests (decisions never depend on token values).
struct gh_sched {
  Sched s;
};

struct gh_dispatcher {
  gh_engine* e = nullptr;
  Sched s;
  static constexpr int kRing = 4;
  int32_t* h_in = nullptr;     // pinned [kRing][IF][3][B] lane inputs
  int32_t* h_next = nullptr;   // pinned [kRing][IF][B] next tokens
  float* h_temp = nullptr;     // pinned [kRing][IF][B] 1 / temperature
  uint32_t* h_seed = nullptr;  // pinned [kRing][IF][B]
  int32_t* d_in = nullptr;     // device [IF][3][B]
  uint32_t* h_slot = nullptr;  // pinned [kRing][IF][rows] this rank's rows' slots
  std::vector<uint32_t> last_slots;  // the slot tables last installed
  cudaEvent_t ev[kRing] = {};
  bool ev_used[kRing] = {};
  std::map<uint64_t, std::pair<size_t, void*>> swapbuf;  // swap id -> pinned host buffer (bytes, ptr)
  // pinned buffers whose swap-in copies were queued: back to the pool once their event has passed
  struct Retired { cudaEvent_t ev; size_t bytes; void* p; };
  std::vector<Retired> retired;
  std::vector<std::pair<size_t, void*>> pool;  // free pinned buffers (cudaFreeHost would synchronise)
  std::unique_ptr<DevMem> din_mem;
  cudaStream_t st = nullptr;
  ~gh_dispatcher() {
    if (st) cudaStreamSynchronize(st);
    for (auto& kv : swapbuf) cudaFreeHost(kv.second.second);
    for (auto& r : retired) { cudaEventDestroy(r.ev); cudaFreeHost(r.p); }
    for (auto& b : pool) cudaFreeHost(b.second);
    if (h_in) cudaFreeHost(h_in);
    if (h_next) cudaFreeHost(h_next);
    if (h_temp) cudaFreeHost(h_temp);
    if (h_seed) cudaFreeHost(h_seed);
    if (h_slot) cudaFreeHost(h_slot);
    for (auto v : ev) if (v) cudaEventDestroy(v);
    if (st) cudaStreamDestroy(st);
  }
  uint32_t B() const { return e->cfg.batch; }
  uint32_t IF() const { return (uint32_t)e->batches.size(); }
  bool tokens_here() const { return e->role != 2; }  // Tier-1 (every TP rank) / colocated
  // the local slot of a lane when this rank holds its KV, else -1
  int64_t holder_slot(uint32_t lane) const {
    const uint32_t ib = lane / B(), row = lane % B();
    if (e->role == 0) return (int64_t)ib * B() + row;
    if (e->role == 2) {
      const int off = e->shard_off[e->shard];
      if ((int)row >= off && (int)row < off + e->my_cnt) return (int64_t)ib * e->my_cnt + (row - off);
    }
    return -1;
  }
};

static SchedConfig sched_config(const gh_dispatch_config* c, uint32_t batch, uint32_t inflight, uint32_t kp,
                                uint32_t pages, uint32_t max_seq) {
  SchedConfig sc;
  sc.batch = batch; sc.inflight = inflight; sc.kp = kp; sc.pages = pages; sc.max_seq = max_seq;
  sc.max_new = c->max_new; sc.on_demand = c->on_demand != 0; sc.swap = c->preempt_swap != 0;
  sc.shortest = c->order_shortest != 0;
  sc.chunk = std::max(1u, c->prefill_chunk);
  return sc;
}

static gh_status disp_apply(gh_dispatcher* d, const std::vector<KvAction>& acts) {
  gh_engine* e = d->e;
  gh_tier2* t = e->t2;
  for (size_t i = 0; i < d->retired.size();) {  // restored buffers whose copies have completed
    if (cudaEventQuery(d->retired[i].ev) == cudaSuccess) {
      cudaEventDestroy(d->retired[i].ev);
      d->pool.push_back({d->retired[i].bytes, d->retired[i].p});
      d->retired[i] = d->retired.back();
      d->retired.pop_back();
    } else {
      cudaGetLastError();  // cudaErrorNotReady
      ++i;
    }
  }
  if (!t) return GH_OK;  // Tier-1 holds no KV
  GH_TRY(t2_updates_begin(t));
  for (const KvAction& a : acts) {
    const int64_t slot = d->holder_slot(a.lane);
    if (slot < 0) continue;
    switch (a.op) {
      case kMap: GH_TRY(t2_map_async(t, (uint32_t)slot, a.n, d->st)); break;
      case kUnmap: GH_TRY(gh_tier2_unmap(t, (uint32_t)slot)); break;
      case kSwapOut: {
        // stream-ordered: after the steps that wrote the positions, before any step that reuses
        // the pages (the copies and the steps share the dispatcher's stream) -- no host wait
        const size_t bytes = std::max<uint64_t>(gh_tier2_kv_swap_bytes(t, a.n), 1);
        void* h = nullptr;
        size_t have = 0;
        int best = -1;  // smallest pooled buffer that fits
        for (int i = 0; i < (int)d->pool.size(); ++i)
          if (d->pool[i].first >= bytes && (best < 0 || d->pool[i].first < d->pool[best].first)) best = i;
        if (best >= 0) {
          have = d->pool[best].first;
          h = d->pool[best].second;
          d->pool[best] = d->pool.back();
          d->pool.pop_back();
        } else {
          GH_CUDA(cudaMallocHost(&h, bytes));
          have = bytes;
        }
        d->swapbuf[a.buf] = {have, h};
        GH_TRY(t2_kv_swap_async(t, (uint32_t)slot, a.n, h, 1, d->st));
        break;
      }
      case kSwapIn: {  // queued before the step that resumes the request
        auto it = d->swapbuf.find(a.buf);
        if (it == d->swapbuf.end()) return fail(GH_EINTERNAL, "swap buffer missing on its shard");
        GH_TRY(t2_kv_swap_async(t, (uint32_t)slot, a.n, it->second.second, 0, d->st));
        cudaEvent_t done;
        GH_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
        GH_CUDA(cudaEventRecord(done, d->st));
        d->retired.push_back({done, it->second.first, it->second.second});
        d->swapbuf.erase(it);
        break;
      }
    }
  }
  return t2_updates_end(t, d->st);
}

// The slot tables of this rank's rows: every lane's own slot, except that with chunked prefill a
// row carrying another lane's prompt token reads and appends that lane's slot.  Installed on the
// dispatcher's stream (pinned ring slot k) whenever they differ from the last installed ones (the
// first step installs them: the engine's tables may have been changed by an earlier caller).
static gh_status disp_slots(gh_dispatcher* d, const std::vector<LaneInput>& in, int k) {
  gh_engine* e = d->e;
  const uint32_t B = d->B(), IF = d->IF();
  const int R = e->rows();
  const int off = e->role == 2 ? e->shard_off[e->shard] : 0;
  std::vector<uint32_t> tab((size_t)IF * R);
  for (uint32_t ib = 0; ib < IF; ++ib)
    for (int i = 0; i < R; ++i) {
      const int64_t s = d->holder_slot(in[(size_t)ib * B + off + i].home);
      if (s < 0) return fail(GH_EINTERNAL, "chunked prefill row borrowed across shards");
      tab[(size_t)ib * R + i] = (uint32_t)s;
    }
  if (tab == d->last_slots) return GH_OK;
  uint32_t* hs = d->h_slot + (size_t)k * IF * B;
  std::copy(tab.begin(), tab.end(), hs);
  for (uint32_t ib = 0; ib < IF; ++ib) {
    auto& b = e->batches[ib];
    GH_CUDA(cudaMemcpyAsync(b.slot, hs + (size_t)ib * R, (size_t)R * 4, cudaMemcpyHostToDevice, d->st));
    b.slot_host.assign(hs + (size_t)ib * R, hs + (size_t)(ib + 1) * R);
  }
  d->last_slots.swap(tab);
  return GH_OK;
}

// one step: plan, KV actions, inputs, engine step, next tokens back (resolved one step later)
static gh_status disp_step(gh_dispatcher* d, bool* idle) {
  gh_engine* e = d->e;
  std::vector<LaneInput> in;
  std::vector<KvAction> acts;
  std::string err = d->s.plan(in, acts);
  if (!err.empty()) return fail(GH_EINFEASIBLE, err);
  bool busy = false;
  for (auto& x : in) busy |= x.src != kIdle;
  GH_TRY(disp_apply(d, acts));
  *idle = !busy;
  if (!busy) return GH_OK;  // nothing to decode: the caller drains the unresolved steps
  const uint32_t B = d->B(), IF = d->IF();
  const int k = (int)(d->s.steps % gh_dispatcher::kRing);
  if (d->ev_used[k]) GH_CUDA(cudaEventSynchronize(d->ev[k]));  // ring slot k's copies are done
  if (d->tokens_here()) {
    int32_t* hin = d->h_in + (size_t)k * IF * 3 * B;
    for (uint32_t l = 0; l < IF * B; ++l) {
      const uint32_t ib = l / B, r = l % B;
      int32_t* b3 = hin + (size_t)ib * 3 * B;
      b3[r] = in[l].src;
      b3[B + r] = in[l].tok;
      b3[2 * B + r] = in[l].pos;
    }
    GH_CUDA(cudaMemcpyAsync(d->d_in, hin, (size_t)IF * 3 * B * 4, cudaMemcpyHostToDevice, d->st));
    std::vector<float> it;
    std::vector<uint32_t> sd;
    if (d->s.sampling(it, sd)) {  // per-row batch-state temperature
      float* ht = d->h_temp + (size_t)k * IF * B;
      uint32_t* hs = d->h_seed + (size_t)k * IF * B;
      std::copy(it.begin(), it.end(), ht);
      std::copy(sd.begin(), sd.end(), hs);
      for (uint32_t ib = 0; ib < IF; ++ib) {
        auto& b = e->batches[ib];
        GH_CUDA(cudaMemcpyAsync(b.inv_temp, ht + (size_t)ib * B, B * 4, cudaMemcpyHostToDevice, d->st));
        GH_CUDA(cudaMemcpyAsync(b.seed, hs + (size_t)ib * B, B * 4, cudaMemcpyHostToDevice, d->st));
        bool any = false;
        for (uint32_t r = 0; r < B; ++r) any |= ht[(size_t)ib * B + r] != 0.f;
        if (any != b.sampling) {
          b.sampling = any;
          if (b.graph) {  // the classifier path changes: recapture the colocated step
            GH_CUDA(cudaStreamSynchronize(d->st));
            cudaGraphExecDestroy(b.graph);
            b.graph = nullptr;
          }
        }
      }
    }
    for (uint32_t ib = 0; ib < IF; ++ib) {
      auto& b = e->batches[ib];
      GH_CUDA(launch_dispatch_inputs(b.tok, b.next, b.pos, d->d_in + (size_t)ib * 3 * B, (int)B, d->st));
    }
  }
  if (e->t2) GH_TRY(disp_slots(d, in, k));
  GH_TRY(gh_engine_step_all(e, d->st));
  if (d->tokens_here()) {
    int32_t* hn = d->h_next + (size_t)k * IF * B;
    for (uint32_t ib = 0; ib < IF; ++ib)
      GH_CUDA(cudaMemcpyAsync(hn + (size_t)ib * B, e->batches[ib].next, B * 4, cudaMemcpyDeviceToHost, d->st));
  }
  GH_CUDA(cudaEventRecord(d->ev[k], d->st));
  d->ev_used[k] = true;
  d->s.commit();
  return GH_OK;
}

// tokens of the oldest unresolved step (its ring slot's copies are complete once its event is)
static gh_status disp_resolve_one(gh_dispatcher* d) {
  const uint64_t step = d->s.steps - d->s.unresolved();  // index of the oldest unresolved step
  const int k = (int)(step % gh_dispatcher::kRing);
  if (d->tokens_here()) {
    GH_CUDA(cudaEventSynchronize(d->ev[k]));
    d->s.resolve(d->h_next + (size_t)k * d->IF() * d->B());
  } else {
    d->s.resolve(nullptr);  // Tier-2 ranks: values are irrelevant, the resolution point is not
  }
  return GH_OK;
}

extern "C" {

gh_status gh_sched_create(const gh_sched_config* c, gh_sched** out) {
  if (!c || !out) return fail(GH_EINVAL, "null argument");
  *out = nullptr;
  gh_dispatch_config dc{c->max_new, c->on_demand, c->preempt_swap, c->order_shortest, c->prefill_chunk};
  auto g = std::make_unique<gh_sched>();
  std::string err = g->s.init(sched_config(&dc, c->batch, c->inflight, c->kp, c->pages, c->max_seq));
  if (!err.empty()) return fail(GH_EINVAL, err);
  *out = g.release();
  return GH_OK;
}
gh_status gh_sched_destroy(gh_sched* g) { delete g; return GH_OK; }
gh_status gh_sched_submit(gh_sched* g, const int32_t* prompt, uint32_t len, float temperature, uint32_t seed,
                          uint32_t max_new, uint64_t* id) {
  if (!g || !prompt || !id) return fail(GH_EINVAL, "null argument");
  std::string err = g->s.submit(prompt, len, temperature, seed, id, max_new);
  return err.empty() ? GH_OK : fail(GH_EINFEASIBLE, err);
}
gh_status gh_sched_plan(gh_sched* g, gh_lane_input* in, gh_kv_action* acts, uint32_t cap, uint32_t* n_acts) {
  if (!g || !in || !n_acts) return fail(GH_EINVAL, "null argument");
  std::vector<LaneInput> li;
  std::vector<KvAction> ka;
  std::string err = g->s.plan(li, ka);
  if (!err.empty()) return fail(GH_EINFEASIBLE, err);
  for (size_t i = 0; i < li.size(); ++i) in[i] = {li[i].src, li[i].tok, li[i].pos, li[i].home};
  *n_acts = (uint32_t)ka.size();
  if (ka.size() > cap) return fail(GH_EINVAL, "action buffer too small");
  for (size_t i = 0; i < ka.size(); ++i) acts[i] = {ka[i].op, ka[i].lane, ka[i].n, ka[i].buf};
  return GH_OK;
}
gh_status gh_sched_commit(gh_sched* g) {
  if (!g) return fail(GH_EINVAL, "null argument");
  g->s.commit();
  return GH_OK;
}
gh_status gh_sched_resolve(gh_sched* g, const int32_t* next) {
  if (!g) return fail(GH_EINVAL, "null argument");
  if (!g->s.unresolved()) return fail(GH_EINVAL, "no unresolved step");
  g->s.resolve(next);
  return GH_OK;
}
int gh_sched_done(const gh_sched* g) { return g && g->s.done() ? 1 : 0; }
uint32_t gh_sched_unresolved(const gh_sched* g) { return g ? g->s.unresolved() : 0; }
static gh_status sched_result(const Sched& s, uint64_t id, int32_t* tokens, uint32_t cap, uint32_t* n) {
  const std::vector<int32_t>* r = s.result(id);
  if (!r) return fail(GH_EINVAL, "request " + std::to_string(id) + " is not finished (or not resolved)");
  *n = (uint32_t)r->size();
  if (tokens) std::copy(r->begin(), r->begin() + std::min<size_t>(cap, r->size()), tokens);
  return GH_OK;
}
static void sched_stats(const Sched& s, gh_dispatch_stats* o) {
  o->steps = s.steps; o->admitted = s.admitted; o->finished = s.finished; o->tokens = s.tokens;
  o->preemptions = s.preemptions; o->swaps = s.swaps; o->peak_pages = s.peak_pages;
  o->lane_steps = s.lane_steps; o->context_sum = s.context_sum;
}
gh_status gh_sched_result(const gh_sched* g, uint64_t id, int32_t* tokens, uint32_t cap, uint32_t* n) {
  if (!g || !n) return fail(GH_EINVAL, "null argument");
  return sched_result(g->s, id, tokens, cap, n);
}
gh_status gh_sched_stats(const gh_sched* g, gh_dispatch_stats* out) {
  if (!g || !out) return fail(GH_EINVAL, "null argument");
  sched_stats(g->s, out);
  return GH_OK;
}

gh_status gh_dispatcher_create(gh_engine* e, const gh_dispatch_config* cfg, gh_dispatcher** out) {
  if (!e || !cfg || !out) return fail(GH_EINVAL, "null argument");
  *out = nullptr;
  if (e->n1 > 1) return fail(GH_EUNSUPPORTED, "the dispatcher drives one Tier-1 span (or TP ranks), not pipeline spans");
  if (cfg->prefill_chunk > 1 && !e->cfg.prefill)
    return fail(GH_EINVAL, "chunked prefill needs a prefill-row engine (gh_engine_config.prefill)");
  GH_CUDA(cudaSetDevice(e->cfg.device));
  auto d = std::make_unique<gh_dispatcher>();
  d->e = e;
  const uint32_t kp = e->role == 0 ? 0 : (uint32_t)e->kp;
  const uint32_t pages = e->cfg.kv_pages;
  std::string err = d->s.init(sched_config(cfg, e->cfg.batch, (uint32_t)e->batches.size(), kp, pages, (uint32_t)e->sh.S));
  if (!err.empty()) return fail(GH_EINVAL, err);
  const size_t n = (size_t)d->IF() * d->B();
  GH_CUDA(cudaStreamCreateWithFlags(&d->st, cudaStreamNonBlocking));
  GH_CUDA(cudaMallocHost((void**)&d->h_in, gh_dispatcher::kRing * n * 3 * 4));
  GH_CUDA(cudaMallocHost((void**)&d->h_next, gh_dispatcher::kRing * n * 4));
  GH_CUDA(cudaMallocHost((void**)&d->h_temp, gh_dispatcher::kRing * n * 4));
  GH_CUDA(cudaMallocHost((void**)&d->h_seed, gh_dispatcher::kRing * n * 4));
  GH_CUDA(cudaMallocHost((void**)&d->h_slot, gh_dispatcher::kRing * n * 4));
  d->din_mem = std::make_unique<DevMem>();
  GH_CUDA(cudaMalloc(&d->din_mem->p, n * 3 * 4));
  d->d_in = (int32_t*)d->din_mem->p;
  for (auto& v : d->ev) GH_CUDA(cudaEventCreateWithFlags(&v, cudaEventDisableTiming));
  *out = d.release();
  return GH_OK;
}
gh_status gh_dispatcher_destroy(gh_dispatcher* d) {
  if (d) {
    cudaSetDevice(d->e->cfg.device);
    delete d;
  }
  return GH_OK;
}
gh_status gh_dispatcher_submit(gh_dispatcher* d, const int32_t* prompt, uint32_t len, float temperature,
                               uint32_t seed, uint32_t max_new, uint64_t* id) {
  if (!d || !prompt || !id) return fail(GH_EINVAL, "null argument");
  if (temperature < 0.f) return fail(GH_EINVAL, "temperature must be >= 0");
  std::string err = d->s.submit(prompt, len, temperature, seed, id, max_new);
  return err.empty() ? GH_OK : fail(GH_EINFEASIBLE, err);
}
gh_status gh_dispatcher_step(gh_dispatcher* d, int* busy) {
  if (!d) return fail(GH_EINVAL, "null argument");
  GH_CUDA(cudaSetDevice(d->e->cfg.device));
  bool idle = false;
  GH_TRY(disp_step(d, &idle));
  if (idle) {  // nothing to decode until every step's tokens are known (preempted requests wait)
    while (d->s.unresolved()) GH_TRY(disp_resolve_one(d));
  } else if (d->s.unresolved() > 1) {
    GH_TRY(disp_resolve_one(d));  // the step before the one just queued
  }
  if (busy) *busy = d->s.done() ? 0 : 1;
  return GH_OK;
}
gh_status gh_dispatcher_run(gh_dispatcher* d, uint64_t* steps) {
  if (!d) return fail(GH_EINVAL, "null argument");
  GH_CUDA(cudaSetDevice(d->e->cfg.device));
  while (!d->s.done()) GH_TRY(gh_dispatcher_step(d, nullptr));
  while (d->s.unresolved()) GH_TRY(disp_resolve_one(d));
  GH_CUDA(cudaStreamSynchronize(d->st));
  if (steps) *steps = d->s.steps;
  return GH_OK;
}
gh_status gh_dispatcher_result(const gh_dispatcher* d, uint64_t id, int32_t* tokens, uint32_t cap, uint32_t* n) {
  if (!d || !n) return fail(GH_EINVAL, "null argument");
  return sched_result(d->s, id, tokens, cap, n);
}
gh_status gh_dispatcher_stats(const gh_dispatcher* d, gh_dispatch_stats* out) {
  if (!d || !out) return fail(GH_EINVAL, "null argument");
  sched_stats(d->s, out);
  return GH_OK;
}

}  // extern "C"

extern "C" gh_status gh_debug_gemm_profile(int on) {
  std::lock_guard<std::mutex> lk(g_prof.mu);
  if (on == 2) {  // timeline mode (see GemmProfiler)
    int dev = 0;
    GH_CUDA(cudaGetDevice(&dev));
    if (!g_prof.tl_buf || g_prof.tl_dev != dev) {
      g_prof.tl_cap = 2048;
      GH_CUDA(cudaMalloc(&g_prof.tl_buf, (size_t)g_prof.tl_cap * kNumSMs * 16 * 8));
      g_prof.tl_dev = dev;
    }
    GH_CUDA(cudaMemset(g_prof.tl_buf, 0, (size_t)g_prof.tl_cap * kNumSMs * 16 * 8));
    g_prof.tl_next = 0;
    g_prof.tl_recs.clear();
    g_prof.timeline = true;
    return GH_OK;
  }
  g_prof.timeline = false;
  g_prof.on = on != 0;
  if (const char* t = getenv("GH_GEMM_TRACE")) sscanf(t, "%dx%d", &g_prof.trace_n, &g_prof.trace_k);
  return GH_OK;
}

extern "C" gh_status gh_debug_gemm_profile_dump(char* buf, uint64_t cap) {
  if (!buf || cap == 0) return fail(GH_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(g_prof.mu);
  std::map<std::tuple<int, int, int, bool>, std::pair<int, double>> agg;
  for (auto& r : g_prof.recs) {
    float ms = 0.f;
    if (cudaEventSynchronize(r.b) == cudaSuccess && cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) {
      auto& a = agg[std::make_tuple(r.N, r.K, r.B, r.tp)];
      a.first += 1;
      a.second += ms * 1e3;
    }
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_prof.recs.clear();
  std::string out;
  if (!g_prof.tl_recs.empty()) {  // timeline: one line per launch, us from the first launch's first CTA
    GH_CUDA(cudaDeviceSynchronize());
    const size_t per = (size_t)kNumSMs * 16;
    std::vector<unsigned long long> h(per * g_prof.tl_recs.size());
    GH_CUDA(cudaMemcpy(h.data(), g_prof.tl_buf, h.size() * 8, cudaMemcpyDeviceToHost));
    unsigned long long t0 = ~0ull;
    for (size_t i = 0; i < per; ++i) if (h[i]) t0 = std::min(t0, h[(i / 16) * 16]);
    char line[256];
    for (size_t l = 0; l < g_prof.tl_recs.size(); ++l) {
      const auto& r = g_prof.tl_recs[l];
      const unsigned long long* t = h.data() + l * per;
      const int ex = r.pair ? 10 : 6;
      unsigned long long first = ~0ull, last = 0;
      std::vector<unsigned long long> w;
      int ctas = 0;
      for (int c = 0; c < kNumSMs; ++c) {
        if (!t[c * 16]) continue;
        ++ctas;
        first = std::min(first, t[c * 16]);
        last = std::max(last, t[c * 16 + ex]);
        if (t[c * 16 + 2]) w.push_back(t[c * 16 + 2]);
      }
      if (!ctas) continue;
      std::sort(w.begin(), w.end());
      const double wm = w.empty() ? 0.0 : (double)(w[w.size() / 2] - t0) / 1e3;
      snprintf(line, sizeof(line), "tl %zu N=%d K=%d B=%d %s ctas=%d start=%.2f wait=%.2f exit=%.2f\n", l, r.N, r.K,
               r.B, r.pair ? "pair" : "splitk", ctas, (double)(first - t0) / 1e3, wm, (double)(last - t0) / 1e3);
      out += line;
    }
    g_prof.tl_recs.clear();
    g_prof.timeline = false;
  }
  for (auto& kv : agg) {
    const auto& k = kv.first;
    const double us = kv.second.second / kv.second.first;
    const double mb = (double)std::get<0>(k) * std::get<1>(k) * 2 / 1e6;
    out += "N=" + std::to_string(std::get<0>(k)) + " K=" + std::to_string(std::get<1>(k)) + " B=" +
           std::to_string(std::get<2>(k)) + (std::get<3>(k) ? " tp-allreduce" : "") + " n=" +
           std::to_string(kv.second.first) + " mean_us=" + std::to_string(us) + " weight_MB=" + std::to_string(mb) +
           " TB/s=" + std::to_string(mb / us) + "\n";
  }
  if (!g_prof.phases.empty()) {  // mean over launches of the per-launch medians (us from the first CTA start)
    static const char* names[16] = {"start", "w_prefetched", "griddep_wait", "first_stage", "last_mma", "epi_done",
                                    "exit", "tfull", "drain", "consumed", "published", "ready", "epi_slice_done",
                                    "allreduce_done", "last", "reduced"};
    out += "trace " + std::to_string(g_prof.trace_n) + "x" + std::to_string(g_prof.trace_k) + " (" +
           std::to_string(g_prof.phases.size()) + " launches):";
    for (int i = 0; i < 16; ++i) {
      double m = 0;
      for (auto& ph : g_prof.phases) m += ph[i];
      out += std::string(" ") + names[i] + "=" + std::to_string(m / g_prof.phases.size());
    }
    out += "\n";
    g_prof.phases.clear();
  }
  snprintf(buf, cap, "%s", out.c_str());
  return GH_OK;
}

extern "C" gh_status gh_debug_gemm_bench(int N, int K, int B, int flags, int stages, int ks, int reps, float* us) {
  if (!us || N <= 0 || K <= 0 || B <= 0 || reps <= 0) return fail(GH_EINVAL, "bad argument");
  if (gh_device_count() == 0) return fail(GH_ECUDA, "no CUDA device");
  GH_CUDA(cudaSetDevice(0));
  GH_CUDA(configure_kernels());
  std::vector<std::unique_ptr<DevMem>> mem;
  Weight W;
  W.N = N; W.K = K; W.dtype_bytes = 2; W.tiled = true;
  GH_TRY(dev_alloc(mem, W.elems() * 2, &W.ptr));
  const uint64_t tid = 7; const int rows = N; const double sd = 0.02;
  GH_CUDA(launch_init_weight(W, make_segs(1, 1, &tid, &rows, &sd, false), 0));
  CUtensorMap tmW, tmX;
  GH_CUDA(make_tmap_bf16(&tmW, W.ptr, (uint64_t)W.n_pad() * W.kb(), 64, 64, 128));
  void *X, *Y;
  GH_TRY(dev_alloc(mem, (size_t)B * K * 2, &X));
  GH_TRY(dev_alloc(mem, (size_t)B * N * 2, &Y));
  GH_CUDA(cudaMemset(X, 0, (size_t)B * K * 2));
  // diagnostics: ks > 0 forces the split-K cluster size, -1 forces split-K, -2 the pair kernel,
  // -3 split-K with the 192-column tile, -4 split-K without it
  if (ks >= 0) gemm_debug_cluster(ks);
  else if (ks >= -2) gemm_debug_pair(-ks);
  else { gemm_debug_pair(1); gemm_debug_wide(ks == -3 ? 2 : 1); }
  GemmPlan p = plan_gemm(N, K, B);
  gemm_debug_cluster(0);
  gemm_debug_pair(0);
  gemm_debug_wide(0);
  GH_CUDA(make_tmap_bf16(&tmX, X, (uint64_t)B, (uint64_t)K, (uint64_t)K, (uint32_t)p.x_box_rows()));
  GemmScratch sc;
  {
    void* q;
    GH_TRY(dev_alloc(mem, kSkWsBytes, &q));
    sc.sk_ws = (float*)q;
    GH_TRY(dev_alloc(mem, kNumSMs * sizeof(unsigned int), &q));
    sc.sk_flags = (unsigned int*)q;
    GH_CUDA(cudaMemset(q, 0, kNumSMs * sizeof(unsigned int)));
  }
  sc.debug_flags = flags;
  EpiParams ep = epi_default();
  ep.kind = EPI_STORE; ep.out = Y; ep.ldo = N;
  gemm_debug_set(stages);
  cudaEvent_t e0, e1;
  GH_CUDA(cudaEventCreate(&e0)); GH_CUDA(cudaEventCreate(&e1));
  for (int i = 0; i < 3; ++i) GH_CUDA(launch_gemm(W, &tmW, X, K, &tmX, B, p, ep, sc, 0));
  GH_CUDA(cudaEventRecord(e0, 0));
  for (int i = 0; i < reps; ++i) GH_CUDA(launch_gemm(W, &tmW, X, K, &tmX, B, p, ep, sc, 0));
  GH_CUDA(cudaEventRecord(e1, 0));
  GH_CUDA(cudaEventSynchronize(e1));
  float ms = 0;
  GH_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0); cudaEventDestroy(e1);
  gemm_debug_set(0);
  *us = ms * 1000.f / reps;
  return GH_OK;
}

extern "C" gh_status gh_debug_gemm_trace(int N, int K, int B, int copies, int reps, float* us,
                                         unsigned long long* trace, int trace_cap) {
  if (!us || N <= 0 || K <= 0 || B <= 0 || reps <= 0 || copies <= 0) return fail(GH_EINVAL, "bad argument");
  if (gh_device_count() == 0) return fail(GH_ECUDA, "no CUDA device");
  const int dbg_flags = reps / 1000;  // diagnostics: flags packed above the repetition count
  reps %= 1000;
  GH_CUDA(cudaSetDevice(0));
  GH_CUDA(configure_kernels());
  std::vector<std::unique_ptr<DevMem>> mem;
  std::vector<Weight> Ws(copies);
  std::vector<CUtensorMap> tms(copies);
  for (int c = 0; c < copies; ++c) {
    Weight& W = Ws[c];
    W.N = N; W.K = K; W.dtype_bytes = 2; W.tiled = true;
    GH_TRY(dev_alloc(mem, W.elems() * 2, &W.ptr));
    const uint64_t tid = 7 + c; const int rows = N; const double sd = 0.02;
    GH_CUDA(launch_init_weight(W, make_segs(1, 1, &tid, &rows, &sd, false), 0));
    GH_CUDA(make_tmap_bf16(&tms[c], W.ptr, (uint64_t)W.n_pad() * W.kb(), 64, 64, 128));
  }
  void *X, *Y;
  GH_TRY(dev_alloc(mem, (size_t)B * K * 2, &X));
  GH_TRY(dev_alloc(mem, (size_t)B * N * 2, &Y));
  GH_CUDA(cudaMemset(X, 0, (size_t)B * K * 2));
  GemmPlan p = plan_gemm(N, K, B);
  CUtensorMap tmX;
  GH_CUDA(make_tmap_bf16(&tmX, X, (uint64_t)B, (uint64_t)K, (uint64_t)K, (uint32_t)p.x_box_rows()));
  GemmScratch sc;
  {
    void* q;
    GH_TRY(dev_alloc(mem, kSkWsBytes, &q));
    sc.sk_ws = (float*)q;
    GH_TRY(dev_alloc(mem, kNumSMs * sizeof(unsigned int), &q));
    sc.sk_flags = (unsigned int*)q;
    GH_CUDA(cudaMemset(q, 0, kNumSMs * sizeof(unsigned int)));
  }
  void* q;
  sc.debug_flags = dbg_flags;
  unsigned long long* dtrace = nullptr;
  if (trace) {
    GH_TRY(dev_alloc(mem, (size_t)p.n_clusters * p.C * 128, &q));
    dtrace = (unsigned long long*)q;
    GH_CUDA(cudaMemset(q, 0, (size_t)p.n_clusters * p.C * 128));
  }
  EpiParams ep = epi_default();
  ep.kind = EPI_STORE; ep.out = Y; ep.ldo = N;
  cudaEvent_t e0, e1;
  GH_CUDA(cudaEventCreate(&e0)); GH_CUDA(cudaEventCreate(&e1));
  for (int i = 0; i < copies; ++i) GH_CUDA(launch_gemm(Ws[i], &tms[i], X, K, &tmX, B, p, ep, sc, 0));
  GH_CUDA(cudaEventRecord(e0, 0));
  for (int i = 0; i < reps; ++i) {
    if (i == reps - 1) sc.trace = dtrace;
    GH_CUDA(launch_gemm(Ws[i % copies], &tms[i % copies], X, K, &tmX, B, p, ep, sc, 0));
  }
  GH_CUDA(cudaEventRecord(e1, 0));
  GH_CUDA(cudaEventSynchronize(e1));
  float ms = 0;
  GH_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0); cudaEventDestroy(e1);
  *us = ms * 1000.f / reps;
  if (trace) GH_CUDA(cudaMemcpy(trace, dtrace, (size_t)std::min(p.n_clusters * p.C, trace_cap / 16) * 128, cudaMemcpyDeviceToHost));
  return GH_OK;
}
