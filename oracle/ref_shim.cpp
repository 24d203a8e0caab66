// ref_shim.cpp — extern "C" wrappers around the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile into
// oracle/_ref/libtierplan_ref.so).  TEST INFRASTRUCTURE ONLY: tests call these to check the
// product's accounting functions (include/gh/gh.h) and emitted kernel-latency CSVs against the
// reference's own implementation.  No reference source is copied into this repository.
#include <cstdint>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>

#include "tierplan/commands.hpp"
#include "tierplan/des.hpp"
#include "tierplan/errors.hpp"
#include "tierplan/model.hpp"
#include "tierplan/netmodel.hpp"
#include "tierplan/optimizer.hpp"
#include "tierplan/profiles.hpp"

using namespace tierplan;

struct ref_spec {  // same layout as gh_model_spec (include/gh/gh.h)
  uint64_t n_layers, d_model, d_kv, d_hidden, n_heads, n_kv_heads, max_seq_len, dtype_bytes, vocab_size;
  float rope_theta, norm_eps;
};

static thread_local std::string g_err;

static TransformerSpec to_spec(const ref_spec* s) {
  TransformerSpec t;
  t.name = "shim";
  t.n_layers = s->n_layers; t.d_model = s->d_model; t.d_kv = s->d_kv; t.d_hidden = s->d_hidden;
  t.n_heads = s->n_heads; t.n_kv_heads = s->n_kv_heads; t.max_seq_len = s->max_seq_len;
  t.dtype_bytes = s->dtype_bytes;
  if (s->vocab_size) t.vocab_size = s->vocab_size;
  return t;
}

template <typename F>
static int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const FeasibilityError& e) {
    g_err = e.what();
    return 3;
  } catch (const ValidationError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_validate(const ref_spec* s) { return guarded([&] { to_spec(s).validate(); }); }

int ref_kv_bytes_per_prompt(const ref_spec* s, uint64_t seq, uint64_t* out) {
  return guarded([&] { *out = kv_bytes_per_prompt(to_spec(s), seq); });
}
int ref_nonattention_footprint(const ref_spec* s, uint64_t batch, uint64_t* mem, uint64_t* flops) {
  return guarded([&] { auto f = nonattention_footprint(to_spec(s), batch); *mem = f.mem_accesses; *flops = f.flops; });
}
int ref_attention_footprint(const ref_spec* s, uint64_t batch, uint64_t seq, uint64_t* mem, uint64_t* flops) {
  return guarded([&] { auto f = attention_footprint(to_spec(s), batch, seq); *mem = f.mem_accesses; *flops = f.flops; });
}
int ref_weights_bytes(const ref_spec* s, uint64_t* out) {
  return guarded([&] { *out = weights_bytes(to_spec(s)); });
}
int ref_payload(const ref_spec* s, uint64_t* out) {
  return guarded([&] {
    auto p = PayloadModel::for_model(to_spec(s));
    out[0] = p.tier1_to_tier2_per_token; out[1] = p.tier2_to_tier1_per_token; out[2] = p.intra_tier1_per_token;
  });
}
int ref_layer_spans(uint64_t n_layers, uint64_t nodes, uint64_t* out) {
  return guarded([&] { auto v = layer_spans(n_layers, nodes); for (size_t i = 0; i < v.size(); ++i) out[i] = v[i]; });
}
int ref_node_weight_bytes(const ref_spec* s, uint64_t nodes, uint64_t* out) {
  return guarded([&] { auto v = node_weight_bytes(to_spec(s), nodes); for (size_t i = 0; i < v.size(); ++i) out[i] = v[i]; });
}
int ref_two_tier_context_slots(const ref_spec* s, uint64_t k1, uint64_t k2, uint64_t mem, uint64_t seq, uint64_t* out) {
  return guarded([&] { *out = two_tier_context_slots(to_spec(s), k1, k2, mem, seq); });
}
int ref_batch_grid(uint64_t max_batch, uint64_t* out, uint64_t cap, uint64_t* n) {
  return guarded([&] {
    auto v = batch_grid(max_batch);
    *n = v.size();
    for (size_t i = 0; i < v.size() && i < cap; ++i) out[i] = v[i];
  });
}
int ref_throughput_from(const int64_t* ts, uint64_t n, uint64_t batch, uint64_t inflight, double* out) {
  return guarded([&] {
    std::vector<Duration> g;
    for (uint64_t i = 0; i < n; ++i) g.push_back(Duration{ts[i]});
    *out = throughput_from(g, batch, inflight);
  });
}
// load_profile (profiles.cpp:226-230): 0 ok (warnings counted), 2 validation error
int ref_profile_check(const char* path, int* n_warnings) {
  return guarded([&] { auto p = load_profile(path); *n_warnings = (int)p.warnings().size(); });
}
// KernelProfile::latency (profiles.cpp:93-129); seq 0 = default (max profiled)
int ref_profile_latency(const char* path, int stage, uint64_t batch, uint64_t seq, int64_t* ns) {
  return guarded([&] {
    auto p = load_profile(path);
    std::optional<Count> s;
    if (seq) s = seq;
    *ns = p.latency((StageKind)stage, batch, s).count();
  });
}
// Run a reference command in-process (commands.hpp:90-93); writes stdout into `out`.
int ref_cmd_simulate(const char* model, const char* cluster, const char* t1_profile, const char* t2_profile,
                     uint64_t k1, uint64_t k2, uint64_t batch, uint64_t seq, uint64_t inflight, char* out,
                     uint64_t cap) {
  std::ostringstream os, es;
  SimulateArgs a;
  a.model_path = model;
  a.cluster_path = cluster;
  a.profile_paths = {t1_profile, t2_profile};
  a.tier1_nodes = k1;
  a.tier2_per_tier1 = k2;
  a.batch = batch;
  if (seq) a.seq_len = seq;
  if (inflight) a.inflight_override = inflight;
  int rc = cmd_simulate(a, os, es);
  std::string s = os.str() + es.str();
  if (out && cap) { strncpy(out, s.c_str(), cap - 1); out[cap - 1] = 0; }
  return rc;
}

// The reference optimizer (commands.hpp:92, optimizer.cpp:515-583) over the given profiles.
int ref_cmd_optimize(const char* model, const char* cluster, const char* t1_profile, const char* t2_profile,
                     uint64_t seq, uint64_t max_nodes, char* out, uint64_t cap) {
  std::ostringstream os, es;
  OptimizeArgs a;
  a.model_path = model;
  a.cluster_path = cluster;
  a.profile_paths = {t1_profile, t2_profile};
  if (seq) a.seq_len = seq;
  if (max_nodes) a.max_nodes = max_nodes;
  a.threads = 1;
  int rc = cmd_optimize(a, os, es);
  std::string s = os.str() + es.str();
  if (out && cap) { strncpy(out, s.c_str(), cap - 1); out[cap - 1] = 0; }
  return rc;
}

}  // extern "C"
