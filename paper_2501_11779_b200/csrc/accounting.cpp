// accounting.cpp — host-only restatement of the reference's hot-path contract functions.
// Each function cites the reference implementation it mirrors; tests/test_accounting.py checks
// every one against the reference library compiled from /root/reference (oracle/_ref).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "gh/gh.h"
#include "internal.hpp"

using namespace gh;

extern "C" {

// TransformerSpec::validate (proj/src/model.cpp:12-38).  vocab_size 0 encodes "absent".
gh_status gh_spec_validate(const gh_model_spec* s) {
  if (!s) return fail(GH_EINVAL, "spec is null");
  const struct { uint64_t v; const char* n; } pos[] = {
      {s->n_layers, "n_layers"}, {s->d_model, "d_model"}, {s->d_kv, "d_kv"},
      {s->d_hidden, "d_hidden"}, {s->n_heads, "n_heads"}, {s->n_kv_heads, "n_kv_heads"},
      {s->max_seq_len, "max_seq_len"}};
  for (const auto& p : pos)
    if (p.v == 0) return fail(GH_EINVAL, std::string(p.n) + " must be strictly positive");
  if (s->d_model % s->n_heads != 0) return fail(GH_EINVAL, "d_model not divisible by n_heads");
  if (s->d_kv % s->n_kv_heads != 0) return fail(GH_EINVAL, "d_kv not divisible by n_kv_heads");
  if (s->dtype_bytes != 1 && s->dtype_bytes != 2 && s->dtype_bytes != 4)
    return fail(GH_EINVAL, "dtype_bytes must be 1, 2 or 4");
  return GH_OK;
}

// kv_bytes_per_prompt (model.cpp:40-46): 2 * dtype * N * S * D_kv
gh_status gh_kv_bytes_per_prompt(const gh_model_spec* s, uint64_t seq_len, uint64_t* out) {
  if (!s || !out) return fail(GH_EINVAL, "null argument");
  if (seq_len > s->max_seq_len)
    return fail(GH_EINVAL, "seq_len " + std::to_string(seq_len) + " exceeds max_seq_len " +
                               std::to_string(s->max_seq_len));
  *out = 2 * s->dtype_bytes * s->n_layers * seq_len * s->d_kv;
  return GH_OK;
}

// nonattention_footprint (model.cpp:48-56)
gh_status gh_nonattention_footprint(const gh_model_spec* s, uint64_t batch, uint64_t* mem,
                                    uint64_t* flops) {
  if (!s || !mem || !flops) return fail(GH_EINVAL, "null argument");
  const uint64_t d = s->d_model, dh = s->d_hidden, dkv = s->d_kv;
  *mem = d * (2 * d + 3 * dh + 2 * dkv) + batch * (8 * d + 3 * dh + 2 * dkv);
  *flops = batch * d * (2 * d + 3 * dh + 2 * dkv);
  return GH_OK;
}

// attention_footprint (model.cpp:58-67)
gh_status gh_attention_footprint(const gh_model_spec* s, uint64_t batch, uint64_t seq_len,
                                 uint64_t* mem, uint64_t* flops) {
  if (!s || !mem || !flops) return fail(GH_EINVAL, "null argument");
  const uint64_t d = s->d_model, h = s->n_heads, dkv = s->d_kv;
  *mem = 2 * batch * (d + seq_len * h + seq_len * dkv);
  *flops = 2 * seq_len * batch * d;
  return GH_OK;
}

// weights_bytes (model.cpp:69-77)
gh_status gh_weights_bytes(const gh_model_spec* s, uint64_t* out) {
  if (!s || !out) return fail(GH_EINVAL, "null argument");
  const uint64_t d = s->d_model;
  uint64_t el = s->n_layers * (2 * d * d + 2 * d * s->d_kv + 3 * d * s->d_hidden);
  if (s->vocab_size) el += 2 * s->vocab_size * d;
  *out = el * s->dtype_bytes;
  return GH_OK;
}

// PayloadModel::for_model (netmodel.cpp:18-24)
gh_status gh_payload_bytes(const gh_model_spec* s, uint64_t out[3]) {
  if (!s || !out) return fail(GH_EINVAL, "null argument");
  out[0] = s->dtype_bytes * (2 * s->d_model + 2 * s->d_kv);
  out[1] = s->dtype_bytes * 2 * s->d_model;
  out[2] = s->dtype_bytes * s->d_model;
  return GH_OK;
}

// layer_spans (optimizer.cpp:116-123): contiguous blocks, remainder to the low ranks
gh_status gh_layer_spans(uint64_t n_layers, uint64_t nodes, uint64_t* spans) {
  if (!spans) return fail(GH_EINVAL, "null argument");
  if (nodes == 0 || n_layers < nodes) return fail(GH_EINVAL, "layer_spans: need 1 <= nodes <= n_layers");
  for (uint64_t i = 0; i < nodes; ++i) spans[i] = n_layers / nodes + (i < n_layers % nodes ? 1 : 0);
  return GH_OK;
}

// node_weight_bytes (optimizer.cpp:125-136)
gh_status gh_node_weight_bytes(const gh_model_spec* s, uint64_t tier1_nodes, uint64_t* out) {
  if (!s || !out) return fail(GH_EINVAL, "null argument");
  std::vector<uint64_t> spans(tier1_nodes ? tier1_nodes : 1);
  gh_status st = gh_layer_spans(s->n_layers, tier1_nodes, spans.data());
  if (st != GH_OK) return st;
  const uint64_t d = s->d_model;
  const uint64_t per_layer = (2 * d * d + 2 * d * s->d_kv + 3 * d * s->d_hidden) * s->dtype_bytes;
  for (uint64_t i = 0; i < tier1_nodes; ++i) out[i] = spans[i] * per_layer;
  if (s->vocab_size) out[0] += 2 * s->vocab_size * d * s->dtype_bytes;
  return GH_OK;
}

// two_tier_context_slots (optimizer.cpp:175-192), 5 % reserve at :186
gh_status gh_two_tier_context_slots(const gh_model_spec* s, uint64_t tier1_nodes,
                                    uint64_t tier2_per_tier1, uint64_t mem, uint64_t seq_len,
                                    uint64_t* out) {
  if (!s || !out) return fail(GH_EINVAL, "null argument");
  if (tier2_per_tier1 == 0) return fail(GH_EINVAL, "two_tier_context_slots: K' must be >= 1");
  if (seq_len > s->max_seq_len)
    return fail(GH_EINVAL, "seq_len " + std::to_string(seq_len) + " exceeds max_seq_len " +
                               std::to_string(s->max_seq_len));
  const uint64_t per_layer = 2 * s->dtype_bytes * seq_len * s->d_kv;
  if (per_layer == 0) return fail(GH_EINVAL, "context slots: per-prompt bytes are zero (seq_len 0?)");
  std::vector<uint64_t> spans(tier1_nodes ? tier1_nodes : 1);
  gh_status st = gh_layer_spans(s->n_layers, tier1_nodes, spans.data());
  if (st != GH_OK) return st;
  const uint64_t usable = mem - mem / 20;
  uint64_t slots = std::numeric_limits<uint64_t>::max();
  for (uint64_t i = 0; i < tier1_nodes; ++i) {
    const uint64_t v = tier2_per_tier1 * (usable / (per_layer * spans[i]));
    if (v < slots) slots = v;
  }
  *out = slots;
  return GH_OK;
}

// batch_grid (profiles.cpp:232-245)
gh_status gh_batch_grid(uint64_t max_batch, uint64_t* out, uint64_t cap, uint64_t* n) {
  if (!n) return fail(GH_EINVAL, "null argument");
  if (max_batch == 0) return fail(GH_EINVAL, "batch_grid: max_batch must be >= 1");
  std::vector<uint64_t> grid;
  for (int k = 0;; ++k) {
    const uint64_t v = (uint64_t)std::llround(std::pow(2.0, (double)k / 2.0));
    if (v > max_batch) break;
    if (grid.empty() || grid.back() != v) grid.push_back(v);
  }
  if (grid.back() != max_batch) grid.push_back(max_batch);
  *n = grid.size();
  for (uint64_t i = 0; i < grid.size() && i < cap && out; ++i) out[i] = grid[i];
  return GH_OK;
}

// Balanced shards (analytic.cpp:119): batch / kp each, the remainder to the low ranks
gh_status gh_shard_plan(uint64_t batch, uint64_t kp, uint64_t* off, uint64_t* cnt) {
  if (!off || !cnt) return fail(GH_EINVAL, "null argument");
  if (kp == 0 || batch < kp) return fail(GH_EINVAL, "shard_plan: need 1 <= kp <= batch");
  uint64_t o = 0;
  for (uint64_t j = 0; j < kp; ++j) {
    cnt[j] = batch / kp + (j < batch % kp ? 1 : 0);
    off[j] = o;
    o += cnt[j];
  }
  return GH_OK;
}

// Rank layout of a tier split (the engine's decomposition, host only): Tier-1 pipeline spans
// (layer_spans, optimizer.cpp:116-123) or Tier-1 tensor-parallel ranks, then K'
// Tier-2 ranks per span holding balanced prompt shards (analytic.cpp:119).
gh_status gh_engine_layout(uint32_t world, uint32_t rank, uint32_t tier1_ranks, uint32_t tier1_tp,
                           uint64_t n_layers, uint32_t batch, gh_rank_layout* out) {
  if (!out) return fail(GH_EINVAL, "null argument");
  if (world == 0 || rank >= world) return fail(GH_EINVAL, "rank outside the world");
  gh_rank_layout L{};
  const uint32_t n1 = tier1_ranks > 1 ? tier1_ranks : 1, tp = tier1_tp > 1 ? tier1_tp : 1;
  L.tp_rank = 0;
  L.shard = -1;
  L.layer_begin = 0;
  L.layer_end = (uint32_t)n_layers;
  L.row_off = 0;
  L.row_cnt = batch;
  if (world == 1) {
    if (tp > 1 || n1 > 1) return fail(GH_EINVAL, "Tier-1 spans / tensor parallelism need a tier split");
    L.role = 0;
    L.span = 0;
    L.kp = 0;
    *out = L;
    return GH_OK;
  }
  if (tp > 1 && n1 > 1) return fail(GH_EUNSUPPORTED, "tier1_tp and tier1_ranks (pipeline spans) together");
  const uint32_t t1 = tp > 1 ? tp : n1;  // Tier-1 ranks
  if (world <= t1 || (world - t1) % n1) return fail(GH_EINVAL, "world size must be T + n1 * K' with K' >= 1");
  if (n1 > n_layers) return fail(GH_EINVAL, "more Tier-1 spans than layers");
  L.kp = (world - t1) / n1;
  if (batch < L.kp) return fail(GH_EINVAL, "batch smaller than the number of Tier-2 ranks");
  L.role = rank < t1 ? 1 : 2;
  L.span = rank < t1 ? (tp > 1 ? 0 : (int)rank) : (int)((rank - t1) / L.kp);
  if (tp > 1 && rank < t1) L.tp_rank = (int)rank;
  std::vector<uint64_t> spans(n1);
  GH_TRY(gh_layer_spans(n_layers, n1, spans.data()));
  uint64_t l0 = 0;
  for (int s = 0; s < L.span; ++s) l0 += spans[s];
  L.layer_begin = (uint32_t)l0;
  L.layer_end = (uint32_t)(l0 + spans[L.span]);
  if (L.role == 2) {
    L.shard = (int)((rank - t1) % L.kp);
    std::vector<uint64_t> off(L.kp), cnt(L.kp);
    GH_TRY(gh_shard_plan(batch, L.kp, off.data(), cnt.data()));
    L.row_off = (uint32_t)off[L.shard];
    L.row_cnt = (uint32_t)cnt[L.shard];
  }
  *out = L;
  return GH_OK;
}

// throughput_from (des.cpp:298-310)
gh_status gh_throughput_from(const int64_t* ts, uint64_t n, uint64_t batch_total,
                             uint64_t inflight, double* tps) {
  if (!ts || !tps) return fail(GH_EINVAL, "null argument");
  if (n < 2) return fail(GH_EINVAL, "throughput_from: need at least 2 generation timestamps");
  const int64_t span = ts[n - 1] - ts[0];
  if (span <= 0) return fail(GH_EINVAL, "throughput_from: generation timestamps must advance");
  const double mean_tbt = (double)span / (double)(n - 1) / 1e9;
  *tps = (double)batch_total * (double)inflight / mean_tbt;
  return GH_OK;
}

// Kernel-latency CSV (profiles.hpp:66-69; parse_profile profiles.cpp:168-224)
gh_status gh_profile_write_csv(const char* path, const char* mode, const char* device,
                               gh_stage stage, uint64_t seq_len, const uint64_t* batches,
                               const double* lat_us, uint64_t n) {
  if (!path || !mode || !device || (n && (!batches || !lat_us))) return fail(GH_EINVAL, "null argument");
  const char* names[] = {"nonattention", "attention", "classifier"};
  if ((int)stage < 0 || (int)stage > 2) return fail(GH_EINVAL, "unknown stage");
  if (!device[0] || strchr(device, ',') || strchr(device, '\n'))
    return fail(GH_EINVAL, "device name must be non-empty and contain no ',' or newline");
  for (uint64_t i = 0; i < n; ++i) {
    if (!(lat_us[i] > 0)) return fail(GH_EINVAL, "latency_us must be positive");
    if (batches[i] == 0) return fail(GH_EINVAL, "batch_size must be >= 1");
  }
  const bool write = mode[0] == 'w';
  FILE* f = fopen(path, write ? "w" : "a");
  if (!f) return fail(GH_EINVAL, std::string("cannot open ") + path);
  if (write) fprintf(f, "device,stage,seq_len,batch_size,latency_us\n");
  for (uint64_t i = 0; i < n; ++i)
    fprintf(f, "%s,%s,%llu,%llu,%.4f\n", device, names[stage], (unsigned long long)seq_len,
            (unsigned long long)batches[i], lat_us[i]);
  fclose(f);
  return GH_OK;
}

}  // extern "C"
