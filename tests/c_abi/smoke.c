/*
 * smoke.c — a compiled C consumer of include/gh/gh.h (C11, no C++), i.e. what a reference-side
 * maintainer links: `cc -std=c11 -I include smoke.c -L paper_2501_11779_b200 -lgh -lcudart`.
 *
 *   smoke cpu <csv_path>       accounting calls (model.cpp:40-77, netmodel.cpp:18-24,
 *                              optimizer.cpp:116-192) and the profile CSV producer
 *                              (profiles.hpp:66-69); prints one JSON line.  No GPU needed.
 *   smoke sched                the dispatcher's decision logic (gh_sched_*) with chunked prefill
 *                              against a toy context-hash model; prints one JSON line.  No GPU.
 *   smoke gpu <prompts.txt>    the INTEGRATION.md per-layer call sequence (gh_tier1_embed ->
 *                              {gh_tier1_pre -> gh_tier2_attend -> gh_tier1_post} x N ->
 *                              gh_tier1_classify) for BASELINE configs[0] (C1: tiny 288x6 fp32,
 *                              4 prompts of length 8, 128 greedy tokens); prints the generated
 *                              token ids, one row per prompt.  tests/test_c_abi.py compares them
 *                              with the oracle's committed C1 tokens (tests/golden/oracle_c1.npz).
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "gh/gh.h"

#define CK(call)                                                                          \
  do {                                                                                    \
    gh_status s_ = (call);                                                                \
    if (s_ != GH_OK) {                                                                    \
      fprintf(stderr, "%s:%d %s -> %s: %s\n", __FILE__, __LINE__, #call, gh_status_name(s_), \
              gh_last_error());                                                           \
      exit(10 + (int)s_);                                                                 \
    }                                                                                     \
  } while (0)
#define CU(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) {                                                              \
      fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #call, cudaGetErrorString(e_)); \
      exit(30);                                                                           \
    }                                                                                     \
  } while (0)

static int run_cpu(const char* csv) {
  /* C2: Llama-2-7B shape at S = 512 (configs/llama2-7b-ctx512.json) */
  gh_model_spec s7 = {32, 4096, 4096, 11008, 32, 32, 512, 2, 32000, 10000.f, 1e-5f};
  uint64_t kv = 0, mem = 0, flops = 0, w = 0, pay[3] = {0, 0, 0}, slots = 0, spans[2] = {0, 0};
  CK(gh_spec_validate(&s7));
  CK(gh_kv_bytes_per_prompt(&s7, 512, &kv));
  CK(gh_nonattention_footprint(&s7, 64, &mem, &flops));
  CK(gh_weights_bytes(&s7, &w));
  CK(gh_payload_bytes(&s7, pay));
  CK(gh_two_tier_context_slots(&s7, 1, 3, 179ull << 30, 512, &slots));
  CK(gh_layer_spans(80, 2, spans));
  /* validation errors keep the reference's taxonomy (ValidationError = exit 2) */
  gh_model_spec bad = s7;
  bad.n_heads = 33;
  const gh_status rc_bad = gh_spec_validate(&bad);
  /* the kernel-latency boundary: header + rows the reference's parse_profile accepts */
  const uint64_t batches[3] = {1, 2, 4};
  const double lat[3] = {10.5, 11.0, 12.25};
  CK(gh_profile_write_csv(csv, "w", "b200", GH_STAGE_NONATTENTION, 512, batches, lat, 3));
  CK(gh_profile_write_csv(csv, "a", "b200", GH_STAGE_ATTENTION, 512, batches, lat, 3));
  printf("{\"abi\": %d, \"kv_bytes_per_prompt\": %llu, \"nonattention_mem\": %llu, \"nonattention_flops\": %llu, "
         "\"weights_bytes\": %llu, \"payload\": [%llu, %llu, %llu], \"two_tier_context_slots\": %llu, "
         "\"layer_spans\": [%llu, %llu], \"invalid_spec_status\": %d, \"devices\": %d}\n",
         gh_abi_version(), (unsigned long long)kv, (unsigned long long)mem, (unsigned long long)flops,
         (unsigned long long)w, (unsigned long long)pay[0], (unsigned long long)pay[1], (unsigned long long)pay[2],
         (unsigned long long)slots, (unsigned long long)spans[0], (unsigned long long)spans[1], (int)rc_bad,
         gh_device_count());
  return 0;
}

static int run_gpu(const char* prompts_path) {
  enum { B = 4, PLEN = 8, NEW = 128 };
  /* C1: the llama2.c "stories15M" shape, fp32 storage (src/paper_2501_11779_b200/spec.py TINY) */
  gh_model_spec spec = {6, 288, 288, 768, 6, 6, 256, 4, 32000, 10000.f, 1e-5f};
  int32_t prompts[B][PLEN];
  FILE* f = fopen(prompts_path, "r");
  if (!f) return 2;
  for (int b = 0; b < B; ++b)
    for (int i = 0; i < PLEN; ++i)
      if (fscanf(f, "%d", &prompts[b][i]) != 1) return 2;
  fclose(f);

  gh_tier1* t1 = NULL;
  gh_tier2* t2 = NULL;
  CK(gh_tier1_create(&spec, 0, 0, (uint32_t)spec.n_layers, 1234, B, &t1));
  CK(gh_tier2_create(&spec, 0, 0, (uint32_t)spec.n_layers, B, &t2));
  const size_t D = spec.d_model, Dkv = spec.d_kv, db = spec.dtype_bytes;
  void *x, *xn, *fwd, *bwd;
  int32_t *tok_d, *pos_d, *next_d;
  uint32_t* slot_d;
  CU(cudaMalloc(&x, B * D * db));
  CU(cudaMalloc(&xn, B * D * db));
  CU(cudaMalloc(&fwd, B * (2 * D + 2 * Dkv) * db));   /* [x|q|k|v] (PayloadModel fwd) */
  CU(cudaMalloc(&bwd, B * 2 * D * db));               /* [x|attn]  (PayloadModel bwd) */
  CU(cudaMalloc((void**)&tok_d, B * 4));
  CU(cudaMalloc((void**)&pos_d, B * 4));
  CU(cudaMalloc((void**)&next_d, B * 4));
  CU(cudaMalloc((void**)&slot_d, B * 4));
  uint32_t slot[B];
  for (int b = 0; b < B; ++b) slot[b] = (uint32_t)b;
  CU(cudaMemcpy(slot_d, slot, sizeof slot, cudaMemcpyHostToDevice));

  int32_t tok[B], pos[B], next[B], out[B][NEW];
  for (int b = 0; b < B; ++b) tok[b] = prompts[b][0];
  for (int t = 0; t < PLEN - 1 + NEW; ++t) {
    for (int b = 0; b < B; ++b) pos[b] = t;
    CK(gh_tier2_check(t2, B, slot, pos));
    CU(cudaMemcpy(tok_d, tok, sizeof tok, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(pos_d, pos, sizeof pos, cudaMemcpyHostToDevice));
    CK(gh_tier1_embed(t1, B, tok_d, x, NULL));
    for (uint32_t l = 0; l < spec.n_layers; ++l) {
      CK(gh_tier1_pre(t1, l, B, x, pos_d, fwd, NULL));               /* F1 -> [x|q|k|v] */
      CK(gh_tier2_attend(t2, l, B, slot_d, pos_d, fwd, bwd, NULL));  /* F2 + append -> [x|attn] */
      CK(gh_tier1_post(t1, l, B, bwd, xn, NULL));                    /* F3 */
      void* tmp = x; x = xn; xn = tmp;
    }
    CK(gh_tier1_classify(t1, B, x, NULL, next_d, NULL));
    CU(cudaMemcpy(next, next_d, sizeof next, cudaMemcpyDeviceToHost));
    for (int b = 0; b < B; ++b) {
      if (t + 1 < PLEN) {
        tok[b] = prompts[b][t + 1];
      } else {
        out[b][t + 1 - PLEN] = next[b];
        tok[b] = next[b];
      }
    }
  }
  for (int b = 0; b < B; ++b) {
    for (int i = 0; i < NEW; ++i) printf(i ? " %d" : "%d", out[b][i]);
    printf("\n");
  }
  CK(gh_tier1_destroy(t1));
  CK(gh_tier2_destroy(t2));
  cudaFree(x); cudaFree(xn); cudaFree(fwd); cudaFree(bwd);
  cudaFree(tok_d); cudaFree(pos_d); cudaFree(next_d); cudaFree(slot_d);
  return 0;
}

/* The dispatcher's decision logic (gh_sched_*, P:471-479 / P:1117) driven from C against a toy
 * model whose next token hashes the whole context of the row's slot: IF 2 x B 6 lanes, 2 Tier-2
 * shards, 9 requests, with and without chunked prefill.  Every request's tokens must equal
 * decoding it alone; prints {"steps": [chunk 1, chunk 4], "equal": 0/1}. */
enum { SB = 6, SIF = 2, SLANES = SB * SIF, SMAXPOS = 256, SNEW = 7, SREQ = 9 };
static int32_t toy_next(const int32_t* ctx, int n) {
  uint32_t h = 2166136261u;
  for (int i = 0; i < n; ++i) h = (h ^ (uint32_t)ctx[i]) * 16777619u;
  return (int32_t)(h % 1000u);
}
static int sched_run(uint32_t chunk, const int32_t prompts[SREQ][40], const int lens[SREQ], uint64_t* steps,
                     int32_t out[SREQ][SNEW]) {
  gh_sched_config c = {SB, SIF, 2, 0, SMAXPOS, SNEW, 0, 0, 0, chunk};
  gh_sched* s = NULL;
  CK(gh_sched_create(&c, &s));
  uint64_t id[SREQ];
  for (int r = 0; r < SREQ; ++r) CK(gh_sched_submit(s, prompts[r], (uint32_t)lens[r], 0.f, 0, 0, &id[r]));
  static int32_t hist[SLANES][SMAXPOS];
  int32_t last[SLANES] = {0}, next[SLANES];
  gh_lane_input in[SLANES];
  gh_kv_action acts[64];
  uint32_t nacts = 0;
  while (!gh_sched_done(s)) {
    CK(gh_sched_plan(s, in, acts, 64, &nacts));
    for (int l = 0; l < SLANES; ++l) {  /* a prefill-row engine appends every row before attention */
      const int32_t tok = in[l].src == 2 ? last[l] : in[l].tok;
      hist[in[l].home][in[l].pos] = tok;
    }
    for (int l = 0; l < SLANES; ++l) next[l] = toy_next(hist[in[l].home], in[l].pos + 1);
    memcpy(last, next, sizeof last);
    CK(gh_sched_commit(s));
    CK(gh_sched_resolve(s, next));
  }
  gh_dispatch_stats st;
  CK(gh_sched_stats(s, &st));
  *steps = st.steps;
  for (int r = 0; r < SREQ; ++r) {
    uint32_t n = 0;
    CK(gh_sched_result(s, id[r], out[r], SNEW, &n));
    if (n != SNEW) return 1;
  }
  CK(gh_sched_destroy(s));
  return 0;
}
static int run_sched(void) {
  int32_t prompts[SREQ][40];
  int lens[SREQ];
  uint32_t x = 12345u;
  for (int r = 0; r < SREQ; ++r) {
    lens[r] = 1 + (r * 7) % 37;
    for (int i = 0; i < lens[r]; ++i) prompts[r][i] = (int32_t)((x = x * 1103515245u + 12345u) >> 16) % 1000;
  }
  int equal = 1;
  uint64_t steps[2];
  const uint32_t chunks[2] = {1, 4};
  for (int k = 0; k < 2; ++k) {
    int32_t out[SREQ][SNEW];
    if (sched_run(chunks[k], prompts, lens, &steps[k], out)) return 3;
    for (int r = 0; r < SREQ; ++r) {  /* decoding the request alone */
      int32_t ctx[40 + SNEW];
      memcpy(ctx, prompts[r], sizeof(int32_t) * (size_t)lens[r]);
      for (int i = 0; i < SNEW; ++i) {
        ctx[lens[r] + i] = toy_next(ctx, lens[r] + i);
        equal &= ctx[lens[r] + i] == out[r][i];
      }
    }
  }
  printf("{\"steps\": [%llu, %llu], \"equal\": %d}\n", (unsigned long long)steps[0], (unsigned long long)steps[1], equal);
  return 0;
}

int main(int argc, char** argv) {
  if (argc == 2 && strcmp(argv[1], "sched") == 0) return run_sched();
  if (argc == 3 && strcmp(argv[1], "cpu") == 0) return run_cpu(argv[2]);
  if (argc == 3 && strcmp(argv[1], "gpu") == 0) return run_gpu(argv[2]);
  fprintf(stderr, "usage: %s cpu <csv> | gpu <prompts.txt> | sched\n", argv[0]);
  return 1;
}
