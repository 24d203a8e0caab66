/*
 * smoke.c — a compiled C consumer of include/gh/gh.h (C11, no C++), i.e. what a reference-side
 * maintainer links: `cc -std=c11 -I include smoke.c -L paper_2501_11779_b200 -lgh -lcudart`.
 *
 *   smoke cpu <csv_path>       accounting calls (model.cpp:40-77, netmodel.cpp:18-24,
 *                              optimizer.cpp:116-192) and the profile CSV producer
 *                              (profiles.hpp:66-69); prints one JSON line.  No GPU needed.
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

int main(int argc, char** argv) {
  if (argc == 3 && strcmp(argv[1], "cpu") == 0) return run_cpu(argv[2]);
  if (argc == 3 && strcmp(argv[1], "gpu") == 0) return run_gpu(argv[2]);
  fprintf(stderr, "usage: %s cpu <csv> | gpu <prompts.txt>\n", argv[0]);
  return 1;
}
