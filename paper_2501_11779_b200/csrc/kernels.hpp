// kernels.hpp — host-side launch interface of the sm_100a kernels (C++; not part of the ABI).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace gh {

struct EpiParams;

// Dense weight matrix W[N, K] (row-major, K contiguous) in device memory.
struct Weight {
  void* ptr = nullptr;
  int N = 0, K = 0;
  int dtype_bytes = 2;
};

// Per-GEMM launch plan (split-K factor, batch tile) chosen on the host.
struct GemmPlan {
  int BN = 0;       // batch tile (16..256)
  int ks = 1;       // K splits
  int n_tiles = 0;  // ceil(N / 128)
  int b_tiles = 0;
  size_t ws_floats = 0;   // split workspace
  size_t tickets = 0;
};
GemmPlan plan_gemm(int N, int K, int Bt);

// Scratch shared by every GEMM of a tier (split workspace, tickets, SIMT staging).
struct GemmScratch {
  float* ws = nullptr;     size_t ws_floats = 0;
  int* tickets = nullptr;  size_t n_tickets = 0;
  float* stage = nullptr;  size_t stage_floats = 0;  // SIMT path fp32 result [Bt][N]
};

// Encode a 2-D bf16 tensor map over a row-major [rows, cols] matrix with row stride ld
// (elements), box {64, box_rows}, 128-byte swizzle.
cudaError_t make_tmap_bf16(CUtensorMap* out, const void* base, uint64_t rows, uint64_t cols,
                           uint64_t ld, uint32_t box_rows);

// Y = X W^T with a fused epilogue.  X: [Bt, K] storage dtype, row stride ldx.
//  bf16: tcgen05 kernel (tmX must describe X with box rows = plan.BN).
//  fp32: SIMT kernel + epilogue kernel (tmX ignored).
cudaError_t launch_gemm(const Weight& W, const CUtensorMap* tmW, const void* X, long ldx,
                        const CUtensorMap* tmX, int Bt, const GemmPlan& plan,
                        const EpiParams& ep, const GemmScratch& scratch, cudaStream_t st);

cudaError_t launch_rmsnorm(int dtype_bytes, const void* x, long ldx, const void* w, void* y,
                           long ldy, void* copy_out, long ldc, int B, int D, float eps,
                           cudaStream_t st);
cudaError_t launch_embed(int dtype_bytes, const void* table, const int32_t* tok, void* x, int B,
                         int D, int V, cudaStream_t st);
cudaError_t launch_argmax_final(const float2* part, int n_tiles, int B, int32_t* next_tok,
                                cudaStream_t st);
cudaError_t launch_argmax_rows(const float* logits, int B, int V, int32_t* next_tok,
                               cudaStream_t st);

struct AttnArgs;
cudaError_t launch_attention(int dtype_bytes, int d_head, const AttnArgs& a, cudaStream_t st);
bool attention_supported(int dtype_bytes, int d_head);

// Synthetic initialisation (deterministic, see common.cuh / DESIGN.md)
// Logical matrix [rows, cols] of tensor `tid` with std `std_`; `row_map` selects which logical
// row lands in physical row r: logical = r for map 0, interleave (r even -> gate r/2 of tidA,
// r odd -> up r/2 of tidB) for map 1.
cudaError_t launch_init_matrix(int dtype_bytes, void* dst, uint64_t seed, uint64_t tid,
                               uint64_t rows, uint64_t cols, double std_, cudaStream_t st);
cudaError_t launch_init_interleaved(int dtype_bytes, void* dst, uint64_t seed, uint64_t tid_even,
                                    uint64_t tid_odd, uint64_t pairs, uint64_t cols, double std_,
                                    cudaStream_t st);
cudaError_t launch_fill_const(int dtype_bytes, void* dst, uint64_t n, float v, cudaStream_t st);
// Fill positions [0, npos) of K and V blocks of `n_slots` slots for layers [l0, l1).
cudaError_t launch_fill_kv(int dtype_bytes, void* arena, uint64_t seed, int l0, int l1,
                           int n_slots, int n_slots_cap, int Hkv, int S, int DH, int npos,
                           cudaStream_t st);
// Set dynamic shared-memory limits of every kernel instantiation (call before graph capture).
cudaError_t configure_kernels();

cudaError_t launch_advance(int32_t* tok, const int32_t* next, int32_t* pos, int n, int inc,
                           cudaStream_t st);

uint64_t& launch_counter();

}  // namespace gh
