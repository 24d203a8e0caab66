// kernels.hpp — host-side launch interface of the sm_100a kernels (C++; not part of the ABI).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace gh {

struct EpiParams;

// Dense weight matrix W[N, K] in device memory.
//  row-major (K contiguous) for fp32 storage;
//  "tile-contiguous" for bf16 (tcgen05 operand): W is cut into 128 x 64 tiles (rows x K), tile
//  (nt, kb) is one contiguous 16 KB block at ((nt * KB + kb) * 128 + r) * 64 + c, zero padded to
//  N_pad = ceil(N/128)*128 and KB = ceil(K/64).  Every TMA box of the GEMM mainloop is therefore
//  one contiguous 16 KB burst of HBM instead of 128 segments of 128 B strided by K.
struct Weight {
  void* ptr = nullptr;
  int N = 0, K = 0;
  int dtype_bytes = 2;
  bool tiled = false;
  int n_pad() const { return (N + 127) / 128 * 128; }
  int kb() const { return (K + 63) / 64; }
  size_t elems() const { return tiled ? (size_t)n_pad() * kb() * 64 : (size_t)N * K; }
};

// Logical source rows of a weight: up to 3 stacked synthetic tensors (e.g. Wq|Wk|Wv), or two
// row-interleaved tensors (W1/W3: physical row 2f = gate f, 2f+1 = up f).
struct RowSegs {
  uint64_t base[3];   // tensor_base(seed, tid) per segment
  int rows[3];        // logical rows per segment (stacked mode)
  float k[3];         // sqrt(3) * std / 2^24 per segment
  int n = 1;
  int interleave2 = 0;
  // Tensor-parallel slice of the logical tensors: physical (r, k) of segment s is logical
  // (row0[s] + r, k0 + k) of a matrix with ldk logical columns (0 = K, no slicing).
  int row0[3] = {0, 0, 0};
  int k0 = 0;
  int ldk = 0;
};

// Per-GEMM launch plan chosen on the host: batch tile and persistent cluster split-K grid.
//  split-K kernel (gemm_tc.cuh): 128-row tiles, clusters of C CTAs split K;
//  pair kernel (gemm_pair.cuh, large batches): 256-row tiles on CTA pairs (C = 2), no K split.
struct GemmPlan {
  bool pair = false;
  bool split = false;  // pair kernel: stream-K k-block ranges (else contiguous tile ranges)
  int BN = 0;         // batch tile (split-K: 16, 32, 64, 128; pair: multiple of 32 up to 256)
  int n_tiles = 0;    // ceil(N / 128), pair: ceil(N / 256)
  int b_tiles = 0;
  int C = 1;          // CTAs per cluster (split-K: K splits 1, 2, 4; pair: 2)
  int n_clusters = 0; // persistent clusters (<= co-resident clusters)
  int slices() const { return n_tiles * C; }  // 128-row (or 128/C-row) output slices: argmax / norm partials
  int x_box_rows() const { return pair ? BN / 2 : BN; }  // activation rows per TMA box
};
// Largest batch whose RMSNorm can be fused into the consuming GEMM's epilogue (the planner
// uses the pair kernel, whose scale table holds 1024 columns, for every batch above 256).
constexpr int kFusedNormMaxBatch = 1024;
GemmPlan plan_gemm(int N, int K, int Bt);
// Plan of a GEMM whose epilogue all-reduces across tensor-parallel ranks: the cluster split-K
// kernel with batch tiles of at most 128 columns (every rank runs the identical plan, so the
// slices the ranks exchange coincide)
GemmPlan plan_gemm_tp(int N, int K, int Bt);

// Scratch shared by every GEMM of a tier (SIMT staging, diagnostics).
struct GemmScratch {
  float* stage = nullptr;  size_t stage_floats = 0;  // SIMT path fp32 result [Bt][N]
  int debug_flags = 0;                                // GEMM_DBG_* (diagnostics only)
  unsigned long long* trace = nullptr;                // per-CTA timestamps (diagnostics only)
  float* sk_ws = nullptr;                             // pair kernel stream-K partials (kSkWsBytes)
  unsigned int* sk_flags = nullptr;                   // [kNumSMs] zero-initialised
  const unsigned int* xwait = nullptr;                // GemmShape::xwait (peer-delivered rows)
  int xwait_n = 0;
  unsigned int xwait_val = 0;
};
constexpr size_t kSkWsBytes = (size_t)74 * 256 * 256 * 4;  // co-resident pairs x 256 columns x 256 rows fp32
void gemm_debug_set(int stages);  // 0 = production pipeline depth
void gemm_debug_cluster(int C);   // 0 = production cluster-size choice
void gemm_debug_pair(int mode);   // 0 = planner's choice, 1 = force split-K (B <= 256), 2 = force pair
void gemm_debug_wide(int mode);   // 0 = planner's choice, 1 = no 192-column tile, 2 = force it

// Encode a 2-D bf16 tensor map over a row-major [rows, cols] matrix with row stride ld
// (elements), box {64, box_rows}, 128-byte swizzle.
cudaError_t make_tmap_bf16(CUtensorMap* out, const void* base, uint64_t rows, uint64_t cols,
                           uint64_t ld, uint32_t box_rows);

// Y = X W^T with a fused epilogue.  X: [Bt, K] storage dtype, row stride ldx.
//  bf16: tcgen05 kernel (tmX must describe X with box rows = plan.BN).
//  fp32: SIMT kernel + epilogue kernel (tmX ignored).
cudaError_t launch_gemm(const Weight& W, const CUtensorMap* tmW, const void* X, long ldx,
                        const CUtensorMap* tmX, int Bt, const GemmPlan& plan,
                        const EpiParams& ep, const GemmScratch& scratch, cudaStream_t st,
                        const void* pf = nullptr, size_t pf_bytes = 0);  // L2 prefetch of the next weights

cudaError_t make_tmap_kv(CUtensorMap* out, const void* base, uint64_t rows, uint64_t positions, uint64_t dh);

cudaError_t launch_rmsnorm(int dtype_bytes, const void* x, long ldx, const void* w, void* y,
                           long ldy, void* copy_out, long ldc, int B, int D, float eps,
                           cudaStream_t st);
cudaError_t launch_embed(int dtype_bytes, const void* table, const int32_t* tok, void* x, int B,
                         int D, int V, float* ss, cudaStream_t st);
cudaError_t launch_argmax_final(const float2* part, int n_tiles, int B, int32_t* next_tok,
                                cudaStream_t st);
// (inv_temp / seed / pos: temperature sampling per row, common.cuh; nullptr = greedy)
cudaError_t launch_argmax_rows(const float* logits, int B, int V, int32_t* next_tok,
                               cudaStream_t st, const float* inv_temp = nullptr,
                               const uint32_t* seed = nullptr, const int* pos = nullptr);

struct AttnArgs;
cudaError_t launch_attention(int dtype_bytes, int d_head, const AttnArgs& a, cudaStream_t st);
bool attention_supported(int dtype_bytes, int d_head);
// Write every row's key / value (fwd message) into the arena at (slot[b], pos[b]).
cudaError_t launch_append_kv(int dtype_bytes, int d_head, const AttnArgs& a, cudaStream_t st);

// Synthetic initialisation (deterministic, see common.cuh / DESIGN.md)
// Logical matrix [rows, cols] of tensor `tid` with std `std_`; `row_map` selects which logical
// row lands in physical row r: logical = r for map 0, interleave (r even -> gate r/2 of tidA,
// r odd -> up r/2 of tidB) for map 1.
RowSegs make_segs(uint64_t seed, int n, const uint64_t* tids, const int* rows, const double* stds,
                  bool interleave2);
// Generate W (logical [N, K] from `segs`) in W's layout (row-major or tile-contiguous).
cudaError_t launch_init_weight(const Weight& W, const RowSegs& segs, cudaStream_t st);
cudaError_t launch_fill_const(int dtype_bytes, void* dst, uint64_t n, float v, cudaStream_t st);
struct AttnArgs;
// Fill positions [0, npos) of K and V of slots [0, n_slots) for layers [l0, l1); `lay` holds the
// arena layout (strides, page table) of one layer, layer_stride the elements per layer; `limit`
// (device [n_slots], may be null) caps each slot's filled positions.
cudaError_t launch_fill_kv(int dtype_bytes, void* arena, uint64_t seed, int l0, int l1, int n_slots,
                           long layer_stride, const AttnArgs& lay, const int* limit, int Hkv, int S, int DH,
                           int npos, cudaStream_t st);
// Set dynamic shared-memory limits of every kernel instantiation (call before graph capture).
cudaError_t configure_kernels();

cudaError_t launch_advance(int32_t* tok, const int32_t* next, int32_t* pos, int n, int inc,
                           cudaStream_t st);
// dispatcher inputs: in = [src (0 idle, 1 host, 2 device feedback) | tok | pos] x n
cudaError_t launch_dispatch_inputs(int32_t* tok, const int32_t* next, int32_t* pos, const int32_t* in, int n,
                                   cudaStream_t st);

uint64_t& launch_counter();

}  // namespace gh
