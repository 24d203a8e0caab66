// kernels.cu — sm_100a kernels of the two-tier decode path and their host launchers.
//
//   tcgen05 GEMM (gemm_tc.cuh)        Tier-1 dense contractions (bf16 storage)
//   SIMT GEMM + epilogue              Tier-1 contractions for fp32 storage (config C1 only)
//   attention (attention.cuh)         Tier-2 F2 with fused KV append
//   rmsnorm / embed / argmax          small Tier-1 ops
//   init / fill                       deterministic synthetic weights and KV pre-fill
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math.h>
#include <algorithm>
#include <mutex>

#include "attention.cuh"
#include "common.cuh"
#include "gemm_tc.cuh"
#include "kernels.hpp"

namespace gh {

uint64_t& launch_counter() {
  static uint64_t n = 0;
  return n;
}
#define GH_COUNT_LAUNCH() (++launch_counter())

// ====================================================================== init / fill
static float ih_k(double std_) { return (float)(1.7320508075688772 * std_ / 16777216.0); }

template <typename T>
__global__ void init_matrix_kernel(T* dst, uint64_t base, uint64_t n, float k) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    St<T>::store(dst, i, randn_scaled(base, i, k));
}
template <>
__global__ void init_matrix_kernel<float>(float* dst, uint64_t base, uint64_t n, float k) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = randn_scaled(base, i, k);
}

template <typename T>
__global__ void init_interleaved_kernel(T* dst, uint64_t base_even, uint64_t base_odd,
                                        uint64_t pairs, uint64_t cols, float k) {
  const uint64_t n = 2 * pairs * cols;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = i / cols, c = i % cols;
    const uint64_t logical = (r >> 1) * cols + c;
    St<T>::store(dst, i, randn_scaled((r & 1) ? base_odd : base_even, logical, k));
  }
}

template <typename T>
__global__ void fill_const_kernel(T* dst, uint64_t n, float v) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    St<T>::store(dst, i, v);
}

// arena[layer][slot][kv][h][S][DH]; fills p < npos of slots [0, n_slots) of every layer
template <typename T>
__global__ void fill_kv_kernel(T* arena, uint64_t seed, int l0, int n_layers, int n_slots,
                               int n_slots_cap, int Hkv, int S, int DH, int npos, float k) {
  const uint64_t per_block = (uint64_t)Hkv * npos * DH;  // one (layer, slot, kv)
  const uint64_t total = (uint64_t)n_layers * n_slots * 2 * per_block;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t blk = i / per_block, r = i % per_block;
    const int kv = (int)(blk % 2);
    const int slot = (int)((blk / 2) % n_slots);
    const int l = (int)(blk / 2 / n_slots);
    const int h = (int)(r / ((uint64_t)npos * DH));
    const int p = (int)((r / DH) % npos);
    const int d = (int)(r % DH);
    const uint64_t base = tensor_base(seed, tid_kv((uint64_t)(l0 + l), (uint64_t)slot, (uint64_t)kv));
    const uint64_t logical = ((uint64_t)h * S + p) * DH + d;
    const uint64_t phys = ((((uint64_t)l * n_slots_cap + slot) * 2 + kv) * Hkv + h) * (uint64_t)S * DH +
                          (uint64_t)p * DH + d;
    St<T>::store(arena, phys, randn_scaled(base, logical, k));
  }
}

static int grid_for(uint64_t n) {
  uint64_t g = (n + 255) / 256;
  return (int)std::min<uint64_t>(g, (uint64_t)kNumSMs * 32);
}

cudaError_t launch_init_matrix(int db, void* dst, uint64_t seed, uint64_t tid, uint64_t rows,
                               uint64_t cols, double std_, cudaStream_t st) {
  const uint64_t n = rows * cols;
  const uint64_t base = tensor_base(seed, tid);
  GH_COUNT_LAUNCH();
  if (db == 4) init_matrix_kernel<float><<<grid_for(n), 256, 0, st>>>((float*)dst, base, n, ih_k(std_));
  else init_matrix_kernel<bf16_t><<<grid_for(n), 256, 0, st>>>((bf16_t*)dst, base, n, ih_k(std_));
  return cudaGetLastError();
}

cudaError_t launch_init_interleaved(int db, void* dst, uint64_t seed, uint64_t tid_even,
                                    uint64_t tid_odd, uint64_t pairs, uint64_t cols, double std_,
                                    cudaStream_t st) {
  const uint64_t n = 2 * pairs * cols;
  const uint64_t be = tensor_base(seed, tid_even), bo = tensor_base(seed, tid_odd);
  GH_COUNT_LAUNCH();
  if (db == 4)
    init_interleaved_kernel<float><<<grid_for(n), 256, 0, st>>>((float*)dst, be, bo, pairs, cols, ih_k(std_));
  else
    init_interleaved_kernel<bf16_t><<<grid_for(n), 256, 0, st>>>((bf16_t*)dst, be, bo, pairs, cols, ih_k(std_));
  return cudaGetLastError();
}

cudaError_t launch_fill_const(int db, void* dst, uint64_t n, float v, cudaStream_t st) {
  GH_COUNT_LAUNCH();
  if (db == 4) fill_const_kernel<float><<<grid_for(n), 256, 0, st>>>((float*)dst, n, v);
  else fill_const_kernel<bf16_t><<<grid_for(n), 256, 0, st>>>((bf16_t*)dst, n, v);
  return cudaGetLastError();
}

cudaError_t launch_fill_kv(int db, void* arena, uint64_t seed, int l0, int l1, int n_slots,
                           int n_slots_cap, int Hkv, int S, int DH, int npos, cudaStream_t st) {
  if (npos <= 0 || n_slots <= 0 || l1 <= l0) return cudaSuccess;
  const uint64_t total = (uint64_t)(l1 - l0) * n_slots * 2 * Hkv * npos * DH;
  GH_COUNT_LAUNCH();
  if (db == 4)
    fill_kv_kernel<float><<<grid_for(total), 256, 0, st>>>((float*)arena, seed, l0, l1 - l0, n_slots,
                                                           n_slots_cap, Hkv, S, DH, npos, ih_k(1.0));
  else
    fill_kv_kernel<bf16_t><<<grid_for(total), 256, 0, st>>>((bf16_t*)arena, seed, l0, l1 - l0, n_slots,
                                                            n_slots_cap, Hkv, S, DH, npos, ih_k(1.0));
  return cudaGetLastError();
}

// ====================================================================== rmsnorm / embed
// y = x * rsqrt(mean(x^2) + eps) * w  (one CTA per row; fp32 math, storage-dtype result).
// Optionally copies the input row to copy_out (the x slot of the fwd message).
template <typename T>
__global__ void rmsnorm_kernel(const T* x, long ldx, const T* w, T* y, long ldy, T* copy_out,
                               long ldc, int D, float eps) {
  const int b = blockIdx.x;
  const T* xr = x + (long)b * ldx;
  __shared__ float red[32];
  float ss = 0.f;
  for (int i = threadIdx.x; i < D; i += blockDim.x) {
    const float v = St<T>::load(xr, i);
    ss = fmaf(v, v, ss);
  }
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const float inv = 1.0f / sqrtf(red[0] / (float)D + eps);
  T* yr = y + (long)b * ldy;
  for (int i = threadIdx.x; i < D; i += blockDim.x) {
    const float v = St<T>::load(xr, i);
    St<T>::store(yr, i, v * inv * St<T>::load(w, i));
    if (copy_out) copy_out[(long)b * ldc + i] = xr[i];
  }
}

cudaError_t launch_rmsnorm(int db, const void* x, long ldx, const void* w, void* y, long ldy,
                           void* copy_out, long ldc, int B, int D, float eps, cudaStream_t st) {
  if (B <= 0) return cudaSuccess;
  GH_COUNT_LAUNCH();
  if (db == 4)
    rmsnorm_kernel<float><<<B, 256, 0, st>>>((const float*)x, ldx, (const float*)w, (float*)y, ldy,
                                             (float*)copy_out, ldc, D, eps);
  else
    rmsnorm_kernel<bf16_t><<<B, 256, 0, st>>>((const bf16_t*)x, ldx, (const bf16_t*)w, (bf16_t*)y, ldy,
                                              (bf16_t*)copy_out, ldc, D, eps);
  return cudaGetLastError();
}

__global__ void embed_kernel(const uint4* table, const int32_t* tok, uint4* x, int row_vecs, int V) {
  const int b = blockIdx.x;
  int t = tok[b];
  t = t < 0 ? 0 : (t >= V ? V - 1 : t);
  const uint4* src = table + (long)t * row_vecs;
  uint4* dst = x + (long)b * row_vecs;
  for (int i = threadIdx.x; i < row_vecs; i += blockDim.x) dst[i] = src[i];
}

cudaError_t launch_embed(int db, const void* table, const int32_t* tok, void* x, int B, int D,
                         int V, cudaStream_t st) {
  if (B <= 0) return cudaSuccess;
  GH_COUNT_LAUNCH();
  embed_kernel<<<B, 128, 0, st>>>((const uint4*)table, tok, (uint4*)x, D * db / 16, V);
  return cudaGetLastError();
}

// ====================================================================== argmax
GH_DEV void argmax_merge(float& v, int& i, float ov, int oi) {
  if (ov > v || (ov == v && oi < i)) { v = ov; i = oi; }
}
__global__ void argmax_final_kernel(const float2* part, int n_tiles, int B, int32_t* next) {
  const int b = blockIdx.x;
  float v = -INFINITY; int idx = 0x7fffffff;
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
    const float2 p = part[(long)t * B + b];
    argmax_merge(v, idx, p.x, __float_as_int(p.y));
  }
  __shared__ float sv[32]; __shared__ int si[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    argmax_merge(v, idx, __shfl_xor_sync(0xffffffffu, v, o), __shfl_xor_sync(0xffffffffu, idx, o));
  if ((threadIdx.x & 31) == 0) { sv[threadIdx.x >> 5] = v; si[threadIdx.x >> 5] = idx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) argmax_merge(v, idx, sv[w], si[w]);
    next[b] = idx;
  }
}
__global__ void argmax_rows_kernel(const float* logits, int V, int32_t* next) {
  const int b = blockIdx.x;
  const float* r = logits + (long)b * V;
  float v = -INFINITY; int idx = 0x7fffffff;
  for (int i = threadIdx.x; i < V; i += blockDim.x) argmax_merge(v, idx, r[i], i);
  __shared__ float sv[32]; __shared__ int si[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    argmax_merge(v, idx, __shfl_xor_sync(0xffffffffu, v, o), __shfl_xor_sync(0xffffffffu, idx, o));
  if ((threadIdx.x & 31) == 0) { sv[threadIdx.x >> 5] = v; si[threadIdx.x >> 5] = idx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) argmax_merge(v, idx, sv[w], si[w]);
    next[b] = idx;
  }
}
cudaError_t launch_argmax_final(const float2* part, int n_tiles, int B, int32_t* next, cudaStream_t st) {
  GH_COUNT_LAUNCH();
  argmax_final_kernel<<<B, 256, 0, st>>>(part, n_tiles, B, next);
  return cudaGetLastError();
}
cudaError_t launch_argmax_rows(const float* logits, int B, int V, int32_t* next, cudaStream_t st) {
  GH_COUNT_LAUNCH();
  argmax_rows_kernel<<<B, 256, 0, st>>>(logits, V, next);
  return cudaGetLastError();
}

// ====================================================================== batch state
__global__ void advance_kernel(int32_t* tok, const int32_t* next, int32_t* pos, int n, int inc) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) { tok[i] = next[i]; pos[i] += inc; }
}
cudaError_t launch_advance(int32_t* tok, const int32_t* next, int32_t* pos, int n, int inc, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  GH_COUNT_LAUNCH();
  advance_kernel<<<(n + 255) / 256, 256, 0, st>>>(tok, next, pos, n, inc);
  return cudaGetLastError();
}

// ====================================================================== SIMT GEMM (fp32 storage)
// One warp per weight row n, 4 batch columns per warp; lanes stride K (coalesced on W and X).
template <typename T>
__global__ void gemm_simt_kernel(const T* W, const T* X, long ldx, float* Y, int N, int K, int Bt) {
  const int n = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int b0 = blockIdx.y * 4;
  const int lane = threadIdx.x & 31;
  if (n >= N) return;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  const T* wr = W + (long)n * K;
  for (int k = lane; k < K; k += 32) {
    const float w = St<T>::load(wr, k);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (b0 + j < Bt) acc[j] = fmaf(w, St<T>::load(X, (long)(b0 + j) * ldx + k), acc[j]);
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float s = warp_sum(acc[j]);
    if (lane == 0 && b0 + j < Bt) Y[(long)(b0 + j) * N + n] = s;
  }
}
template <typename T>
__global__ void epilogue_simt_kernel(const float* Y, int N, int Bt, const EpiParams ep) {
  const long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (i >= (long)N * Bt) return;
  const int b = (int)(i / N), n = (int)(i % N);
  const float partner = Y[(long)b * N + (n ^ 1)];
  epi_store_one<T>(ep, n, b, Y[i], partner);
}

// ====================================================================== tcgen05 GEMM dispatch
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  });
  return fn;
}

cudaError_t make_tmap_bf16(CUtensorMap* out, const void* base, uint64_t rows, uint64_t cols,
                           uint64_t ld, uint32_t box_rows) {
  auto enc = get_encode();
  if (!enc) return cudaErrorNotSupported;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

static const int kBNs[] = {16, 32, 48, 64, 96, 128, 192, 256};
static int ctas_per_sm(int BN) { return BN <= 96 ? 2 : 1; }

GemmPlan plan_gemm(int N, int K, int Bt) {
  GemmPlan p;
  int bt_cap = std::min(Bt, 256);
  p.BN = 256;
  for (int bn : kBNs) if (bn >= bt_cap) { p.BN = bn; break; }
  p.b_tiles = (Bt + p.BN - 1) / p.BN;
  p.n_tiles = (N + kBlockM - 1) / kBlockM;
  const int kb_total = (K + kBlockK - 1) / kBlockK;
  const int tiles = p.n_tiles * p.b_tiles;
  const int slots = kNumSMs * ctas_per_sm(p.BN);
  // time model (arbitrary units): streaming time of the busiest SM + split fix-up reads
  const double tile_bytes = (double)kBlockM * K * 2 + (double)p.BN * K * 2;
  const double partial = (double)kBlockM * p.BN * 4;
  double best = 1e300;
  int best_ks = 1;
  const int ks_max = std::max(1, std::min(16, kb_total / 4));
  for (int ks = 1; ks <= ks_max; ++ks) {
    const int ctas = tiles * ks;
    const int waves = (ctas + slots - 1) / slots;
    const int per_sm = std::min(ctas_per_sm(p.BN), (ctas + kNumSMs - 1) / kNumSMs);
    const double stream = waves * (tile_bytes / ks) * per_sm / 44.0;  // ns @ 44 GB/s per SM
    const double fix = ks > 1 ? (ks * partial) / 100.0 + 1500.0 : 0.0;  // ns
    const double t = stream + fix;
    if (t < best * 0.97) { best = t; best_ks = ks; }
  }
  p.ks = best_ks;
  if (p.ks > 1) {
    p.ws_floats = (size_t)tiles * p.ks * kBlockM * p.BN;
    p.tickets = (size_t)tiles;
  }
  return p;
}

// pipeline depth per batch tile: <= ~113 KB (2 CTAs / SM) for BN <= 96, else ~200 KB
template <int BN> struct TcStages {
  static constexpr int value = (BN == 16) ? 6 : (BN == 32 || BN == 48) ? 5
                             : (BN == 64 || BN == 96) ? 4 : (BN == 128) ? 6 : (BN == 192) ? 5 : 4;
};
template <int BN>
static cudaError_t configure_tc() {
  constexpr int S = TcStages<BN>::value;
  return cudaFuncSetAttribute(gemm_tc_kernel<BN, S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              GemmSmem<BN, S>::kTotal);
}
template <int BN>
static cudaError_t launch_tc(const CUtensorMap* tmW, const CUtensorMap* tmX, const GemmShape& gs,
                             const GemmPlan& p, const EpiParams& ep, cudaStream_t st) {
  constexpr int S = TcStages<BN>::value;
  using L = GemmSmem<BN, S>;
  dim3 grid(p.n_tiles, p.b_tiles, p.ks);
  GH_COUNT_LAUNCH();
  gemm_tc_kernel<BN, S><<<grid, kGemmThreads, L::kTotal, st>>>(*tmW, *tmX, gs, ep);
  return cudaGetLastError();
}

cudaError_t launch_gemm(const Weight& W, const CUtensorMap* tmW, const void* X, long ldx,
                        const CUtensorMap* tmX, int Bt, const GemmPlan& p, const EpiParams& ep,
                        const GemmScratch& sc, cudaStream_t st) {
  if (Bt <= 0) return cudaSuccess;
  if (W.dtype_bytes == 4) {
    // fp32 storage: CUDA-core GEMM into fp32 staging, then the scalar epilogue
    if ((size_t)Bt * W.N > sc.stage_floats) return cudaErrorInvalidValue;
    float* Y = (ep.kind == EPI_LOGITS_ARGMAX && ep.logits) ? ep.logits : sc.stage;
    dim3 grid((W.N + 7) / 8, (Bt + 3) / 4);
    GH_COUNT_LAUNCH();
    gemm_simt_kernel<float><<<grid, 256, 0, st>>>((const float*)W.ptr, (const float*)X, ldx, Y, W.N, W.K, Bt);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (ep.kind == EPI_LOGITS_ARGMAX) return cudaSuccess;  // caller runs argmax_rows on Y
    const long n = (long)W.N * Bt;
    GH_COUNT_LAUNCH();
    epilogue_simt_kernel<float><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(Y, W.N, Bt, ep);
    return cudaGetLastError();
  }
  GemmShape gs;
  gs.N = W.N; gs.K = W.K; gs.Bt = Bt; gs.ks = p.ks;
  gs.kb_total = (W.K + kBlockK - 1) / kBlockK;
  gs.ws = sc.ws; gs.tickets = sc.tickets;
  if (p.ks > 1 && (p.ws_floats > sc.ws_floats || p.tickets > sc.n_tickets)) return cudaErrorInvalidValue;
  switch (p.BN) {
    case 16: return launch_tc<16>(tmW, tmX, gs, p, ep, st);
    case 32: return launch_tc<32>(tmW, tmX, gs, p, ep, st);
    case 48: return launch_tc<48>(tmW, tmX, gs, p, ep, st);
    case 64: return launch_tc<64>(tmW, tmX, gs, p, ep, st);
    case 96: return launch_tc<96>(tmW, tmX, gs, p, ep, st);
    case 128: return launch_tc<128>(tmW, tmX, gs, p, ep, st);
    case 192: return launch_tc<192>(tmW, tmX, gs, p, ep, st);
    case 256: return launch_tc<256>(tmW, tmX, gs, p, ep, st);
  }
  return cudaErrorInvalidValue;
}

// ====================================================================== attention dispatch
template <typename T, int DH>
static cudaError_t configure_attn() {
  return cudaFuncSetAttribute(attn_decode_kernel<T, DH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              AttnCfg<T, DH>::kSmem);
}
template <typename T, int DH>
static cudaError_t launch_attn_t(const AttnArgs& a, cudaStream_t st) {
  using C = AttnCfg<T, DH>;
  const int units = a.B * a.H;
  if (units <= 0) return cudaSuccess;
  const int grid = std::min(units, kNumSMs);
  GH_COUNT_LAUNCH();
  attn_decode_kernel<T, DH><<<grid, C::kThreads, C::kSmem, st>>>(a);
  return cudaGetLastError();
}

bool attention_supported(int db, int dh) {
  return (db == 2 || db == 4) && (dh == 48 || dh == 64 || dh == 128);
}

cudaError_t launch_attention(int db, int dh, const AttnArgs& a, cudaStream_t st) {
  if (db == 2) {
    switch (dh) {
      case 48: return launch_attn_t<bf16_t, 48>(a, st);
      case 64: return launch_attn_t<bf16_t, 64>(a, st);
      case 128: return launch_attn_t<bf16_t, 128>(a, st);
    }
  } else if (db == 4) {
    switch (dh) {
      case 48: return launch_attn_t<float, 48>(a, st);
      case 64: return launch_attn_t<float, 64>(a, st);
      case 128: return launch_attn_t<float, 128>(a, st);
    }
  }
  return cudaErrorInvalidValue;
}

cudaError_t configure_kernels() {
  cudaError_t e = cudaSuccess;
  auto chk = [&](cudaError_t r) { if (e == cudaSuccess) e = r; };
  chk(configure_tc<16>()); chk(configure_tc<32>()); chk(configure_tc<48>()); chk(configure_tc<64>());
  chk(configure_tc<96>()); chk(configure_tc<128>()); chk(configure_tc<192>()); chk(configure_tc<256>());
  chk(configure_attn<bf16_t, 48>()); chk(configure_attn<bf16_t, 64>()); chk(configure_attn<bf16_t, 128>());
  chk(configure_attn<float, 48>()); chk(configure_attn<float, 64>()); chk(configure_attn<float, 128>());
  return e;
}

}  // namespace gh
