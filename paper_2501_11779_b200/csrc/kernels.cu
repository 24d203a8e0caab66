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
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>

#include "attention.cuh"
#include "attention_gqa.cuh"
#include "common.cuh"
#include "gemm_pair.cuh"
#include "gemm_tc.cuh"
#include "kernels.hpp"

namespace gh {

uint64_t& launch_counter() {
  static uint64_t n = 0;
  return n;
}
#define GH_COUNT_LAUNCH() (++launch_counter())

// launch with programmatic stream serialization (PDL), see common.cuh
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  static const bool pdl = getenv("GH_NO_PDL") == nullptr;  // diagnostics A/B switch
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  GH_COUNT_LAUNCH();
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// ====================================================================== init / fill
static float ih_k(double std_) { return (float)(1.7320508075688772 * std_ / 16777216.0); }

template <typename T>
__global__ void init_weight_kernel(T* dst, uint64_t n_phys, int N, int K, int KB, int tiled, RowSegs sg) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_phys;
       i += (uint64_t)gridDim.x * blockDim.x) {
    int n, k;
    if (tiled) {
      const uint64_t tile = i >> 13, w = i & 8191;
      n = (int)((tile / KB) * 128 + (w >> 6));
      k = (int)((tile % KB) * 64 + (w & 63));
    } else {
      n = (int)(i / K);
      k = (int)(i % K);
    }
    float v = 0.f;
    if (n < N && k < K) {
      int seg, r;
      if (sg.interleave2) { seg = n & 1; r = n >> 1; }
      else {
        seg = 0; r = n;
        while (seg + 1 < sg.n && r >= sg.rows[seg]) { r -= sg.rows[seg]; ++seg; }
      }
      const uint64_t ldk = sg.ldk ? (uint64_t)sg.ldk : (uint64_t)K;
      v = randn_scaled(sg.base[seg], (uint64_t)(sg.row0[seg] + r) * ldk + (uint64_t)(sg.k0 + k), sg.k[seg]);
    }
    St<T>::store(dst, i, v);
  }
}

template <typename T>
__global__ void fill_const_kernel(T* dst, uint64_t n, float v) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    St<T>::store(dst, i, v);
}

// Fills p < npos of slots [0, n_slots) of every layer; `lay` gives the physical layout (contiguous
// slots or pages, kv_offset) and the value depends only on the logical (layer, slot, kv, h, p, d).
template <typename T>
__global__ void fill_kv_kernel(T* arena, uint64_t seed, int l0, int n_layers, int n_slots, long layer_stride,
                               const AttnArgs lay, const int* limit, int Hkv, int S, int DH, int npos, float k) {
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
    if (limit && p >= limit[slot]) continue;  // paged: positions past the slot's mapping
    const uint64_t base = tensor_base(seed, tid_kv((uint64_t)(l0 + l), (uint64_t)slot, (uint64_t)kv));
    const uint64_t logical = ((uint64_t)h * S + p) * DH + d;
    const uint64_t phys = (uint64_t)l * layer_stride + kv_offset(lay, slot, h, p, DH) + kv * lay.kv_stride + d;
    St<T>::store(arena, phys, randn_scaled(base, logical, k));
  }
}

// Append the key / value of every row of the fwd message to the arena at (slot[b], pos[b]) ahead of
// the attention kernel, for steps in which several rows of one prompt (chunked prefill) attend
// each other's positions.  16 bytes per thread; either arena layout (kv_offset).
template <typename T>
__global__ void append_kv_kernel(const AttnArgs a, int DH) {
  constexpr int kVec = 16 / sizeof(T);
  griddep_launch_dependents();
  griddep_wait();  // the fwd message comes from the QKV GEMM
  const int per_row = 2 * a.Dkv / kVec;
  const long total = (long)a.B * per_row;
  const T* fwd = (const T*)a.msg_fwd;
  T* arena = (T*)a.arena;
  const long ld_fwd = 2L * a.D + 2L * a.Dkv;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const int b = (int)(i / per_row), r = (int)(i % per_row) * kVec;
    const int kv = r / a.Dkv, e = r % a.Dkv, h = e / DH, d = e % DH;
    const uint4 v = *(const uint4*)(fwd + b * ld_fwd + 2L * a.D + r);
    *(uint4*)(arena + kv_offset(a, (int)a.slot[b], h, a.pos[b], DH) + kv * a.kv_stride + d) = v;
  }
}

static int grid_for(uint64_t n) {
  uint64_t g = (n + 255) / 256;
  return (int)std::min<uint64_t>(g, (uint64_t)kNumSMs * 32);
}

RowSegs make_segs(uint64_t seed, int n, const uint64_t* tids, const int* rows, const double* stds,
                  bool interleave2) {
  RowSegs sg{};
  sg.n = n;
  sg.interleave2 = interleave2 ? 1 : 0;
  for (int i = 0; i < n; ++i) {
    sg.base[i] = tensor_base(seed, tids[i]);
    sg.rows[i] = rows[i];
    sg.k[i] = ih_k(stds[i]);
  }
  return sg;
}

cudaError_t launch_init_weight(const Weight& W, const RowSegs& sg, cudaStream_t st) {
  const uint64_t n = W.elems();
  GH_COUNT_LAUNCH();
  if (W.dtype_bytes == 4)
    init_weight_kernel<float><<<grid_for(n), 256, 0, st>>>((float*)W.ptr, n, W.N, W.K, W.kb(), W.tiled, sg);
  else
    init_weight_kernel<bf16_t><<<grid_for(n), 256, 0, st>>>((bf16_t*)W.ptr, n, W.N, W.K, W.kb(), W.tiled, sg);
  return cudaGetLastError();
}

cudaError_t launch_fill_const(int db, void* dst, uint64_t n, float v, cudaStream_t st) {
  GH_COUNT_LAUNCH();
  if (db == 4) fill_const_kernel<float><<<grid_for(n), 256, 0, st>>>((float*)dst, n, v);
  else fill_const_kernel<bf16_t><<<grid_for(n), 256, 0, st>>>((bf16_t*)dst, n, v);
  return cudaGetLastError();
}

cudaError_t launch_fill_kv(int db, void* arena, uint64_t seed, int l0, int l1, int n_slots, long layer_stride,
                           const AttnArgs& lay, const int* limit, int Hkv, int S, int DH, int npos, cudaStream_t st) {
  if (npos <= 0 || n_slots <= 0 || l1 <= l0) return cudaSuccess;
  const uint64_t total = (uint64_t)(l1 - l0) * n_slots * 2 * Hkv * npos * DH;
  GH_COUNT_LAUNCH();
  if (db == 4)
    fill_kv_kernel<float><<<grid_for(total), 256, 0, st>>>((float*)arena, seed, l0, l1 - l0, n_slots, layer_stride,
                                                           lay, limit, Hkv, S, DH, npos, ih_k(1.0));
  else
    fill_kv_kernel<bf16_t><<<grid_for(total), 256, 0, st>>>((bf16_t*)arena, seed, l0, l1 - l0, n_slots,
                                                            layer_stride, lay, limit, Hkv, S, DH, npos, ih_k(1.0));
  return cudaGetLastError();
}

// ====================================================================== rmsnorm / embed
// y = x * rsqrt(mean(x^2) + eps) * w  (one CTA per row; fp32 math, storage-dtype result).
// 16-byte vector loads, the row stays in registers between the reduction and the scaling.
// Optionally copies the input row to copy_out (the x slot of the fwd message).
template <typename T, int kMaxVec>
__global__ void __launch_bounds__(128) rmsnorm_kernel(const T* x, long ldx, const T* w, T* y, long ldy,
                                                      T* copy_out, long ldc, int D, float eps) {
  constexpr int kV = 16 / sizeof(T);
  const int b = blockIdx.x;
  const int nv = D / kV;
  const uint4* xr = (const uint4*)(x + (long)b * ldx);
  griddep_launch_dependents();
  griddep_wait();
  __shared__ float red[4];
  uint4 buf[kMaxVec];
  float ss = 0.f;
#pragma unroll
  for (int j = 0; j < kMaxVec; ++j) {
    const int i = threadIdx.x + j * 128;
    if (i < nv) {
      buf[j] = xr[i];
      float f[kV];
      chunk_to_f32<T>(buf[j], f);
#pragma unroll
      for (int e = 0; e < kV; ++e) ss = fmaf(f[e], f[e], ss);
    }
  }
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  const float tot = (red[0] + red[1]) + (red[2] + red[3]);
  const float inv = 1.0f / sqrtf(tot / (float)D + eps);
  const uint4* wr = (const uint4*)w;
  uint4* yr = (uint4*)(y + (long)b * ldy);
  uint4* cr = copy_out ? (uint4*)(copy_out + (long)b * ldc) : nullptr;
#pragma unroll
  for (int j = 0; j < kMaxVec; ++j) {
    const int i = threadIdx.x + j * 128;
    if (i < nv) {
      float f[kV], g[kV];
      chunk_to_f32<T>(buf[j], f);
      chunk_to_f32<T>(wr[i], g);
      uint4 o;
      pack_f32<T>(f, g, inv, o);
      yr[i] = o;
      if (cr) cr[i] = buf[j];
    }
  }
}

cudaError_t launch_rmsnorm(int db, const void* x, long ldx, const void* w, void* y, long ldy,
                           void* copy_out, long ldc, int B, int D, float eps, cudaStream_t st) {
  if (B <= 0) return cudaSuccess;
  const int nv = D * db / 16;
  if (nv > 128 * 16 || (D * db) % 16) return cudaErrorInvalidValue;
  if (db == 4)
    return launch_pdl(rmsnorm_kernel<float, 16>, B, 128, 0, st, (const float*)x, ldx, (const float*)w,
                      (float*)y, ldy, (float*)copy_out, ldc, D, eps);
  if (nv <= 128 * 4)
    return launch_pdl(rmsnorm_kernel<bf16_t, 4>, B, 128, 0, st, (const bf16_t*)x, ldx, (const bf16_t*)w,
                      (bf16_t*)y, ldy, (bf16_t*)copy_out, ldc, D, eps);
  return launch_pdl(rmsnorm_kernel<bf16_t, 16>, B, 128, 0, st, (const bf16_t*)x, ldx, (const bf16_t*)w,
                    (bf16_t*)y, ldy, (bf16_t*)copy_out, ldc, D, eps);
}

// x[b] = E[tok[b]]; optionally ss[b] = sum of squares of the row (fused RMSNorm of layer 0)
template <typename T>
__global__ void embed_kernel(const uint4* table, const int32_t* tok, uint4* x, int row_vecs, int V, float* ss) {
  const int b = blockIdx.x;
  griddep_launch_dependents();
  griddep_wait();
  int t = tok[b];
  t = t < 0 ? 0 : (t >= V ? V - 1 : t);
  const uint4* src = table + (long)t * row_vecs;
  uint4* dst = x + (long)b * row_vecs;
  float sq = 0.f;
  for (int i = threadIdx.x; i < row_vecs; i += blockDim.x) {
    const uint4 c = src[i];
    dst[i] = c;
    float f[16 / sizeof(T)];
    chunk_to_f32<T>(c, f);
#pragma unroll
    for (int e = 0; e < (int)(16 / sizeof(T)); ++e) sq = fmaf(f[e], f[e], sq);
  }
  if (ss) {
    __shared__ float red[4];
    sq = warp_sum(sq);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
    __syncthreads();
    if (threadIdx.x == 0) ss[b] = (red[0] + red[1]) + (red[2] + red[3]);
  }
}

cudaError_t launch_embed(int db, const void* table, const int32_t* tok, void* x, int B, int D, int V, float* ss,
                         cudaStream_t st) {
  if (B <= 0) return cudaSuccess;
  if (db == 4)
    return launch_pdl(embed_kernel<float>, B, 128, 0, st, (const uint4*)table, tok, (uint4*)x, D * db / 16, V, ss);
  return launch_pdl(embed_kernel<bf16_t>, B, 128, 0, st, (const uint4*)table, tok, (uint4*)x, D * db / 16, V, ss);
}

// ====================================================================== argmax
GH_DEV void argmax_merge(float& v, int& i, float ov, int oi) {
  if (ov > v || (ov == v && oi < i)) { v = ov; i = oi; }
}
__global__ void argmax_final_kernel(const float2* part, int n_tiles, int B, int32_t* next) {
  const int b = blockIdx.x;
  griddep_launch_dependents();
  griddep_wait();
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
__global__ void argmax_rows_kernel(const float* logits, int V, int32_t* next, const float* inv_temp,
                                   const uint32_t* seed, const int* pos) {
  const int b = blockIdx.x;
  griddep_launch_dependents();
  griddep_wait();
  const float* r = logits + (long)b * V;
  float v = -INFINITY; int idx = 0x7fffffff;
  const float it = inv_temp ? inv_temp[b] : 0.f;
  if (it > 0.f) {  // temperature sampling (common.cuh)
    const uint64_t key = sample_key(seed[b], pos[b]);
    for (int i = threadIdx.x; i < V; i += blockDim.x) argmax_merge(v, idx, sample_score(r[i], it, key, i), i);
  } else {
    for (int i = threadIdx.x; i < V; i += blockDim.x) argmax_merge(v, idx, r[i], i);
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
cudaError_t launch_argmax_final(const float2* part, int n_tiles, int B, int32_t* next, cudaStream_t st) {
  return launch_pdl(argmax_final_kernel, B, 256, 0, st, part, n_tiles, B, next);
}
cudaError_t launch_argmax_rows(const float* logits, int B, int V, int32_t* next, cudaStream_t st,
                               const float* inv_temp, const uint32_t* seed, const int* pos) {
  return launch_pdl(argmax_rows_kernel, B, 256, 0, st, logits, V, next, inv_temp, seed, pos);
}

// ====================================================================== batch state
__global__ void advance_kernel(int32_t* tok, const int32_t* next, int32_t* pos, int n, int inc) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  // no early griddepcontrol.launch_dependents: the next step's kernels start only after this one
  // completes, so the attention kernel's pre-wait reads (pos / slot and the cached K / V,
  // a.kv_early) see this step's positions and arena even through a chain of early triggers
  griddep_wait();
  if (i < n) { tok[i] = next[i]; pos[i] += inc; }
}
cudaError_t launch_advance(int32_t* tok, const int32_t* next, int32_t* pos, int n, int inc, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  return launch_pdl(advance_kernel, (n + 255) / 256, 256, 0, st, tok, next, pos, n, inc);
}

// Dispatcher inputs of one in-flight batch (sched.hpp): in = [src | tok | pos] x n rows; a row
// whose src is 2 (device feedback) takes the token its previous step generated.
__global__ void dispatch_inputs_kernel(int32_t* tok, const int32_t* next, int32_t* pos, const int32_t* in, int n) {
  griddep_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    tok[i] = in[i] == 2 ? next[i] : in[n + i];
    pos[i] = in[2 * n + i];
  }
}
cudaError_t launch_dispatch_inputs(int32_t* tok, const int32_t* next, int32_t* pos, const int32_t* in, int n,
                                   cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  // like the advance kernel, the batch-state writer never triggers its dependents early
  return launch_pdl(dispatch_inputs_kernel, (n + 255) / 256, 256, 0, st, tok, next, pos, in, n);
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

// KV arena [rows][positions][d_h] (bf16, d_h = 128) as a 3-D tensor map with 64 x 64 boxes and the
// 128-byte swizzle (tensor-core GQA attention)
cudaError_t make_tmap_kv(CUtensorMap* out, const void* base, uint64_t rows, uint64_t positions, uint64_t dh) {
  auto enc = get_encode();
  if (!enc) return cudaErrorNotSupported;
  cuuint64_t dims[3] = {dh, positions, rows};
  cuuint64_t strides[2] = {dh * 2, positions * dh * 2};
  cuuint32_t box[3] = {64, 64, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

static const int kBNs[] = {16, 32, 64, 128};  // batches > 128 use several batch tiles
static int stages_override = getenv("GH_GEMM_STAGES") ? atoi(getenv("GH_GEMM_STAGES")) : 0;  // diagnostics
static int cluster_override = getenv("GH_GEMM_CLUSTER") ? atoi(getenv("GH_GEMM_CLUSTER")) : 0;  // diagnostics

template <int BN>
static int tc_stages() {
  using L = GemmSmem<BN>;
  const int smax = L::max_stages(227 * 1024);
  return std::max(2, std::min(smax, stages_override ? stages_override : smax));
}

// co-resident clusters of C CTAs for the BN instantiation (cudaOccupancyMaxActiveClusters)
template <int BN>
static int max_clusters(int C) {
  static std::map<int, int> cache;
  auto it = cache.find(C);
  if (it != cache.end()) return it->second;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C * (kNumSMs / C));
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = GemmSmem<BN>::bytes(tc_stages<BN>());
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, gemm_tc_kernel<BN>, &cfg) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    n = kNumSMs / C;
  }
  n = std::min(n, kNumSMs / C);  // persistent grid: at most one CTA of this kernel per SM
  cache[C] = n;
  return n;
}

static int max_clusters_bn(int BN, int C) {
  switch (BN) {
    case 16: return max_clusters<16>(C);
    case 32: return max_clusters<32>(C);
    case 64: return max_clusters<64>(C);
    case 128: return max_clusters<128>(C);
    default: return max_clusters<192>(C);
  }
}

// diagnostics: 1 = split-K only, 2 = pair whenever possible (GH_GEMM_PAIR or gemm_debug_pair)
static int pair_override = getenv("GH_GEMM_PAIR") ? atoi(getenv("GH_GEMM_PAIR")) : 0;
static int wide_override = 0;  // diagnostics: 1 = never BN = 192, 2 = always when 128 < B <= 192

static int pair_stages(int BN) { return std::max(2, PairSmem::max_stages(BN, 227 * 1024)); }

// co-resident CTA pairs of the pair kernel (cudaOccupancyMaxActiveClusters, largest tile)
static int max_pairs() {
  static int n = -1;
  if (n >= 0) return n;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kNumSMs);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = PairSmem::bytes(kPairMaxBN, pair_stages(kPairMaxBN));
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaOccupancyMaxActiveClusters(&n, gemm_pair_kernel, &cfg) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    n = kNumSMs / 2;
  }
  return n;
}

// Per-k-block cycles of one CTA, bounded by the L2->SM operand stream (~57 B/clk/SM measured
// with the MMA disabled, tools/gemm_sweep.py) or by the tensor core (4096 bf16 MAC/clk/SM).
static double kblock_clk(double bytes_per_sm, double mma_clk) {
  return std::max(bytes_per_sm / 57.0, mma_clk) + 40.0;
}

// Pair plan for a large batch: the batch is cut into b_tiles tiles of BN columns (multiple of 32,
// <= 256) and the work is spread over the co-resident pairs either tile by tile (contiguous tile
// ranges) or by stream-K (contiguous k-block ranges, split tiles finished by their owner from the
// contributors' fp32 partials).  Cost in SM clocks: the per-pair mainloop (kblock_clk per
// k-block) but never below the weights' HBM streaming time, plus the stream-K fixup (the owner
// reads every contributor's 128 x BN partial at ~25 B/clk, measured) and the last epilogue.
static double hbm_floor_clk(int N, int K) { return (double)N * K * 2 / 3300.0; }  // ~6.5 TB/s at 1965 MHz
static double epi_clk(int BN) { return BN / 32 * 500.0; }

static GemmPlan plan_pair(int N, int K, int Bt, double* cost_out) {
  GemmPlan best;
  double best_cost = 1e30;
  const int KB = (K + kBlockK - 1) / kBlockK;
  const int n_tiles = (N + 2 * kBlockM - 1) / (2 * kBlockM);
  const int npairs = std::min(max_pairs(), (int)(kSkWsBytes / (256 * 256 * 4)));
  const double floor = hbm_floor_clk(N, K);
  int last_bn = 0;
  for (int bt = (Bt + kPairMaxBN - 1) / kPairMaxBN; bt <= (Bt + 31) / 32; ++bt) {
    const int BN = ((Bt + bt - 1) / bt + 31) / 32 * 32;
    if (BN == last_bn) continue;
    last_bn = BN;
    const int b_tiles = (Bt + BN - 1) / BN;
    const double tkb = kblock_clk(16384.0 + BN * 64.0, 2.0 * BN);
    static const int force_split = getenv("GH_PAIR_SPLIT") ? atoi(getenv("GH_PAIR_SPLIT")) : -1;  // diagnostics
    for (int split = 0; split < 2; ++split) {
      if (force_split >= 0 && split != force_split) continue;
      const long tiles = (long)n_tiles * b_tiles, units = tiles * KB;
      double cost;
      int np;
      if (!split) {
        np = (int)std::min<long>(tiles, npairs);
        cost = std::max((double)((tiles + np - 1) / np) * KB * tkb, floor) + epi_clk(BN);
      } else {
        np = (int)std::min<long>(units, npairs);
        const double per = (double)units / np;
        const double contrib = per >= KB ? 1.0 : std::ceil(KB / per);  // partials an owner adds
        const double part = 128.0 * BN * 4;
        cost = std::max(std::ceil(per) * tkb, floor) + contrib * part / 25.0 + part / 64.0 + epi_clk(BN);
      }
      if (cost < best_cost - 1e-9) {
        best_cost = cost;
        best.pair = true; best.split = split; best.BN = BN; best.b_tiles = b_tiles; best.n_tiles = n_tiles;
        best.C = 2; best.n_clusters = np;
      }
    }
  }
  *cost_out = best_cost;
  return best;
}

// Choose the cluster size C minimising the k-blocks on the critical path of one CTA:
// rounds(C) * (ceil(KB / C) + reduction overhead), rounds = ceil(tiles / co-resident clusters).
// Batches above 128 columns also consider the pair kernel (always used above 256).
// split-K plan for batch tile BN (cost in k-blocks on the critical path -> *kb_out)
static GemmPlan plan_splitk(int N, int KB, int Bt, int BN, double* kb_out, int min_c = 1) {
  GemmPlan p;
  p.BN = BN;
  p.b_tiles = (Bt + p.BN - 1) / p.BN;
  p.n_tiles = (N + kBlockM - 1) / kBlockM;
  const int tiles = p.n_tiles * p.b_tiles;
  double best = 1e30;
  // C = 8 (clusters of 8 CTAs) is excluded: only ~16 such clusters fit (GPC packing) and it
  // measured 2-3x slower than C <= 4 for every decode shape (tools/gemm_sweep.py).
  for (int C : {1, 2, 4}) {
    if (C < min_c) continue;
    if (C == 1 && p.BN > 64) continue;  // the reduction keeps BN/C <= 64 rows per thread
    if (C > 1 && (p.BN / C < 4 || C > KB)) continue;
    if (cluster_override && C != cluster_override) continue;
    const int ncl = std::min(tiles, max_clusters_bn(p.BN, C));
    const int rounds = (tiles + ncl - 1) / ncl;
    const double cost = rounds * ((KB + C - 1) / C + (C > 1 ? 1.0 : 0.0));
    if (cost < best - 1e-9) { best = cost; p.C = C; p.n_clusters = ncl; }
  }
  *kb_out = best;
  return p;
}
static double splitk_clk(const GemmPlan& p, double kb, int N, int K) {
  return std::max(kb * kblock_clk(16384.0 + p.BN * 128.0, 2.0 * p.BN), hbm_floor_clk(N, K)) + 5100.0;
}

GemmPlan plan_gemm(int N, int K, int Bt) {
  const int KB = (K + kBlockK - 1) / kBlockK;
  const int bt_cap = std::min(Bt, 128);
  int bn = 128;
  for (int b : kBNs) if (b >= bt_cap) { bn = b; break; }
  double best = 0;
  GemmPlan p = plan_splitk(N, KB, Bt, bn, &best);
  // 129..192 columns: one wide batch tile (BN = 192) instead of two 128-column tiles
  if (Bt > 128 && Bt <= 192 && wide_override != 1) {
    double kbw = 0;
    GemmPlan pw = plan_splitk(N, KB, Bt, 192, &kbw, 4);  // C = 4: 32-row runs (C = 2 spills registers)
    if (kbw < 1e29 && (wide_override == 2 || splitk_clk(pw, kbw, N, K) < splitk_clk(p, best, N, K))) {
      p = pw;
      best = kbw;
    }
  }
  if ((Bt > 128 && pair_override != 1) || pair_override == 2 || Bt > 256) {
    double pc = 0;
    GemmPlan pp = plan_pair(N, K, Bt, &pc);
    // split-K cluster kernel: critical-path k-blocks, HBM floor, reduction + epilogue tail (~2.6 us)
    const double sc = splitk_clk(p, best, N, K);
    if (Bt > 256 || pair_override == 2 || pc < sc) p = pp;
  }
  static const bool verbose = getenv("GH_GEMM_VERBOSE") != nullptr;  // diagnostics
  if (verbose)
    fprintf(stderr, "[gh] gemm N=%d K=%d B=%d: %s BN=%d b_tiles=%d n_tiles=%d C=%d clusters=%d\n", N, K, Bt,
            p.pair ? (p.split ? "pair stream-K" : "pair tiles") : "split-K", p.BN, p.b_tiles, p.n_tiles, p.C,
            p.n_clusters);
  return p;
}

GemmPlan plan_gemm_tp(int N, int K, int Bt) {
  const int KB = (K + kBlockK - 1) / kBlockK;
  const int bt_cap = std::min(Bt, 128);
  int bn = 128;
  for (int b : kBNs) if (b >= bt_cap) { bn = b; break; }
  double best = 0;
  // the all-reducing epilogue holds at most 32 rows per thread (BN / C <= 32)
  GemmPlan p = plan_splitk(N, KB, Bt, bn, &best, std::max(1, bn / 32));
  static const bool verbose = getenv("GH_GEMM_VERBOSE") != nullptr;  // diagnostics
  if (verbose)
    fprintf(stderr, "[gh] gemm (tp all-reduce) N=%d K=%d B=%d: split-K BN=%d b_tiles=%d n_tiles=%d C=%d clusters=%d\n",
            N, K, Bt, p.BN, p.b_tiles, p.n_tiles, p.C, p.n_clusters);
  return p;
}

template <int BN>
static cudaError_t configure_tc() {
  return cudaFuncSetAttribute(gemm_tc_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
}
template <int BN>
static cudaError_t launch_tc(const CUtensorMap* tmW, const CUtensorMap* tmX, GemmShape gs,
                             const GemmPlan& p, const EpiParams& ep, cudaStream_t st) {
  using L = GemmSmem<BN>;
  gs.stages = tc_stages<BN>();
  const int smem = L::bytes(gs.stages);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  static const bool pdl = getenv("GH_NO_PDL") == nullptr;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = p.C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.n_clusters * p.C);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  GH_COUNT_LAUNCH();
  return cudaLaunchKernelEx(&cfg, gemm_tc_kernel<BN>, *tmW, *tmX, gs, ep);
}

static cudaError_t launch_pair(const CUtensorMap* tmW, const CUtensorMap* tmX, GemmShape gs, const GemmPlan& p,
                               const EpiParams& ep, cudaStream_t st) {
  gs.BN = p.BN;
  gs.stages = pair_stages(p.BN);
  const int smem = PairSmem::bytes(p.BN, gs.stages);
  if (smem > 227 * 1024 || p.BN % 32 || p.BN > kPairMaxBN) return cudaErrorInvalidValue;
  if (ep.ss_in && gs.Bt > kPairMaxInvCols) return cudaErrorInvalidValue;
  static const bool pdl = getenv("GH_NO_PDL") == nullptr;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * p.n_clusters);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  GH_COUNT_LAUNCH();
  return cudaLaunchKernelEx(&cfg, gemm_pair_kernel, *tmW, *tmX, gs, ep);
}

void gemm_debug_cluster(int C) { cluster_override = C; }
void gemm_debug_pair(int mode) { pair_override = mode; }
void gemm_debug_wide(int mode) { wide_override = mode; }
void gemm_debug_set(int stages) { stages_override = stages; }

cudaError_t launch_gemm(const Weight& W, const CUtensorMap* tmW, const void* X, long ldx,
                        const CUtensorMap* tmX, int Bt, const GemmPlan& p, const EpiParams& ep,
                        const GemmScratch& sc, cudaStream_t st, const void* pf, size_t pf_bytes) {
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
  gs.N = W.N; gs.K = W.K; gs.Bt = Bt;
  gs.n_tiles = p.n_tiles; gs.b_tiles = p.b_tiles;
  gs.kb_total = (W.K + kBlockK - 1) / kBlockK;
  gs.flags = sc.debug_flags;
  gs.trace = sc.trace;
  gs.BN = p.BN;
  gs.pf = pf;
  gs.pf_bytes = pf ? pf_bytes : 0;
  gs.sk_ws = sc.sk_ws;
  gs.sk_flags = sc.sk_flags;
  gs.sk_split = p.split ? 1 : 0;
  gs.xwait = sc.xwait;
  gs.xwait_n = sc.xwait_n;
  gs.xwait_val = sc.xwait_val;
  if (p.pair) {
    if (!sc.sk_ws || !sc.sk_flags) return cudaErrorInvalidValue;
    return launch_pair(tmW, tmX, gs, p, ep, st);
  }
  if (ep.ss_in && Bt > kMaxInvCols) return cudaErrorInvalidValue;
  switch (p.BN) {
    case 16: return launch_tc<16>(tmW, tmX, gs, p, ep, st);
    case 32: return launch_tc<32>(tmW, tmX, gs, p, ep, st);
    case 64: return launch_tc<64>(tmW, tmX, gs, p, ep, st);
    case 128: return launch_tc<128>(tmW, tmX, gs, p, ep, st);
    case 192: return launch_tc<192>(tmW, tmX, gs, p, ep, st);
  }
  return cudaErrorInvalidValue;
}

// ====================================================================== attention dispatch
template <typename T, int DH, int W>
static cudaError_t configure_attn_w() {
  cudaError_t e = cudaFuncSetAttribute(attn_decode_kernel<T, DH, W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       AttnCfg<T, DH, W>::kSmem);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(attn_decode_kernel<T, DH, W>, cudaFuncAttributePreferredSharedMemoryCarveout,
                              (int)cudaSharedmemCarveoutMaxShared);
}
template <typename T, int DH, int G>
static cudaError_t configure_attn_gqa() {
  cudaError_t e = cudaFuncSetAttribute(attn_gqa_kernel<T, DH, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       GqaCfg<T, DH, G>::kSmem);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(attn_gqa_kernel<T, DH, G>, cudaFuncAttributePreferredSharedMemoryCarveout,
                              (int)cudaSharedmemCarveoutMaxShared);
}
template <int G>
static cudaError_t configure_attn_gqa_tc() {
  return cudaFuncSetAttribute(attn_gqa_tc_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, GqaTcCfg<G>::kSmem);
}
template <typename T, int DH>
static cudaError_t configure_attn() {
  cudaError_t e = configure_attn_w<T, DH, 8>();
  if (e == cudaSuccess) e = configure_attn_w<T, DH, 16>();
  if (e == cudaSuccess) e = configure_attn_gqa<T, DH, 2>();
  if (e == cudaSuccess) e = configure_attn_gqa<T, DH, 4>();
  if (e == cudaSuccess) e = configure_attn_gqa<T, DH, 8>();
  return e;
}
static int attn_warps() {  // consumer warps per CTA (diagnostics override GH_ATTN_WARPS)
  static const int w = getenv("GH_ATTN_WARPS") ? atoi(getenv("GH_ATTN_WARPS")) : 8;
  return w;
}
template <typename T, int DH, int W>
static cudaError_t launch_attn_w(const AttnArgs& a, cudaStream_t st) {
  using C = AttnCfg<T, DH, W>;
  const int units = a.B * a.H;
  if (units <= 0) return cudaSuccess;
  const int grid = std::min(units, kNumSMs);
  return launch_pdl(attn_decode_kernel<T, DH, W>, grid, C::kThreads, C::kSmem, st, a);
}
template <typename T, int DH, int G>
static cudaError_t launch_attn_gqa(const AttnArgs& a, cudaStream_t st) {
  using C = GqaCfg<T, DH, G>;
  const int units = a.B * a.Hkv;
  if (units <= 0) return cudaSuccess;
  const int grid = std::min(units, kNumSMs);
  return launch_pdl(attn_gqa_kernel<T, DH, G>, grid, C::kThreads, C::kSmem, st, a);
}
// group size handled by the group-shared kernel (one unit per KV head): 2, 4 or 8, else 0
static int gqa_group(const AttnArgs& a) {
  static const bool off = getenv("GH_NO_GQA") != nullptr;  // diagnostics: per-query-head kernel
  const int G = a.Hkv > 0 && a.H % a.Hkv == 0 ? a.H / a.Hkv : 1;
  return (!off && (G == 2 || G == 4 || G == 8)) ? G : 0;
}
template <int G>
static cudaError_t launch_attn_gqa_tc(const AttnArgs& a, cudaStream_t st) {
  using C = GqaTcCfg<G>;
  const int units = a.B * a.Hkv;
  if (units <= 0) return cudaSuccess;
  const int grid = std::min(units, kNumSMs);
  return launch_pdl(attn_gqa_tc_kernel<G>, grid, C::kThreads, C::kSmem, st, *a.kv_tmap, a);
}
template <typename T, int DH>
static cudaError_t launch_attn_t(const AttnArgs& a, cudaStream_t st) {
  static const bool no_tc = getenv("GH_NO_GQA_TC") != nullptr;  // diagnostics: CUDA-core GQA kernel
  // MHA on the tensor-core kernel too (G = 1): at the same HBM traffic it spends less energy per
  // byte than the CUDA-core dot products, which holds the bandwidth under the 1000 W cap
  // (sustained 6.96 vs 6.53 TB/s at 7B, B 85, ctx 2048)
  static const bool mha_cc = getenv("GH_MHA_CUDA_CORE") != nullptr;  // diagnostics: CUDA-core MHA kernel
  const bool head_blocks = a.tp > 1;  // tensor-parallel message layout: the tensor-core kernel only
  if constexpr (sizeof(T) == 2 && DH == 128) {
    if (a.kv_tmap && (!no_tc || head_blocks)) switch (gqa_group(a)) {
        case 2: return launch_attn_gqa_tc<2>(a, st);
        case 4: return launch_attn_gqa_tc<4>(a, st);
        case 8: return launch_attn_gqa_tc<8>(a, st);
      }
    if (a.kv_tmap && (head_blocks || (!no_tc && !mha_cc)) && a.H == a.Hkv) return launch_attn_gqa_tc<1>(a, st);
  }
  if (head_blocks) return cudaErrorNotSupported;
  switch (gqa_group(a)) {
    case 2: return launch_attn_gqa<T, DH, 2>(a, st);
    case 4: return launch_attn_gqa<T, DH, 4>(a, st);
    case 8: return launch_attn_gqa<T, DH, 8>(a, st);
  }
  return attn_warps() == 16 ? launch_attn_w<T, DH, 16>(a, st) : launch_attn_w<T, DH, 8>(a, st);
}

bool attention_supported(int db, int dh) {
  return (db == 2 || db == 4) && (dh == 48 || dh == 64 || dh == 128);
}

cudaError_t launch_append_kv(int db, int dh, const AttnArgs& a, cudaStream_t st) {
  const long chunks = (long)a.B * 2 * a.Dkv * db / 16;
  const int grid = (int)std::min<long>((chunks + 255) / 256, (long)kNumSMs * 8);
  if (chunks == 0) return cudaSuccess;
  if (db == 4) return launch_pdl(append_kv_kernel<float>, grid, 256, 0, st, a, dh);
  return launch_pdl(append_kv_kernel<bf16_t>, grid, 256, 0, st, a, dh);
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
  chk(configure_tc<16>()); chk(configure_tc<32>()); chk(configure_tc<64>()); chk(configure_tc<128>());
  chk(configure_tc<192>());
  chk(configure_attn_gqa_tc<1>()); chk(configure_attn_gqa_tc<2>()); chk(configure_attn_gqa_tc<4>());
  chk(configure_attn_gqa_tc<8>());
  chk(cudaFuncSetAttribute(gemm_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  chk(configure_attn<bf16_t, 48>()); chk(configure_attn<bf16_t, 64>()); chk(configure_attn<bf16_t, 128>());
  chk(configure_attn<float, 48>()); chk(configure_attn<float, 64>()); chk(configure_attn<float, 128>());
  return e;
}

}  // namespace gh
