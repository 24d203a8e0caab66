// gemm_tc.cuh — Tier-1 dense contractions on the 5th-generation tensor cores (sm_100a).
//
//   Y[b, n] = sum_k X[b, k] * W[n, k]          (X: activations [B, K], W: weights [N, K])
//
// Decode batches are skinny (B = 4..1024) while weights are wide, so the kernel computes the
// transposed product D = W_tile * X^T ("swap-AB"): the 128 weight rows of a tile are the UMMA
// M dimension and the batch is the UMMA N dimension (16..256).  Both operands are K-major and
// staged by TMA with the 128-byte swizzle; one elected thread issues tcgen05.mma with the
// fp32 accumulator in TMEM; four epilogue warps drain TMEM with tcgen05.ld and apply the fused
// epilogue (residual add, RoPE + message packing, SwiGLU, logits + partial argmax).
//
// At decode batch sizes the kernel is weight-bandwidth bound, so the grid is split along K
// (split-K, `ks` CTAs per output tile) until ~all SMs stream weights.  Split partials are
// combined deterministically: every split writes its fp32 partial tile to a workspace, the
// last split to arrive (atomic ticket) sums the partials in split order and runs the epilogue.
//
// Warp roles (192 threads): warp 0 = TMA producer, warp 1 = TMEM allocator + MMA issuer,
// warps 2..5 = epilogue (warp w drains TMEM lanes 32*(w%4) .. +31).
#pragma once
#include <cuda.h>
#include "common.cuh"
#include "params.hpp"

namespace gh {

constexpr int kBlockM = 128;   // weight rows per tile (UMMA M)
constexpr int kBlockK = 64;    // 64 bf16 = 128 B = one swizzle atom row
constexpr int kGemmThreads = 192;

template <int BN, int STAGES>
struct GemmSmem {
  static constexpr int kABytes = kBlockM * kBlockK * 2;  // 16 KB
  static constexpr int kBBytes = BN * kBlockK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kBarOffset = STAGES * kStageBytes;
  static constexpr int kTotal = kBarOffset + 256 + 1024;  // barriers + alignment slack
  static constexpr uint32_t kTmemCols = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
};

GH_DEV float silu_f(float g) { return g / (1.0f + __expf(-g)); }

// Scalar epilogue for STORE / STORE_RESID / QKV_ROPE / SWIGLU at output (row n, batch b).
// `partner` is the accumulator of row n^1 (RoPE pair / interleaved gate-up pair).
template <typename T>
GH_DEV void epi_store_one(const EpiParams& ep, int n, int b, float v, float partner) {
  T* out = (T*)ep.out;
  switch (ep.kind) {
    case EPI_STORE:
      St<T>::store(out, (long)b * ep.ldo + n, v);
      break;
    case EPI_STORE_RESID:
      St<T>::store(out, (long)b * ep.ldo + n, v + St<T>::load((const T*)ep.resid, (long)b * ep.ldr + n));
      break;
    case EPI_QKV_ROPE: {
      float x = v;
      if (n < ep.rope_rows) {
        const float2 cs = ep.rope[(long)ep.pos[b] * (ep.d_head >> 1) + ((n % ep.d_head) >> 1)];
        // pair (a, c) = (even, odd): even' = a cos - c sin, odd' = a sin + c cos
        x = (n & 1) ? (partner * cs.y + v * cs.x) : (v * cs.x - partner * cs.y);
      }
      St<T>::store(out, (long)b * ep.ldo + n, x);
      break;
    }
    case EPI_SWIGLU:
      if (!(n & 1)) St<T>::store(out, (long)b * ep.ldo + (n >> 1), silu_f(v) * partner);
      break;
    default:
      break;
  }
}

// Apply the epilogue to 16 accumulator columns [c0, c0+16) of weight row `n` (this thread).
// All 32 lanes of the warp must call it (RoPE / SwiGLU exchange with lane^1).
GH_DEV void epilogue_chunk(const EpiParams& ep, const GemmShape& gs, int n, int b0, int c0,
                           float (&v)[16], float* red_smem, int tile_n) {
  const bool row_ok = n < gs.N;
  if (ep.kind != EPI_LOGITS_ARGMAX) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const float partner = __shfl_xor_sync(0xffffffffu, v[j], 1);
      const int b = b0 + c0 + j;
      if (row_ok && b < gs.Bt) epi_store_one<bf16_t>(ep, n, b, v[j], partner);
    }
    return;
  }
  // logits (optional) + (max, argmax) across the tile's 128 rows per batch column
  const int wq = (threadIdx.x >> 5) & 3;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int b = b0 + c0 + j;
    float val = row_ok ? v[j] : -INFINITY;
    int idx = row_ok ? n : 0x7fffffff;
    if (ep.logits && row_ok && b < gs.Bt) ep.logits[(long)b * ep.ldl + n] = v[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, val, o);
      const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
      if (ov > val || (ov == val && oi < idx)) { val = ov; idx = oi; }
    }
    if ((threadIdx.x & 31) == 0) {
      red_smem[(wq * 16 + j) * 2] = val;
      red_smem[(wq * 16 + j) * 2 + 1] = __int_as_float(idx);
    }
  }
  asm volatile("bar.sync 1, 128;\n" ::: "memory");
  if (threadIdx.x >= 64 && threadIdx.x < 64 + 16) {
    const int j = threadIdx.x - 64;
    float best = red_smem[j * 2];
    int bi = __float_as_int(red_smem[j * 2 + 1]);
#pragma unroll
    for (int w = 1; w < 4; ++w) {
      const float ov = red_smem[(w * 16 + j) * 2];
      const int oi = __float_as_int(red_smem[(w * 16 + j) * 2 + 1]);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    const int b = b0 + c0 + j;
    if (b < gs.Bt) ep.part[(long)tile_n * gs.Bt + b] = make_float2(best, __int_as_float(bi));
  }
  asm volatile("bar.sync 1, 128;\n" ::: "memory");
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                   const GemmShape gs, const EpiParams ep) {
  using L = GemmSmem<BN, STAGES>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + L::kBarOffset);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint32_t* tmem_slot = (uint32_t*)(tmem_full + 1);
  int* flag_smem = (int*)(tmem_slot + 1);

  const int warp = threadIdx.x >> 5;
  const int tile_n = blockIdx.x;
  const int tile_b = blockIdx.y;
  const int split = blockIdx.z;
  const int n0 = tile_n * kBlockM;
  const int b0 = tile_b * BN;
  const int kb0 = (int)(((long)split * gs.kb_total) / gs.ks);
  const int kb1 = (int)(((long)(split + 1) * gs.kb_total) / gs.ks);
  const int nkb = kb1 - kb0;

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmW);
    prefetch_tmap(&tmX);
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(tmem_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<L::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer
    if (elect_one()) {
      const uint64_t pol_w = policy_evict_first();  // weights stream through once
      const uint64_t pol_x = policy_evict_last();   // activations are re-read by every tile
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* sa = smem + s * L::kStageBytes;
        uint8_t* sb = sa + L::kABytes;
        mbar_arrive_expect_tx(&full[s], L::kStageBytes);
        const int kc = (kb0 + i) * kBlockK;
        tma_load_2d(sa, &tmW, kc, n0, &full[s], pol_w);
        tma_load_2d(sb, &tmX, kc, b0, &full[s], pol_x);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    const uint32_t idesc = umma_idesc_bf16(kBlockM, BN);
    for (int i = 0; i < nkb; ++i) {
      const int s = i % STAGES;
      const uint32_t ph = (i / STAGES) & 1;
      mbar_wait(&full[s], ph);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sa = smem_u32(smem + s * L::kStageBytes);
        const uint32_t sb = sa + L::kABytes;
        const uint64_t da = umma_desc_sw128(sa);
        const uint64_t db = umma_desc_sw128(sb);
#pragma unroll
        for (int k = 0; k < kBlockK / 16; ++k) {
          // +32 bytes along K inside the 128-byte swizzle atom = +2 in the >>4 address field
          umma_bf16(tmem_base, da + (uint64_t)(k * 2), db + (uint64_t)(k * 2), idesc,
                    (i > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(&empty[s]);
        if (i == nkb - 1) umma_commit(tmem_full);
      }
      __syncwarp();
    }
  } else {
    // ---------------- epilogue warps 2..5
    const int q = warp & 3;          // TMEM lane quarter this warp may access
    const int row = q * 32 + (threadIdx.x & 31);
    const int n = n0 + row;
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    // argmax reduction scratch: stage 0 is free once every MMA has completed
    float* red_smem = (float*)smem;
    const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16);
    const long tile_id = (long)tile_n * gridDim.y + tile_b;

    if (gs.ks == 1) {
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t r[16];
        tmem_ld16(taddr + c0, r);
        tmem_ld_wait();
        float v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
        epilogue_chunk(ep, gs, n, b0, c0, v, red_smem, tile_n);
      }
    } else {
      // split-K: publish the partial, take a ticket; the last split reduces in split order.
      float* wsl = gs.ws + tile_id * (long)gs.ks * kBlockM * BN;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t r[16];
        tmem_ld16(taddr + c0, r);
        tmem_ld_wait();
        float4* dst = (float4*)(wsl + ((long)split * (BN / 16) + c0 / 16) * kBlockM * 16 + row * 16);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          __stcg(dst + j, make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                      __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3])));
      }
      __threadfence();
      asm volatile("bar.sync 1, 128;\n" ::: "memory");
      if (threadIdx.x == 64) {
        int t = atomicAdd(&gs.tickets[tile_id], 1);
        *flag_smem = (t == gs.ks - 1);
        if (t == gs.ks - 1) gs.tickets[tile_id] = 0;  // reset for the next launch
      }
      asm volatile("bar.sync 1, 128;\n" ::: "memory");
      if (*flag_smem) {
        __threadfence();
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 16) {
          float v[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = 0.f;
          for (int s = 0; s < gs.ks; ++s) {
            const float4* src =
                (const float4*)(wsl + ((long)s * (BN / 16) + c0 / 16) * kBlockM * 16 + row * 16);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              float4 t4 = __ldcg(src + j);
              v[4 * j] += t4.x; v[4 * j + 1] += t4.y; v[4 * j + 2] += t4.z; v[4 * j + 3] += t4.w;
            }
          }
          epilogue_chunk(ep, gs, n, b0, c0, v, red_smem, tile_n);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_free<L::kTmemCols>(tmem_base);
}

}  // namespace gh
