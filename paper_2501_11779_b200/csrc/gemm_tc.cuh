// gemm_tc.cuh — Tier-1 dense contractions on the 5th-generation tensor cores (sm_100a).
//
//   Y[b, n] = sum_k X[b, k] * W[n, k]          (X: activations [B, K], W: weights [N, K])
//
// Decode batches are skinny (B = 4..1024) while weights are wide, so the kernel computes the
// transposed product D = W_tile * X^T ("swap-AB"): the 128 weight rows of a tile are the UMMA
// M dimension and the batch is the UMMA N dimension (16..256).  Both operands are K-major and
// staged by TMA with the 128-byte swizzle (weights are stored tile-contiguous, kernels.hpp, so
// each weight box is one contiguous 16 KB read); one elected thread issues tcgen05.mma with the
// fp32 accumulator in TMEM; four epilogue warps drain TMEM with tcgen05.ld and apply the fused
// epilogue (residual add, RoPE + message packing, SwiGLU, logits + partial argmax).
//
// Scheduling is persistent stream-K: the linearised (tile, k-block) iteration space is cut into
// gridDim.x equal contiguous ranges, one per CTA (one CTA per SM), so every SM streams the same
// number of weight bytes.  A CTA's range is a sequence of "segments" (a k-range of one tile).
// The accumulator is double-buffered in TMEM so the epilogue of segment j overlaps the TMA/MMA
// mainloop of segment j+1.  A tile cut across CTAs ("pieces") is combined deterministically:
// each piece writes its fp32 partial to a workspace, the last piece to arrive (atomic ticket)
// sums all pieces in piece order and runs the epilogue — no CTA ever waits for another.
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
constexpr int kEpiCols = 64;   // epilogue column group (staging width)

// Shared memory: [stage ring][epilogue staging][barriers]
//   epilogue staging: otile [64][128] bf16 | rtile [64][128] bf16 | pos [64] int | argmax 512 B
struct EpiSmem {
  static constexpr int kO = 0;
  static constexpr int kR = kEpiCols * 256;
  static constexpr int kPos = 2 * kEpiCols * 256;
  static constexpr int kRed = kPos + kEpiCols * 4;
  static constexpr int kBytes = kRed + 512;
};

template <int BN>
struct GemmSmem {
  static constexpr int kABytes = kBlockM * kBlockK * 2;  // 16 KB
  static constexpr int kBBytes = BN * kBlockK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kMaxStages = 16;
  static constexpr uint32_t kAccCols = BN < 32 ? 32 : BN;  // one accumulator buffer
  static constexpr uint32_t kTmemCols = 2 * kAccCols <= 64 ? 64 : 2 * kAccCols <= 128 ? 128
                                      : 2 * kAccCols <= 256 ? 256 : 512;
  static constexpr int kBarBytes = (2 * kMaxStages + 4) * 8 + 16;
  GH_HD static int epi_offset(int stages) { return stages * kStageBytes; }
  GH_HD static int bar_offset(int stages) { return stages * kStageBytes + EpiSmem::kBytes; }
  GH_HD static int bytes(int stages) { return bar_offset(stages) + kBarBytes + 1024; }
  static int max_stages(int budget) {
    int s = (budget - EpiSmem::kBytes - kBarBytes - 1024) / kStageBytes;
    return s > kMaxStages ? kMaxStages : s;
  }
};

GH_DEV float silu_f(float g) { return g / (1.0f + __expf(-g)); }

// Scalar epilogue for STORE / STORE_RESID / QKV_ROPE / SWIGLU at output (row n, batch b).
// `partner` is the accumulator of row n^1 (RoPE pair / interleaved gate-up pair).  Used by the
// fp32 (SIMT) path; the tcgen05 path below implements the same math on staged tiles.
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

// ------------------------------------------------------------------ tile epilogue
// The accumulator tile is 128 weight rows (n) x BN batch columns (b); thread `row` of the four
// epilogue warps owns weight row n0+row.  Outputs are row-major [b][n], so 64-column groups are
// staged through shared memory and written (and the residual read) with coalesced 16-byte
// accesses; per-column scalars (positions, RoPE factors) are loaded in independent batches.
GH_DEV void epi_bar() { asm volatile("bar.sync 1, 128;\n" ::: "memory"); }

// coalesced copy of a [rows][cols] bf16 tile between global (row stride ld) and shared memory
template <bool kToShared>
GH_DEV void tile_copy(uint16_t* sm, int sm_ld, uint16_t* gm, long ld, int rows, int cols, int valid_cols) {
  const int t = threadIdx.x - 64;
  const bool vec = valid_cols == cols && ((uintptr_t)gm & 15) == 0 && (ld % 8) == 0;
  if (vec) {
    const int cpr = cols / 8;
    for (int i = t; i < rows * cpr; i += 128) {
      const int r = i / cpr, c = (i % cpr) * 8;
      if (kToShared) *(uint4*)(sm + r * sm_ld + c) = *(const uint4*)(gm + (long)r * ld + c);
      else *(uint4*)(gm + (long)r * ld + c) = *(const uint4*)(sm + r * sm_ld + c);
    }
  } else {
    for (int i = t; i < rows * cols; i += 128) {
      const int r = i / cols, c = i % cols;
      if (c >= valid_cols) continue;
      if (kToShared) sm[r * sm_ld + c] = gm[(long)r * ld + c];
      else gm[(long)r * ld + c] = sm[r * sm_ld + c];
    }
  }
}

// before a column group [g0, g0+64): residual tile / positions into shared memory
GH_DEV void epi_group_begin(const EpiParams& ep, const GemmShape& gs, int n0, int g0, uint8_t* esm) {
  const int rows = min(kEpiCols, gs.Bt - g0);
  epi_bar();  // the previous group's staged tile has been stored
  if (ep.kind == EPI_STORE_RESID)
    tile_copy<true>((uint16_t*)(esm + EpiSmem::kR), 128, (uint16_t*)ep.resid + (long)g0 * ep.ldr + n0,
                    ep.ldr, rows, 128, min(128, gs.N - n0));
  if (ep.kind == EPI_QKV_ROPE) {
    int* ps = (int*)(esm + EpiSmem::kPos);
    for (int i = threadIdx.x - 64; i < rows; i += 128) ps[i] = ep.pos[g0 + i];
  }
  epi_bar();
}

// 16 accumulator columns [c0, c0+16) (absolute batch index b = c0 + j, group base g0)
GH_DEV void epi_chunk(const EpiParams& ep, const GemmShape& gs, int row, int n0, int g0, int c0,
                      const float* v, uint8_t* esm, int tile_n) {
  const int n = n0 + row;
  const bool row_ok = n < gs.N;
  const int lc = c0 - g0;  // local column in the staging tile
  uint16_t* ot = (uint16_t*)(esm + EpiSmem::kO);
  switch (ep.kind) {
    case EPI_STORE:
#pragma unroll
      for (int j = 0; j < 16; ++j) ot[(lc + j) * 128 + row] = f32_to_bf16(v[j]);
      return;
    case EPI_STORE_RESID: {
      const uint16_t* rt = (const uint16_t*)(esm + EpiSmem::kR);
#pragma unroll
      for (int j = 0; j < 16; ++j)
        ot[(lc + j) * 128 + row] = f32_to_bf16(v[j] + bf16_to_f32(rt[(lc + j) * 128 + row]));
      return;
    }
    case EPI_QKV_ROPE: {
      const int* ps = (const int*)(esm + EpiSmem::kPos);
      const bool rope = n < ep.rope_rows;
      const int half = ep.d_head >> 1, pair = (n % ep.d_head) >> 1;
      const bool odd = (n & 1) != 0;
      float2 cs[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {  // independent loads, issued back to back
        const int b = min(c0 + j, gs.Bt - 1) - g0;
        cs[j] = rope ? __ldg(ep.rope + (long)ps[b] * half + pair) : make_float2(1.f, 0.f);
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float partner = __shfl_xor_sync(0xffffffffu, v[j], 1);
        // pair (a, c) = (even, odd): even' = a cos - c sin, odd' = a sin + c cos
        const float x = odd ? (partner * cs[j].y + v[j] * cs[j].x) : (v[j] * cs[j].x - partner * cs[j].y);
        ot[(lc + j) * 128 + row] = f32_to_bf16(x);
      }
      return;
    }
    case EPI_SWIGLU: {
      const bool odd = (row & 1) != 0;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float up = __shfl_xor_sync(0xffffffffu, v[j], 1);
        if (!odd) ot[(lc + j) * 128 + (row >> 1)] = f32_to_bf16(silu_f(v[j]) * up);
      }
      return;
    }
    default:
      break;
  }
  // EPI_LOGITS_ARGMAX: logits (optional) + (max, argmax) across the tile's 128 rows per column
  float* red = (float*)(esm + EpiSmem::kRed);
  const int wq = (threadIdx.x >> 5) & 3;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int b = c0 + j;
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
      red[(wq * 16 + j) * 2] = val;
      red[(wq * 16 + j) * 2 + 1] = __int_as_float(idx);
    }
  }
  epi_bar();
  if (threadIdx.x >= 64 && threadIdx.x < 64 + 16) {
    const int j = threadIdx.x - 64;
    float best = red[j * 2];
    int bi = __float_as_int(red[j * 2 + 1]);
#pragma unroll
    for (int w = 1; w < 4; ++w) {
      const float ov = red[(w * 16 + j) * 2];
      const int oi = __float_as_int(red[(w * 16 + j) * 2 + 1]);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    const int b = c0 + j;
    if (b < gs.Bt) ep.part[(long)tile_n * gs.Bt + b] = make_float2(best, __int_as_float(bi));
  }
  epi_bar();
}

GH_DEV void epi_group_end(const EpiParams& ep, const GemmShape& gs, int n0, int g0, uint8_t* esm) {
  if (ep.kind == EPI_LOGITS_ARGMAX) return;
  epi_bar();
  const int rows = min(kEpiCols, gs.Bt - g0);
  uint16_t* ot = (uint16_t*)(esm + EpiSmem::kO);
  uint16_t* out = (uint16_t*)ep.out;
  if (ep.kind == EPI_SWIGLU)
    tile_copy<false>(ot, 128, out + (long)g0 * ep.ldo + n0 / 2, ep.ldo, rows, 64, min(64, (gs.N - n0) / 2));
  else
    tile_copy<false>(ot, 128, out + (long)g0 * ep.ldo + n0, ep.ldo, rows, 128, min(128, gs.N - n0));
}

// ------------------------------------------------------------------ stream-K schedule
// Iteration space: tiles x KB, tile t = tile_n * b_tiles + tile_b (batch tiles of one weight
// tile are adjacent, so they stream the same weights close in time and share them in L2).
struct StreamK {
  long T;         // total iterations
  int KB, G;
  GH_HD long begin(int c) const { return (long)c * T / G; }
  GH_HD int cta_of(long it) const { return (int)(((it + 1) * (long)G - 1) / T); }
};

template <int BN>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                   const GemmShape gs, const EpiParams ep) {
  using L = GemmSmem<BN>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int S = gs.stages;
  uint8_t* esm = smem + L::epi_offset(S);
  uint64_t* full = (uint64_t*)(smem + L::bar_offset(S));
  uint64_t* empty = full + L::kMaxStages;
  uint64_t* tfull = empty + L::kMaxStages;   // [2] accumulator ready
  uint64_t* tempty = tfull + 2;              // [2] accumulator drained
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
  int* flag_smem = (int*)(tmem_slot + 1);

  const int warp = threadIdx.x >> 5;
  const int KB = gs.kb_total;
  const StreamK sk{(long)gs.n_tiles * gs.b_tiles * KB, KB, (int)gridDim.x};
  const long it_begin = sk.begin(blockIdx.x), it_end = sk.begin(blockIdx.x + 1);

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmW);
    prefetch_tmap(&tmX);
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 4); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<L::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer: every k-block of every segment, one continuous ring
    if (elect_one()) {
      const bool hint = !(gs.flags & GEMM_DBG_NO_HINT);
      const bool load_x = !(gs.flags & GEMM_DBG_NO_X);
      const uint64_t pol_w = hint ? policy_evict_first() : 0;  // weights stream through once
      const uint64_t pol_x = hint ? policy_evict_last() : 0;   // activations are re-read by every tile
      int i = 0;
      for (long it = it_begin; it < it_end; ++it, ++i) {
        const int tile = (int)(it / KB), kb = (int)(it % KB);
        const int tile_n = tile / gs.b_tiles, tile_b = tile % gs.b_tiles;
        const int s = i % S;
        const uint32_t ph = (i / S) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* sa = smem + s * L::kStageBytes;
        uint8_t* sb = sa + L::kABytes;
        mbar_arrive_expect_tx(&full[s], load_x ? L::kStageBytes : L::kABytes);
        // W is tile-contiguous: tile (tile_n, kb) = rows [(tile_n*KB + kb)*128, +128) of [*, 64]
        if (hint) {
          tma_load_2d(sa, &tmW, 0, (tile_n * KB + kb) * kBlockM, &full[s], pol_w);
          if (load_x) tma_load_2d(sb, &tmX, kb * kBlockK, tile_b * BN, &full[s], pol_x);
        } else {
          tma_load_2d_nohint(sa, &tmW, 0, (tile_n * KB + kb) * kBlockM, &full[s]);
          if (load_x) tma_load_2d_nohint(sb, &tmX, kb * kBlockK, tile_b * BN, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: one accumulator buffer per segment, alternating
    const uint32_t idesc = umma_idesc_bf16(kBlockM, BN);
    const bool no_mma = gs.flags & GEMM_DBG_NO_MMA;
    int i = 0, j = 0;
    for (long it = it_begin; it < it_end; ++j) {
      const int kb0 = (int)(it % KB);
      const int kb1 = (int)min((long)KB, kb0 + (it_end - it));
      const int acc = j & 1;
      mbar_wait(&tempty[acc], ((j >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * L::kAccCols;
      for (int kb = kb0; kb < kb1; ++kb, ++i) {
        const int s = i % S;
        mbar_wait(&full[s], (i / S) & 1);
        tc_fence_after();
        if (elect_one()) {
          if (no_mma) {
            mbar_arrive(&empty[s]);
            if (kb == kb1 - 1) mbar_arrive(&tfull[acc]);
          } else {
            const uint32_t sa = smem_u32(smem + s * L::kStageBytes);
            const uint64_t da = umma_desc_sw128(sa);
            const uint64_t db = umma_desc_sw128(sa + L::kABytes);
#pragma unroll
            for (int k = 0; k < kBlockK / 16; ++k)
              // +32 bytes along K inside the 128-byte swizzle atom = +2 in the >>4 address field
              umma_bf16(d_tmem, da + (uint64_t)(k * 2), db + (uint64_t)(k * 2), idesc,
                        (kb > kb0 || k > 0) ? 1u : 0u);
            umma_commit(&empty[s]);
            if (kb == kb1 - 1) umma_commit(&tfull[acc]);
          }
        }
        __syncwarp();
      }
      it += kb1 - kb0;
    }
  } else {
    // ---------------- epilogue warps 2..5
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row = q * 32 + (threadIdx.x & 31);
    int j = 0;
    for (long it = it_begin; it < it_end; ++j) {
      const int tile = (int)(it / KB);
      const int kb0 = (int)(it % KB);
      const int kb1 = (int)min((long)KB, kb0 + (it_end - it));
      it += kb1 - kb0;
      const int tile_n = tile / gs.b_tiles, tile_b = tile % gs.b_tiles;
      const int n0 = tile_n * kBlockM, b0 = tile_b * BN;
      const int acc = j & 1;
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * L::kAccCols;
      mbar_wait(&tfull[acc], (j >> 1) & 1);
      tc_fence_after();
      const bool whole = kb0 == 0 && kb1 == KB;
      const bool skip = gs.flags & GEMM_DBG_NO_EPI;

      if (whole && BN <= 64) {
        // drain the accumulator into registers, release TMEM, then run the epilogue
        float v[BN];
#pragma unroll
        for (int c0 = 0; c0 < BN; c0 += 16) {
          uint32_t r[16];
          tmem_ld16(taddr + c0, r);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 16; ++e) v[c0 + e] = __uint_as_float(r[e]);
        }
        tc_fence_before();
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(&tempty[acc]);
        if (!skip) {
          epi_group_begin(ep, gs, n0, b0, esm);
#pragma unroll
          for (int c0 = 0; c0 < BN; c0 += 16)
            if (b0 + c0 < gs.Bt) epi_chunk(ep, gs, row, n0, b0, b0 + c0, v + c0, esm, tile_n);
          epi_group_end(ep, gs, n0, b0, esm);
        }
      } else if (whole) {
        // wide batch tile: epilogue straight from TMEM, 64-column groups
        if (!skip) {
          for (int g = 0; g < BN && b0 + g < gs.Bt; g += kEpiCols) {
            epi_group_begin(ep, gs, n0, b0 + g, esm);
            for (int c = g; c < g + kEpiCols && b0 + c < gs.Bt; c += 16) {
              uint32_t r[16];
              tmem_ld16(taddr + c, r);
              tmem_ld_wait();
              float v[16];
#pragma unroll
              for (int e = 0; e < 16; ++e) v[e] = __uint_as_float(r[e]);
              epi_chunk(ep, gs, row, n0, b0 + g, b0 + c, v, esm, tile_n);
            }
            epi_group_end(ep, gs, n0, b0 + g, esm);
          }
        }
        tc_fence_before();
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(&tempty[acc]);
      } else {
        // a piece of a tile shared with other CTAs: publish the fp32 partial, take a ticket;
        // the last piece to arrive sums all pieces in piece order and runs the epilogue.
        const int c_first = sk.cta_of((long)tile * KB), c_last = sk.cta_of((long)tile * KB + KB - 1);
        const int n_pieces = c_last - c_first + 1;
        const int piece = blockIdx.x - c_first;
        float* wst = gs.ws + (long)tile * gs.max_pieces * kBlockM * BN;
        for (int c0 = 0; c0 < BN; c0 += 16) {
          uint32_t r[16];
          tmem_ld16(taddr + c0, r);
          tmem_ld_wait();
          float4* dst = (float4*)(wst + ((long)piece * (BN / 16) + c0 / 16) * kBlockM * 16 + row * 16);
#pragma unroll
          for (int e = 0; e < 4; ++e)
            __stcg(dst + e, make_float4(__uint_as_float(r[4 * e]), __uint_as_float(r[4 * e + 1]),
                                        __uint_as_float(r[4 * e + 2]), __uint_as_float(r[4 * e + 3])));
        }
        tc_fence_before();
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(&tempty[acc]);
        __threadfence();
        epi_bar();
        if (threadIdx.x == 64) {
          const int t = atomicAdd(&gs.tickets[tile], 1);
          *flag_smem = (t == n_pieces - 1);
          if (t == n_pieces - 1) gs.tickets[tile] = 0;  // reset for the next launch
        }
        epi_bar();
        if (*flag_smem && !skip) {
          __threadfence();
          for (int g = 0; g < BN && b0 + g < gs.Bt; g += kEpiCols) {
            epi_group_begin(ep, gs, n0, b0 + g, esm);
            for (int c = g; c < g + kEpiCols && b0 + c < gs.Bt; c += 16) {
              float v[16];
#pragma unroll
              for (int e = 0; e < 16; ++e) v[e] = 0.f;
              for (int p = 0; p < n_pieces; ++p) {
                const float4* src =
                    (const float4*)(wst + ((long)p * (BN / 16) + c / 16) * kBlockM * 16 + row * 16);
                float4 t4[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) t4[e] = __ldcg(src + e);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  v[4 * e] += t4[e].x; v[4 * e + 1] += t4[e].y; v[4 * e + 2] += t4[e].z; v[4 * e + 3] += t4[e].w;
                }
              }
              epi_chunk(ep, gs, row, n0, b0 + g, b0 + c, v, esm, tile_n);
            }
            epi_group_end(ep, gs, n0, b0 + g, esm);
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_free<L::kTmemCols>(tmem_base);
}

}  // namespace gh
