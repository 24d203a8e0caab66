// gemm_pair.cuh — large-batch Tier-1 contractions on CTA pairs (tcgen05 cta_group::2, sm_100a).
//
//   Y[b, n] = sum_k X[b, k] * W[n, k]      (same swap-AB product and epilogues as gemm_tc.cuh)
//
// When the Tier-1 batch exceeds one 128-column tile (B·K' prompts of a two-tier in-flight batch,
// 192..1024), the split-K kernel becomes L2-bandwidth bound: every 128 x 128 tile pulls 16 KB of
// weights and 16 KB of activations per k-block into one SM for only 256 MMA cycles (measured
// ~57 B/clk/SM of L2->SM throughput, tools/gemm_sweep.py).  This kernel runs each output tile on
// a CTA pair (a 2-CTA cluster on one TPC) with M = 256 weight rows and N = BN <= 256 batch
// columns: each CTA stages its own 128 weight rows and HALF of the activation tile, and the
// leader's single tcgen05.mma.cta_group::2 reads both CTAs' shared memory.  Per SM that is
// 16 KB + BN/2 x 128 B per k-block for 2·BN MMA cycles (BN = 256: 64 B/clk, near the L2 limit,
// instead of 128 B/clk), with the fp32 accumulator of 128 rows x BN columns in each CTA's TMEM
// (double-buffered: 2 x 256 columns = all 512).
//
// Barriers: full[s] lives in the leader and counts the bytes of BOTH CTAs' TMA loads
// (cp.async.bulk.tensor .cta_group::2 signals the leader's barrier); empty[s] and the
// accumulator-ready barrier are signalled in both CTAs by one multicast tcgen05.commit; the
// accumulator-drained barrier lives in the leader and counts the 4 epilogue warps of each CTA.
// No K split: every tile is reduced entirely in TMEM, so there is no cross-CTA reduction.
//
// Epilogue: per 32-column chunk, the 4 epilogue warps move TMEM rows into a swizzled shared
// staging tile [32 columns][128 rows] and re-read it as (column, run of 32 rows) so the fused
// epilogues of gemm_tc.cuh (epi_slice) write coalesced 64-byte runs.
#pragma once
#include <cuda.h>
#include "common.cuh"
#include "gemm_tc.cuh"
#include "params.hpp"

namespace gh {

constexpr int kPairMaxBN = 256;
constexpr int kPairMaxInvCols = 1024;  // fused-RMSNorm scales kept in smem (batch columns)

struct PairSmem {
  static constexpr int kABytes = kBlockM * kBlockK * 2;  // 16 KB: this CTA's 128 weight rows
  static constexpr int kStageBytesMax = kABytes + kPairMaxBN / 2 * kBlockK * 2;
  static constexpr int kMaxStages = 16;
  static constexpr int kStgBytes = 32 * 128 * 4;  // epilogue staging: 32 columns x 128 rows fp32
  static constexpr uint32_t kAccCols = kPairMaxBN;
  static constexpr uint32_t kTmemCols = 512;
  static constexpr int kBarBytes = (2 * kMaxStages + 8) * 8 + 16 + kPairMaxInvCols * 4;
  GH_HD static int b_bytes(int BN) { return BN / 2 * kBlockK * 2; }
  GH_HD static int stage_bytes(int BN) { return kABytes + b_bytes(BN); }
  GH_HD static int stg_offset(int BN, int stages) { return stages * stage_bytes(BN); }
  GH_HD static int bar_offset(int BN, int stages) { return stg_offset(BN, stages) + kStgBytes; }
  GH_HD static int bytes(int BN, int stages) { return bar_offset(BN, stages) + kBarBytes + 1024; }
  static int max_stages(int BN, int budget) {
    const int s = (budget - kStgBytes - kBarBytes - 1024) / stage_bytes(BN);
    return s > kMaxStages ? kMaxStages : s;
  }
};

// staging index of (column c, row r): 16-byte chunks of a column XOR-swizzled so that both the
// row-per-thread writes and the (column, 32-row run)-per-thread float4 reads are conflict-free
GH_DEV int pair_stg_index(int c, int r) {
  return c * 128 + ((((r >> 2) ^ (((c & 1) << 2) | ((r >> 5) & 3)))) << 2) + (r & 3);
}

__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                     const GemmShape gs, const EpiParams ep) {
  using L = PairSmem;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int S = gs.stages;
  const int BN = gs.BN;
  const int kStage = L::stage_bytes(BN);
  float* stg = (float*)(smem + L::stg_offset(BN, S));
  uint64_t* full = (uint64_t*)(smem + L::bar_offset(BN, S));  // used in the leader only
  uint64_t* empty = full + L::kMaxStages;
  uint64_t* tfull = empty + L::kMaxStages;  // [2] accumulator ready (both CTAs)
  uint64_t* tempty = tfull + 2;             // [2] accumulator drained (leader, 8 warps)
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
  float* inv_smem = (float*)(tempty + 4);

  const int warp = threadIdx.x >> 5;
  const int KB = gs.kb_total;
  const int rank = (int)cluster_ctarank();  // 0 = leader
  const int pid = (int)cluster_id_x(), npair = (int)cluster_count_x();
  const int n_tiles_total = gs.n_tiles * gs.b_tiles;
  const int my_tiles = pid < n_tiles_total ? (n_tiles_total - 1 - pid) / npair + 1 : 0;

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmW);
    prefetch_tmap(&tmX);
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 8); }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair<L::kTmemCols>(tmem_slot);
  tc_fence_before();
  cluster_sync_all();  // barriers of both CTAs initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_launch_dependents();

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs): own 128 weight rows + own half of the batch tile
    if (elect_one()) {
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      const int total = my_tiles * KB;
      const int pre = min(S, total);
      const int half = BN / 2;
      auto w_row = [&](int i) {
        const int tile = pid + (i / KB) * npair;
        // tile-contiguous weights: 128-row tile (2*tile_n + rank, kb)
        return ((2 * (tile / gs.b_tiles) + rank) * KB + i % KB) * kBlockM;
      };
      auto x_row = [&](int i) { return (pid + (i / KB) * npair) % gs.b_tiles * BN + rank * half; };
      const uint32_t full0 = mapa_shared(smem_u32(full), 0);
      // weights do not depend on the previous kernel: request them before griddepcontrol.wait
      for (int i = 0; i < pre; ++i) {
        if (rank == 0) mbar_arrive_expect_tx(&full[i], 2 * kStage);
        tma_load_2d_pair(smem + i * kStage, &tmW, 0, w_row(i), full0 + i * 8, pol_w);
      }
      griddep_wait();
      for (int i = 0; i < pre; ++i)
        tma_load_2d_pair(smem + i * kStage + L::kABytes, &tmX, (i % KB) * kBlockK, x_row(i), full0 + i * 8, pol_x);
      for (int i = pre; i < total; ++i) {
        const int s = i % S;
        mbar_wait(&empty[s], ((i / S) & 1) ^ 1);
        if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * kStage);
        uint8_t* sa = smem + s * kStage;
        tma_load_2d_pair(sa, &tmW, 0, w_row(i), full0 + s * 8, pol_w);
        tma_load_2d_pair(sa + L::kABytes, &tmX, (i % KB) * kBlockK, x_row(i), full0 + s * 8, pol_x);
      }
      prefetch_l2_share(gs.pf, gs.pf_bytes, blockIdx.x, gridDim.x);
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader only): one accumulator buffer per tile, alternating
    if (rank == 0) {
      const uint32_t idesc = umma_idesc_bf16(2 * kBlockM, BN);
      const bool no_mma = gs.flags & GEMM_DBG_NO_MMA;
      int i = 0;
      for (int j = 0; j < my_tiles; ++j) {
        const int acc = j & 1;
        mbar_wait(&tempty[acc], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * L::kAccCols;
        for (int k = 0; k < KB; ++k, ++i) {
          const int s = i % S;
          mbar_wait(&full[s], (i / S) & 1);
          tc_fence_after();
          if (elect_one()) {
            if (!no_mma) {
              const uint32_t sa = smem_u32(smem + s * kStage);
              const uint64_t da = umma_desc_sw128(sa);
              const uint64_t db = umma_desc_sw128(sa + L::kABytes);
#pragma unroll
              for (int kk = 0; kk < kBlockK / 16; ++kk)
                umma_bf16_pair(d_tmem, da + (uint64_t)(kk * 2), db + (uint64_t)(kk * 2), idesc,
                               (k > 0 || kk > 0) ? 1u : 0u);
            }
            umma_commit_pair(&empty[s], 0x3);
            if (k == KB - 1) umma_commit_pair(&tfull[acc], 0x3);
          }
          __syncwarp();
        }
      }
    }
  } else {
    // ---------------- epilogue warps 2..5 (both CTAs): rows rank*128 + 32*(warp%4) + lane
    const int q = warp & 3;
    const int row = q * 32 + (threadIdx.x & 31);
    const int t = threadIdx.x - 64;
    const int cb = t >> 2, rl = (t & 3) * 32;  // staged read: column cb, rows rl..rl+31
    const bool skip = gs.flags & GEMM_DBG_NO_EPI;
    const uint32_t tempty0 = mapa_shared(smem_u32(tempty), 0);
    griddep_wait();  // residual / positions / norm statistics belong to earlier kernels
    if (ep.ss_in) {
      compute_inv_rms(ep, gs, inv_smem);
      epi_bar();
    }
    for (int j = 0; j < my_tiles; ++j) {
      const int tile = pid + j * npair;
      const int tile_n = tile / gs.b_tiles, tile_b = tile % gs.b_tiles;
      const int n0 = (2 * tile_n + rank) * kBlockM, b0 = tile_b * BN;
      const int acc = j & 1;
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * L::kAccCols;
      mbar_wait(&tfull[acc], (j >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t r0[16], r1[16];
        tmem_ld16(taddr + c0, r0);
        tmem_ld16(taddr + c0 + 16, r1);
        tmem_ld_wait();
        if (c0 + 32 >= BN) {  // accumulator buffer fully read: the leader may reuse it
          tc_fence_before();
          __syncwarp();
          if ((threadIdx.x & 31) == 0) mbar_arrive_cluster(tempty0 + acc * 8);
        }
        if (skip) continue;
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          stg[pair_stg_index(e, row)] = __uint_as_float(r0[e]);
          stg[pair_stg_index(e + 16, row)] = __uint_as_float(r1[e]);
        }
        epi_bar();
        float v[32];
#pragma unroll
        for (int e = 0; e < 32; e += 4) {
          const float4 a = *(const float4*)(stg + pair_stg_index(cb, rl + e));
          v[e] = a.x; v[e + 1] = a.y; v[e + 2] = a.z; v[e + 3] = a.w;
        }
        epi_slice<32, 32>(ep, gs, n0 + rl, b0 + c0 + cb, v, 2 * tile_n + rank, inv_smem);
        epi_bar();  // staging is reused by the next chunk
      }
    }
  }
  tc_fence_before();
  cluster_sync_all();  // the peer's last remote arrivals and TMEM reads are done
  if (warp == 1) tmem_free_pair<L::kTmemCols>(tmem_base);
}

}  // namespace gh
