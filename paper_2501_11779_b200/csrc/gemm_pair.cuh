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
  static constexpr int kBarBytes = (2 * kMaxStages + 16) * 8 + 16 + kPairMaxInvCols * 8;  // + RoPE positions
  static constexpr int kFixSlots = 8;  // stream-K fixup: 16 KB partial blocks in flight
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

// staging index of (column c, row r): 16-byte chunks of odd columns XOR-swizzled by one so that
// both the row-per-thread writes and the float4 reads of the epilogue mapping (4 threads per
// column, rows q*8 + 32j + 0..7) are conflict-free
GH_DEV int pair_stg_index(int c, int r) { return c * 128 + (((r >> 2) ^ (c & 1)) << 2) + (r & 3); }

// Stream-K work split (deterministic).  The T = n_tiles x b_tiles output tiles are cut into
// T x KB units (one 64-deep k-block of one tile); CTA pair p processes the contiguous units
// [p*U/P, (p+1)*U/P), so every pair streams the same number of k-blocks whatever the tile count
// (no wave quantisation).  A tile whose units span several pairs is finished by its OWNER, the
// pair that processes its k-block 0 (at the END of the owner's range); the other pairs process
// the tile's later k-blocks at the START of their ranges, so their fp32 partials (written to a
// global workspace, one slot per pair) are ready early, and the owner adds them in pair order
// (a fixed summation order: results do not depend on timing).  Owners wait only on pairs that
// are co-resident (the grid never exceeds the co-resident pairs), contributors never wait.
struct SkPiece {
  int tile, kb0, kb1;  // k-blocks [kb0, kb1) of tile
};
// tiles == true: tile-aligned ranges (no split tiles) -- the planner's choice when the fixups
// would cost more than the wave quantisation they remove
GH_DEV long sk_start(int p, int P, long U, int KB, bool tiles) {
  return tiles ? (long)p * (U / KB) / P * KB : (long)p * U / P;
}
struct SkRange {
  long u, u1;
  int KB;
  GH_DEV SkRange(int p, int P, long U, int kb, bool tiles)
      : u(sk_start(p, P, U, kb, tiles)), u1(sk_start(p + 1, P, U, kb, tiles)), KB(kb) {}
  GH_DEV bool next(SkPiece& pc) {
    if (u >= u1) return false;
    pc.tile = (int)(u / KB);
    pc.kb0 = (int)(u % KB);
    pc.kb1 = (int)min((long)KB, pc.kb0 + (u1 - u));
    u += pc.kb1 - pc.kb0;
    return true;
  }
};

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
  uint64_t* pbar = (uint64_t*)(inv_smem + kPairMaxInvCols);  // [kFixSlots] stream-K fixup blocks
  int* pos_smem = (int*)(pbar + L::kFixSlots);                // [kPairMaxInvCols] RoPE positions

  const int warp = threadIdx.x >> 5;
  const int KB = gs.kb_total;
  const int rank = (int)cluster_ctarank();  // 0 = leader
  const int pid = (int)cluster_id_x(), npair = (int)cluster_count_x();
  const int bt = gs.b_tiles;
  const long U = (long)gs.n_tiles * bt * KB;
  const bool sk_tiles = !gs.sk_split || (gs.flags & GEMM_DBG_SK_TILES);
  unsigned long long* trace = gs.trace ? gs.trace + blockIdx.x * 16 : nullptr;  // diagnostics
  if (trace && threadIdx.x == 0) trace[0] = globaltimer();

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmW);
    prefetch_tmap(&tmX);
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 8); }
    for (int a = 0; a < L::kFixSlots; ++a) mbar_init(&pbar[a], 1);
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
      const int half = BN / 2;
      const uint32_t full0 = mapa_shared(smem_u32(full), 0);
      SkRange rg(pid, npair, U, KB, sk_tiles);
      SkPiece pc;
      int i = 0, pre_done = 0;
      // weights do not depend on the previous kernel: the first S stages of weights are requested
      // before griddepcontrol.wait, their activations after it
      int pre_tile[L::kMaxStages], pre_kb[L::kMaxStages];
      while (rg.next(pc)) {
        for (int kb = pc.kb0; kb < pc.kb1; ++kb, ++i) {
          const int s = i % S;
          const int w_row = ((2 * (pc.tile / bt) + rank) * KB + kb) * kBlockM;  // tile-contiguous W
          const int x_row = (pc.tile % bt) * BN + rank * half;
          if (i >= S) mbar_wait(&empty[s], ((i / S) & 1) ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * kStage);
          tma_load_2d_pair(smem + s * kStage, &tmW, 0, w_row, full0 + s * 8, pol_w);
          if (i < S) {
            pre_tile[i] = x_row;
            pre_kb[i] = kb;
            if (i == S - 1) {
              if (trace) trace[1] = globaltimer();
              griddep_wait();
              wait_peer_rows(gs);
              if (trace) trace[2] = globaltimer();
              for (int k = 0; k < S; ++k)
                tma_load_2d_pair(smem + k * kStage + L::kABytes, &tmX, pre_kb[k] * kBlockK, pre_tile[k],
                                 full0 + k * 8, pol_x);
              pre_done = 1;
            }
          } else {
            tma_load_2d_pair(smem + s * kStage + L::kABytes, &tmX, kb * kBlockK, x_row, full0 + s * 8, pol_x);
          }
        }
      }
      if (!pre_done) {  // fewer than S k-blocks in this pair's range
        if (trace) trace[1] = globaltimer();
        griddep_wait();
        wait_peer_rows(gs);
        if (trace) trace[2] = globaltimer();
        for (int k = 0; k < i; ++k)
          tma_load_2d_pair(smem + k * kStage + L::kABytes, &tmX, pre_kb[k] * kBlockK, pre_tile[k], full0 + k * 8,
                           pol_x);
      }
      prefetch_l2_share(gs.pf, gs.pf_bytes, blockIdx.x, gridDim.x);
      if (trace) trace[3] = globaltimer();  // all loads issued
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader only): one accumulator buffer per piece, alternating
    if (rank == 0) {
      const uint32_t idesc = umma_idesc_bf16(2 * kBlockM, BN);
      const bool no_mma = gs.flags & GEMM_DBG_NO_MMA;
      SkRange rg(pid, npair, U, KB, sk_tiles);
      SkPiece pc;
      int i = 0, j = 0;
      while (rg.next(pc)) {
        const int acc = j & 1;
        mbar_wait(&tempty[acc], ((j >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * L::kAccCols;
        for (int kb = pc.kb0; kb < pc.kb1; ++kb, ++i) {
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
                               (kb > pc.kb0 || kk > 0) ? 1u : 0u);
            }
            umma_commit_pair(&empty[s], 0x3);
            if (kb == pc.kb1 - 1) umma_commit_pair(&tfull[acc], 0x3);
          }
          __syncwarp();
        }
        ++j;
      }
      if (trace && elect_one()) trace[4] = globaltimer();  // last MMA issued
    }
  } else {
    // ---------------- epilogue warps 2..5 (both CTAs): rows rank*128 + 32*(warp%4) + lane
    const int q = warp & 3;
    const int row = q * 32 + (threadIdx.x & 31);
    const int t = threadIdx.x - 64;
    const int cb = t >> 2, rl = (t & 3) * 8;  // staged read: column cb, rows rl + 32j + 0..7
    const bool skip = gs.flags & GEMM_DBG_NO_EPI;
    const uint32_t tempty0 = mapa_shared(smem_u32(tempty), 0);
    // partial slot of pair p, CTA rank r: ws[p][r][column][128 rows] fp32 (a 32-column chunk is
    // one contiguous 16 KB block)
    auto ws_col = [&](int p, int c) { return gs.sk_ws + ((long)(2 * p + rank) * kPairMaxBN + c) * kBlockM; };
    // fixup ring in the (then idle) pipeline stages: block b = (chunk b / nc, contributor b % nc)
    const int n_slots = min(L::kFixSlots, S * kStage / 16384);
    uint32_t pphase = 0;  // parity bits of the fixup barriers (one per slot)
    griddep_wait();  // residual / positions / norm statistics belong to earlier kernels
    wait_peer_rows(gs);
    // positions of every batch column once (the RoPE table lookups then need no dependent load)
    const bool pos_cached = ep.kind == EPI_QKV_ROPE && gs.Bt <= kPairMaxInvCols;
    if (pos_cached)
      for (int b = t; b < gs.Bt; b += 128) pos_smem[b] = __ldg(ep.pos + b);
    if (ep.ss_in) compute_inv_rms(ep, gs, inv_smem);
    if (ep.ss_in || pos_cached) epi_bar();
    SkRange rg(pid, npair, U, KB, sk_tiles);
    SkPiece pc;
    int j = 0;
    while (rg.next(pc)) {
      const int acc = j & 1;
      ++j;
      const int tile_n = pc.tile / bt, tile_b = pc.tile % bt;
      const int n0 = (2 * tile_n + rank) * kBlockM, b0 = tile_b * BN;
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * L::kAccCols;
      const bool owner = pc.kb0 == 0;
      // contributors to an owned tile: the following pairs whose ranges start inside it
      int c_end = pid + 1;
      if (owner && pc.kb1 < KB)
        while (c_end < npair && sk_start(c_end, npair, U, KB, sk_tiles) < (long)(pc.tile + 1) * KB) ++c_end;
      mbar_wait(&tfull[acc], ((j - 1) >> 1) & 1);
      tc_fence_after();
      if (trace && t == 0) trace[owner ? 5 : 8] = globaltimer();  // piece accumulated
      const int nc = owner ? c_end - pid - 1 : 0;  // contributors (only ever on this pair's last piece)
      const int nblk = nc * (BN / 32);
      auto issue = [&](int b) {  // bulk-copy fixup block b into its ring slot
        const int slot = b % n_slots, k = b / nc, c = pid + 1 + b % nc;
        mbar_arrive_expect_tx(&pbar[slot], 16384);
        bulk_g2s(smem + slot * 16384, ws_col(c, 32 * k), 16384, &pbar[slot], policy_evict_first());
      };
      if (nc > 0) {  // wait for the contributors' partials, start streaming them into shared memory
        if (t == 0) {
          for (int c = pid + 1; c < c_end; ++c) flag_wait(gs.sk_flags + 2 * c + rank, 1u);
          asm volatile("fence.proxy.async.global;" ::: "memory");
          for (int b = 0; b < min(n_slots, nblk); ++b) issue(b);
        }
        if (trace && t == 0) trace[6] = globaltimer();  // partials available
      }
      unsigned long long ta = 0, tb = 0, tc = 0, td = 0, tx;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        tx = trace ? globaltimer() : 0;
        // this chunk's global epilogue inputs first: their latency overlaps the TMEM drain
        EpiPre<32> pre;
        if (owner && !skip) epi_prefetch<32, 32>(ep, gs, n0 + rl, b0 + c0 + cb, pre, pos_cached ? pos_smem : nullptr);
        uint32_t r0[16], r1[16];
        tmem_ld16(taddr + c0, r0);
        tmem_ld16(taddr + c0 + 16, r1);
        tmem_ld_wait();
        if (trace) { const unsigned long long n = globaltimer(); ta += n - tx; tx = n; }
        if (c0 + 32 >= BN) {  // accumulator buffer fully read: the leader may reuse it
          tc_fence_before();
          __syncwarp();
          // relaxed: the TMEM reads are ordered by the tcgen05 fences; a release here would wait
          // for this thread's earlier global stores
          if ((threadIdx.x & 31) == 0) mbar_arrive_cluster_relaxed(tempty0 + acc * 8);
        }
        float v[32];
#pragma unroll
        for (int e = 0; e < 16; ++e) { v[e] = __uint_as_float(r0[e]); v[e + 16] = __uint_as_float(r1[e]); }
        if (!owner) {  // contributor: publish the partial (coalesced: a warp writes 32 rows of a column)
#pragma unroll
          for (int e = 0; e < 32; ++e) ws_col(pid, c0 + e)[row] = v[e];
          continue;
        }
        for (int i = 0; i < nc; ++i) {  // contributors in pair order: deterministic
          const int b = (c0 / 32) * nc + i, slot = b % n_slots;
          mbar_wait(&pbar[slot], (pphase >> slot) & 1);
          pphase ^= 1u << slot;
          const float* blk = (const float*)(smem + slot * 16384);
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] += blk[e * kBlockM + row];
          epi_bar();  // every thread is done with the slot
          if (t == 0 && b + n_slots < nblk) issue(b + n_slots);
        }
        if (trace) { const unsigned long long n = globaltimer(); tb += n - tx; tx = n; }
        if (skip) continue;
#pragma unroll
        for (int e = 0; e < 32; ++e) stg[pair_stg_index(e, row)] = v[e];
        epi_bar();
        float o[32];
#pragma unroll
        for (int e = 0; e < 32; e += 4) {
          const float4 a = *(const float4*)(stg + pair_stg_index(cb, rl + (e >> 3) * 32 + (e & 7)));
          o[e] = a.x; o[e + 1] = a.y; o[e + 2] = a.z; o[e + 3] = a.w;
        }
        if (trace) { const unsigned long long n = globaltimer(); tc += n - tx; tx = n; }
        epi_slice<32, 32, 32>(ep, gs, n0 + rl, b0 + c0 + cb, o, 2 * tile_n + rank, inv_smem,
                              pos_cached ? pos_smem : nullptr, &pre);
        epi_bar();  // staging is reused by the next chunk
        if (trace) { const unsigned long long n = globaltimer(); td += n - tx; tx = n; }
      }
      if (trace && t == 0 && owner) { trace[11] = ta; trace[12] = tb; trace[13] = tc; trace[14] = td; }
      if (!owner) {  // partial stored: release it to the owner
        __threadfence();
        epi_bar();
        if (trace && t == 0) trace[9] = globaltimer();  // partial published
        if (t == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(gs.sk_flags + 2 * pid + rank), "r"(1u) : "memory");
      } else if (c_end > pid + 1) {  // partials consumed: re-arm the contributors' flags
        epi_bar();
        if (t == 0)
          for (int c = pid + 1; c < c_end; ++c) gs.sk_flags[2 * c + rank] = 0u;
      }
    }
  }
  if (trace && threadIdx.x == 64) trace[7] = globaltimer();  // epilogue done
  tc_fence_before();
  cluster_sync_all();  // the peer's last remote arrivals and TMEM reads are done
  if (warp == 1) tmem_free_pair<L::kTmemCols>(tmem_base);
  if (trace && threadIdx.x == 0) trace[10] = globaltimer();
}

}  // namespace gh
