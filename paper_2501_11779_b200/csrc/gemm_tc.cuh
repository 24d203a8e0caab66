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
// Scheduling is persistent "cluster split-K": the grid is a set of thread-block clusters of C
// CTAs (C in {1, 2, 4, 8}, chosen per GEMM shape on the host); cluster c processes output tiles
// c, c + n_clusters, ... and CTA rank r of the cluster computes k-blocks [r*KB/C, (r+1)*KB/C) of
// every tile it visits, so weights are streamed by up to all 148 SMs even when the GEMM has
// fewer output tiles than SMs.  The accumulator is double-buffered in TMEM so the epilogue of
// tile j overlaps the TMA/MMA mainloop of tile j+1.  The C fp32 partials of a tile are combined
// through distributed shared memory: every CTA publishes its partial into its own shared
// memory, signals its peers with remote mbarrier arrivals, then reduces a 128/C-row slice of the
// tile by reading all C partials in rank order (deterministic) and runs the epilogue on that
// slice with direct, coalesced global stores.  Clusters are gang-scheduled, so waiting on peers
// can never deadlock, and no global workspace or atomics are involved.
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

GH_DEV float silu_f(float g) { return g / (1.0f + __expf(-g)); }
// tensor-core epilogues (bf16 storage, tolerance-checked): fast reciprocal instead of IEEE division
GH_DEV float silu_fast(float g) { return __fdividef(g, 1.0f + __expf(-g)); }

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

// ------------------------------------------------------------------ cluster split-K epilogue
GH_DEV void epi_bar() { asm volatile("bar.sync 1, 128;\n" ::: "memory"); }  // the 4 epilogue warps

// Slice epilogue: thread t of the 128 epilogue threads owns batch column b and En weight rows n
// of the output tile, as En/8 chunks of 8 consecutive rows RS rows apart (RS = 8: one run of En
// consecutive rows).  It has the fully reduced fp32 values in `v` and writes its outputs directly
// (row-major [b][n]).  RS > 8 lets the threads sharing a column interleave their chunks so that
// every store instruction of a warp covers whole 32-byte sectors.
template <int En, int RS>
GH_DEV void store_run_bf16(uint16_t* dst, const float* v) {
  if ((((uintptr_t)dst) & 15) == 0 && En % 8 == 0) {
#pragma unroll
    for (int e = 0; e < En; e += 8) {
      uint4 o;
      o.x = pack_bf16x2(v[e], v[e + 1]);
      o.y = pack_bf16x2(v[e + 2], v[e + 3]);
      o.z = pack_bf16x2(v[e + 4], v[e + 5]);
      o.w = pack_bf16x2(v[e + 6], v[e + 7]);
      *(uint4*)(dst + (e >> 3) * RS) = o;
    }
  } else {
#pragma unroll
    for (int e = 0; e < En; ++e) dst[(e >> 3) * RS + (e & 7)] = f32_to_bf16(v[e]);
  }
}

constexpr int kMaxInvCols = 256;  // batch columns whose fused-RMSNorm scale is kept in smem (larger: unfused)

// 1/rms of every batch column of the GEMM input, from the producer's per-slice sums of squares
// (summed in slice order: deterministic).  Run once per CTA by the epilogue warps.
GH_DEV void compute_inv_rms(const EpiParams& ep, const GemmShape& gs, float* inv) {
  const float* __restrict__ ssp = ep.ss_in;
  const int ns = ep.ss_in_slices, Bt = gs.Bt;
  const float dim = (float)ep.ss_dim, eps = ep.ss_eps;
  const int t = threadIdx.x - 64;
  if (Bt <= 128) {  // one column per thread: 16 slices in flight
    if (t < Bt) {
      float ss = 0.f;
#pragma unroll 16
      for (int s = 0; s < ns; ++s) ss += __ldg(ssp + (long)s * Bt + t);  // slice order: deterministic
      inv[t] = 1.0f / sqrtf(ss / dim + eps);
    }
    return;
  }
  // up to 8 columns per thread (Bt <= 1024) summed together, so that 8 x 4 loads are in flight
  // at once (the sums of a large batch otherwise serialise on load latency); slice order is kept
  constexpr int kCols = 8;
  for (int b0 = 0; b0 < Bt; b0 += 128 * kCols) {
    float acc[kCols];
#pragma unroll
    for (int k = 0; k < kCols; ++k) acc[k] = 0.f;
#pragma unroll 4
    for (int s = 0; s < ns; ++s) {
#pragma unroll
      for (int k = 0; k < kCols; ++k) {
        const int b = b0 + t + 128 * k;
        if (b < Bt) acc[k] += __ldg(ssp + (long)s * Bt + b);
      }
    }
#pragma unroll
    for (int k = 0; k < kCols; ++k) {
      const int b = b0 + t + 128 * k;
      if (b < Bt) inv[b] = 1.0f / sqrtf(acc[k] / dim + eps);
    }
  }
}

// Global inputs of a slice epilogue (residual rows, x rows to copy, RoPE table entries), loaded
// ahead of the epilogue arithmetic so that their latency overlaps the TMEM drain / staging
// (epi_prefetch); ok == false: the tile edge or alignment needs the direct path in epi_slice.
template <int En>
struct EpiPre {
  uint4 a[En / 8 > 0 ? En / 8 : 1];  // residual (STORE_RESID) or x to copy (QKV_ROPE)
  float2 cs[En / 2 > 0 ? En / 2 : 1];  // RoPE (cos, sin) of every row pair (QKV_ROPE)
  bool ok;
};

template <int En, int RS = 8>
GH_DEV void epi_prefetch(const EpiParams& ep, const GemmShape& gs, int n, int b, EpiPre<En>& p,
                         const int* pos_smem = nullptr) {
  auto off = [](int e) { return (e >> 3) * RS + (e & 7); };
  p.ok = false;
  if (En % 8 || b >= gs.Bt || n + off(En - 1) >= gs.N) return;
  if (ep.kind == EPI_STORE_RESID) {
    const uint16_t* rp = (const uint16_t*)ep.resid + (long)b * ep.ldr + n;
    if (((uintptr_t)rp & 15) != 0) return;
#pragma unroll
    for (int j = 0; j < En / 8; ++j) p.a[j] = __ldg((const uint4*)(rp + j * RS));
    p.ok = true;
  } else if (ep.kind == EPI_QKV_ROPE) {
    if (ep.xcopy_src && n < ep.xcopy_rows) {
      const uint16_t* xs = (const uint16_t*)ep.xcopy_src + (long)b * ep.xcopy_ld + n;
      const uint16_t* xd = (const uint16_t*)ep.out + (long)b * ep.ldo + n - ep.xcopy_rows;
      if (n + off(En - 1) >= ep.xcopy_rows || ((uintptr_t)xs & 15) || ((uintptr_t)xd & 15)) return;
#pragma unroll
      for (int j = 0; j < En / 8; ++j) p.a[j] = __ldg((const uint4*)(xs + j * RS));
    }
    if (n < ep.rope_rows) {
      const float2* cs = ep.rope + (long)(pos_smem ? pos_smem[b] : __ldg(ep.pos + b)) * (ep.d_head >> 1);
      int hb = 0;
#pragma unroll
      for (int e = 0; e < En; e += 2) {
        if ((e & 7) == 0) hb = ((n + off(e)) % ep.d_head) >> 1;
        p.cs[e >> 1] = __ldg(cs + hb + ((e & 7) >> 1));
      }
    }
    p.ok = true;
  }
}

template <int BN, int En, int RS = 8>
GH_DEV void epi_slice(const EpiParams& ep, const GemmShape& gs, int n, int b, float (&v)[En], int slice,
                      const float* inv, const int* pos_smem = nullptr, const EpiPre<En>* pre = nullptr) {
  // element e of this thread is output row n + off(e)
  auto off = [](int e) { return (e >> 3) * RS + (e & 7); };
  const bool col_ok = b < gs.Bt;
  const bool full = n + off(En - 1) < gs.N;
  const bool pok = pre && pre->ok;
  if (ep.ss_in && col_ok) {  // fused RMSNorm of the GEMM input
    const float sc = inv[b];
#pragma unroll
    for (int e = 0; e < En; ++e) v[e] *= sc;
  }
  bool resid_added = false;
  if (pok && ep.kind == EPI_STORE_RESID) {  // residual from the prefetched rows
#pragma unroll
    for (int j = 0; j < En / 8; ++j) {
      const uint32_t w[4] = {pre->a[j].x, pre->a[j].y, pre->a[j].z, pre->a[j].w};
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        v[8 * j + 2 * h] += __uint_as_float(w[h] << 16);
        v[8 * j + 2 * h + 1] += __uint_as_float(w[h] & 0xffff0000u);
      }
    }
    resid_added = true;
  }
  if (ep.ss_out) {  // sums of squares of the rounded outputs, reduced over the slice's threads
    constexpr int kRuns = 128 / BN;
    float sq = 0.f;
    if (col_ok && ep.kind == EPI_STORE_RESID) {
      if (resid_added) {
#pragma unroll
        for (int e = 0; e < En; ++e) {
          const float y = bf16_to_f32(f32_to_bf16(v[e]));
          sq = fmaf(y, y, sq);
        }
      } else {
        const uint16_t* rp = (const uint16_t*)ep.resid + (long)b * ep.ldr + n;
#pragma unroll
        for (int e = 0; e < En; ++e) {
          if (full || n + off(e) < gs.N) {
            const float y = bf16_to_f32(f32_to_bf16(v[e] + bf16_to_f32(rp[off(e)])));
            sq = fmaf(y, y, sq);
          }
        }
      }
    }
#pragma unroll
    for (int o = 1; o < kRuns; o <<= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    if (col_ok && ((threadIdx.x - 64) % kRuns) == 0) ep.ss_out[(long)slice * gs.Bt + b] = sq;
  }
  if (gs.flags & GEMM_DBG_NO_STORE) {  // diagnostics: no output stores
    if (col_ok && v[0] == 12345.f) ((float*)ep.out)[0] = v[1];
    return;
  }
  switch (ep.kind) {
    case EPI_STORE:
    case EPI_STORE_RESID: {
      if (!col_ok) return;
      if (ep.kind == EPI_STORE_RESID && !resid_added) {
        const uint16_t* rp = (const uint16_t*)ep.resid + (long)b * ep.ldr + n;
        if (full && En % 8 == 0 && ((uintptr_t)rp & 15) == 0) {
          uint4 rr[En / 8 > 0 ? En / 8 : 1];
#pragma unroll
          for (int e = 0; e < En / 8; ++e) rr[e] = __ldg((const uint4*)(rp + e * RS));
#pragma unroll
          for (int e = 0; e < En / 8; ++e) {
            const uint32_t w[4] = {rr[e].x, rr[e].y, rr[e].z, rr[e].w};
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              v[8 * e + 2 * h] += __uint_as_float(w[h] << 16);
              v[8 * e + 2 * h + 1] += __uint_as_float(w[h] & 0xffff0000u);
            }
          }
        } else {
#pragma unroll
          for (int e = 0; e < En; ++e) v[e] += (full || n + off(e) < gs.N) ? bf16_to_f32(rp[off(e)]) : 0.f;
        }
      }
      uint16_t* op = (uint16_t*)ep.out + (long)b * ep.ldo + n;
      if (full) store_run_bf16<En, RS>(op, v);
      else
#pragma unroll
        for (int e = 0; e < En; ++e)
          if (n + off(e) < gs.N) op[off(e)] = f32_to_bf16(v[e]);
      return;
    }
    case EPI_QKV_ROPE: {
      if (!col_ok) return;
      if (pok) {  // prefetched x rows and RoPE entries
        if (ep.xcopy_src && n < ep.xcopy_rows) {
          uint16_t* xd = (uint16_t*)ep.out + (long)b * ep.ldo + n - ep.xcopy_rows;
#pragma unroll
          for (int j = 0; j < En / 8; ++j) *(uint4*)(xd + j * RS) = pre->a[j];
        }
        if (n < ep.rope_rows) {
#pragma unroll
          for (int e = 0; e < En; e += 2) {
            const float2 c = pre->cs[e >> 1];
            const float a = v[e], o = v[e + 1];
            v[e] = a * c.x - o * c.y;
            v[e + 1] = a * c.y + o * c.x;
          }
        }
        store_run_bf16<En, RS>((uint16_t*)ep.out + (long)b * ep.ldo + n, v);
        return;
      }
      if (ep.xcopy_src && n < ep.xcopy_rows) {  // x into the message's x slot (fused RMSNorm path)
        const uint16_t* xs = (const uint16_t*)ep.xcopy_src + (long)b * ep.xcopy_ld + n;
        uint16_t* xd = (uint16_t*)ep.out + (long)b * ep.ldo + n - ep.xcopy_rows;
        if (En % 8 == 0 && n + off(En - 1) < ep.xcopy_rows && ((uintptr_t)xs & 15) == 0 && ((uintptr_t)xd & 15) == 0) {
#pragma unroll
          for (int e = 0; e < En; e += 8) *(uint4*)(xd + off(e)) = __ldg((const uint4*)(xs + off(e)));
        } else {
#pragma unroll
          for (int e = 0; e < En; ++e)
            if (n + off(e) < ep.xcopy_rows) xd[off(e)] = xs[off(e)];
        }
      }
      if (n < ep.rope_rows) {
        const float2* cs = ep.rope + (long)(pos_smem ? pos_smem[b] : ep.pos[b]) * (ep.d_head >> 1);
        int hb = 0;  // (row % d_head) / 2 at the start of the current 8-row chunk (a chunk never crosses a head)
#pragma unroll
        for (int e = 0; e < En; e += 2) {
          if ((e & 7) == 0) hb = ((n + off(e)) % ep.d_head) >> 1;
          const float2 c = cs[hb + ((e & 7) >> 1)];
          const float a = v[e], o = v[e + 1];
          // pair (a, o) = (even, odd): even' = a cos - o sin, odd' = a sin + o cos
          v[e] = a * c.x - o * c.y;
          v[e + 1] = a * c.y + o * c.x;
        }
      }
      uint16_t* op = (uint16_t*)ep.out + (long)b * ep.ldo + n;
      if (full) store_run_bf16<En, RS>(op, v);
      else
#pragma unroll
        for (int e = 0; e < En; ++e)
          if (n + off(e) < gs.N) op[off(e)] = f32_to_bf16(v[e]);
      return;
    }
    case EPI_SWIGLU: {
      if (!col_ok) return;
      float h[En / 2];
#pragma unroll
      for (int e = 0; e < En / 2; ++e) h[e] = silu_fast(v[2 * e]) * v[2 * e + 1];
      // output element e/2 of chunk j lands at (n + j*RS)/2 + (e%8)/2: chunks of 4, RS/2 apart
      uint16_t* op = (uint16_t*)ep.out + (long)b * ep.ldo + (n >> 1);
      if (full && En % 8 == 0 && (((uintptr_t)op) & 7) == 0) {
#pragma unroll
        for (int e = 0; e < En / 2; e += 4) {
          uint2 o;
          o.x = pack_bf16x2(h[e], h[e + 1]);
          o.y = pack_bf16x2(h[e + 2], h[e + 3]);
          *(uint2*)(op + (e >> 2) * (RS / 2)) = o;
        }
      } else {
#pragma unroll
        for (int e = 0; e < En / 2; ++e)
          if (n + off(2 * e) < gs.N) op[off(2 * e) >> 1] = f32_to_bf16(h[e]);
      }
      return;
    }
    default: {
      // EPI_LOGITS_ARGMAX: logits (optional) and (max, argmax) over the slice per column b
      float best = -INFINITY;
      int bi = 0x7fffffff;
#pragma unroll
      for (int e = 0; e < En; ++e) {
        const int r = n + off(e);
        if (r < gs.N && (v[e] > best || (v[e] == best && r < bi))) { best = v[e]; bi = r; }
      }
      if (ep.logits && col_ok) {
        float* lp = ep.logits + (long)b * ep.ldl + n;
#pragma unroll
        for (int e = 0; e < En; ++e)
          if (n + off(e) < gs.N) lp[off(e)] = v[e];
      }
      // reduce over the 128/BN threads that share column b (adjacent lanes)
      constexpr int kRuns = 128 / BN;
#pragma unroll
      for (int o = 1; o < kRuns; o <<= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
      }
      if (col_ok && ((threadIdx.x - 64) % kRuns) == 0)
        ep.part[(long)slice * gs.Bt + b] = make_float2(best, __int_as_float(bi));
      return;
    }
  }
}

template <int BN>
struct GemmSmem {
  static constexpr int kABytes = kBlockM * kBlockK * 2;  // 16 KB
  static constexpr int kBBytes = BN * kBlockK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kMaxStages = 16;
  // receive buffer: C pushed partial slices [C][BN][128/C] (one tile of fp32 in total)
  static constexpr int kEpiBytes = BN * 128 * 4;
  static constexpr uint32_t kAccCols = BN < 32 ? 32 : BN;  // one accumulator buffer
  static constexpr uint32_t kTmemCols = 2 * kAccCols <= 64 ? 64 : 2 * kAccCols <= 128 ? 128
                                      : 2 * kAccCols <= 256 ? 256 : 512;
  static constexpr int kBarBytes = (2 * kMaxStages + 8) * 8 + 16 + kMaxInvCols * 4;
  GH_HD static int epi_offset(int stages) { return stages * kStageBytes; }
  GH_HD static int bar_offset(int stages) { return stages * kStageBytes + kEpiBytes; }
  GH_HD static int bytes(int stages) { return bar_offset(stages) + kBarBytes + 1024; }
  static int max_stages(int budget) {
    int s = (budget - kEpiBytes - kBarBytes - 1024) / kStageBytes;
    return s > kMaxStages ? kMaxStages : s;
  }
};

// Receive buffer of the CTA that owns rows [r*R, (r+1)*R) of a tile (R = 128/C):
//   recv[src rank p][batch column b][row_local]   (fp32, C*BN*R floats = one full partial)
// Every CTA pushes each of its partial values into the owner's buffer with posted DSMEM stores
// while it drains TMEM, so the owner reduces from local shared memory (no remote round trip).
// The 16-byte chunks of a row are XOR-swizzled by the batch column so that the owner's float4
// reads of consecutive columns hit distinct banks.
template <int BN, int C>
GH_DEV int recv_index(int p, int b, int rl) {
  constexpr int R = 128 / C;
  return (p * BN + b) * R + ((((rl >> 2) ^ (b & (R / 4 - 1)))) << 2) + (rl & 3);
}
template <int BN, int C>
GH_DEV void push_partial(uint32_t recv_saddr, int rank, int row, const float* v16, int c0) {
  constexpr int R = 128 / C;
  const int owner = row / R, rl = row % R;
  const uint32_t dst = mapa_shared(recv_saddr, owner);
#pragma unroll
  for (int e = 0; e < 16; ++e)
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(dst + (uint32_t)recv_index<BN, C>(rank, c0 + e, rl) * 4),
                 "f"(v16[e]) : "memory");
}

// Tier-1 tensor parallelism: all-reduce of this thread's fully K-reduced fp32 values v (output
// rows rl .. rl+En-1 of the slice, batch column b) across the ep.tp_n ranks, inside the epilogue,
// with no fence and no separate flag: every value travels to each peer as one 8-byte word
// {value, sequence number} (a single NVLink write, so the pair is seen whole or not at all), and a
// peer's partial is known to have arrived when its words carry this all-reduce's sequence number
// (the low-latency scheme of NCCL's LL protocol).  Every rank then sums the tp_n partials in rank
// order, so the result (and everything computed from it) is bit-identical on all ranks.  All ranks
// run the same plan (plan_gemm_tp) and visit their tiles in the same order, and every CTA of the
// persistent grid is resident, so the waits cannot deadlock; receive buffers alternate between
// two parities, so a word can only be overwritten after its reader has consumed it.
// Receive buffer of rank p: [src rank][slice fi][row in slice][BN columns] of {value, seq}.  A slice
// is one contiguous block and consecutive threads hold consecutive columns, so each store of a warp
// writes a contiguous run (256 B when a thread owns a whole column run); columns past the batch are
// not sent.
GH_DEV void st_sys_u2(uint2* p, uint32_t a, uint32_t b, bool weak) {
  if (weak) asm volatile("st.global.cg.v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(a), "r"(b));
  else asm volatile("st.relaxed.sys.global.v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(a), "r"(b) : "memory");
}
GH_DEV uint2 ld_sys_u2(const uint2* p, bool weak) {
  uint2 r;
  if (weak) asm volatile("ld.global.cg.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  else asm volatile("ld.relaxed.sys.global.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p) : "memory");
  return r;
}
template <int BN, int C, int En>
GH_DEV void tp_allreduce(const EpiParams& ep, const GemmShape& gs, int rl, int b, float (&v)[En], int fi) {
  constexpr int R = 128 / C;
  if (b >= gs.Bt || (ep.tp_dbg & 4)) return;  // columns past the batch: nothing to exchange
  const long blk = (long)gs.b_tiles * gs.n_tiles * 128 * BN;  // one source rank's words
  const long at = (long)fi * R * BN + (long)rl * BN + (b % BN);
  const uint32_t seq = ep.tp_seq;
  // (rank loops are unrolled over kMaxTp so that tp_dst[] is indexed by constants)
  if (!(ep.tp_dbg & 2)) {
#pragma unroll
    for (int p = 0; p < kMaxTp; ++p) {
      if (p >= ep.tp_n || p == ep.tp_rank) continue;
      uint2* dst = (uint2*)ep.tp_dst[p] + ep.tp_rank * blk + at;
#pragma unroll
      for (int e = 0; e < En; ++e) st_sys_u2(dst + (long)e * BN, __float_as_uint(v[e]), seq, ep.tp_dbg & 16);
    }
  }
  const uint2* src = (const uint2*)(ep.tp_rank == 0 ? ep.tp_dst[0] : ep.tp_rank == 1 ? ep.tp_dst[1]
                                    : ep.tp_rank == 2 ? ep.tp_dst[2] : ep.tp_dst[3]) + at;  // local buffer
  const bool wait = !(ep.tp_dbg & 1), weak = ep.tp_dbg & 8;
  // words in flight per poll (register budget); never more than the thread's run
  constexpr int kC = En < 8 ? En : (BN == 64 ? 4 : 8);
  static_assert(kC <= En && En % kC == 0, "chunks tile the run");
#pragma unroll
  for (int c = 0; c < En; c += kC) {
    float a[kC];
#pragma unroll
    for (int p = 0; p < kMaxTp; ++p) {  // rank order: identical sums on every rank
      if (p >= ep.tp_n) break;
      float x[kC];
      if (p == ep.tp_rank) {
#pragma unroll
        for (int e = 0; e < kC; ++e) x[e] = v[c + e];
      } else {
        // the chunk's words requested at once (a poll per word would serialise the loads behind
        // their branches), then only the stale ones polled again
        const uint2* w_at = src + p * blk + (long)c * BN;
        uint2 w[kC];
#pragma unroll
        for (int e = 0; e < kC; ++e) w[e] = ld_sys_u2(w_at + (long)e * BN, weak);
        bool stale = false;
#pragma unroll
        for (int e = 0; e < kC; ++e) stale |= w[e].y != seq;
        while (wait && stale) {
          stale = false;
#pragma unroll
          for (int e = 0; e < kC; ++e)
            if (w[e].y != seq) {
              w[e] = ld_sys_u2(w_at + (long)e * BN, weak);
              stale |= w[e].y != seq;
            }
        }
#pragma unroll
        for (int e = 0; e < kC; ++e) x[e] = __uint_as_float(w[e].x);
      }
#pragma unroll
      for (int e = 0; e < kC; ++e) a[e] = p == 0 ? x[e] : a[e] + x[e];
    }
#pragma unroll
    for (int e = 0; e < kC; ++e) v[c + e] = a[e];
  }
}

template <int BN, int C>
GH_DEV void reduce_and_store(const EpiParams& ep, const GemmShape& gs, const float* recv, int r, int n0,
                             int b0, int tile_n, uint32_t consumed_saddr, unsigned long long* tr,
                             const float* inv, uint64_t* ready, uint32_t ready_parity) {
  // thread -> (column b, run of En rows inside this CTA's slice of R = 128/C rows)
  constexpr int R = 128 / C;
  constexpr int En = BN / C;
  constexpr int kRuns = 128 / BN;
  const int t = threadIdx.x - 64;
  const int b = t / kRuns;
  const int rl = (t % kRuns) * En;
  // the epilogue's global inputs are requested before waiting for the peers' partials (runs of
  // up to 32 rows: longer runs would not fit the register budget)
  constexpr int Ep = En <= 32 ? En : 1;
  EpiPre<Ep> pre;
  pre.ok = false;
  if constexpr (En <= 32) epi_prefetch<En>(ep, gs, n0 + r * R + rl, b0 + b, pre);
  mbar_wait_cluster(ready, ready_parity);  // every peer's push into my buffer is visible
  if (tr) tr[11] = globaltimer();
  float v[En];
#pragma unroll
  for (int e = 0; e < En; e += 4) {
    float4 a = *(const float4*)(recv + recv_index<BN, C>(0, b, rl + e));
#pragma unroll
    for (int p = 1; p < C; ++p) {  // rank order: deterministic
      const float4 q = *(const float4*)(recv + recv_index<BN, C>(p, b, rl + e));
      a.x += q.x; a.y += q.y; a.z += q.z; a.w += q.w;
    }
    v[e] = a.x; v[e + 1] = a.y; v[e + 2] = a.z; v[e + 3] = a.w;
  }
  if (tr) tr[15] = globaltimer();
  // my receive buffer is free again: every peer may push its next tile
  epi_bar();
  if (threadIdx.x == 64)
    for (int p = 0; p < C; ++p) mbar_arrive_cluster_relaxed(mapa_shared(consumed_saddr, p));
  if constexpr (En <= 32) {  // plan_gemm_tp keeps runs <= 32 rows (register budget)
    if (ep.tp_n > 1) {
      tp_allreduce<BN, C, En>(ep, gs, rl, b0 + b, v, (b0 / BN) * gs.n_tiles * C + tile_n * C + r);
      if (tr) tr[13] = globaltimer();  // (diagnostics) all-reduce done
    }
  } else {
    if (ep.tp_n > 1) __trap();
  }
  if constexpr (En <= 32) epi_slice<BN, En>(ep, gs, n0 + r * R + rl, b0 + b, v, tile_n * C + r, inv, nullptr, &pre);
  else epi_slice<BN, En>(ep, gs, n0 + r * R + rl, b0 + b, v, tile_n * C + r, inv);
}

// Wide batch tiles (BN > 128, one batch tile for 129..192 columns): thread t owns whole
// columns t, t + 128, ... of the CTA's R-row slice (no cross-thread reduction in the epilogue),
// processed one at a time; the receive buffer is released after the last one.
template <int BN, int C>
GH_DEV void reduce_and_store_wide(const EpiParams& ep, const GemmShape& gs, const float* recv, int r, int n0,
                                  int b0, int tile_n, uint32_t consumed_saddr, const float* inv, uint64_t* ready,
                                  uint32_t ready_parity) {
  constexpr int R = 128 / C;
  constexpr int En = R;
  constexpr int Ep = En <= 32 ? En : 1;
  const int t = threadIdx.x - 64;
#pragma unroll 1
  for (int k = 0; k < (BN + 127) / 128; ++k) {
    const int b = t + 128 * k;
    EpiPre<Ep> pre;
    pre.ok = false;
    if constexpr (En <= 32)
      if (b < BN) epi_prefetch<En>(ep, gs, n0 + r * R, b0 + b, pre);
    if (k == 0) mbar_wait_cluster(ready, ready_parity);  // every peer's push into my buffer is visible
    if (b < BN) {
      float v[En];
#pragma unroll
      for (int e = 0; e < En; e += 4) {
        float4 a = *(const float4*)(recv + recv_index<BN, C>(0, b, e));
#pragma unroll
        for (int p = 1; p < C; ++p) {  // rank order: deterministic
          const float4 q = *(const float4*)(recv + recv_index<BN, C>(p, b, e));
          a.x += q.x; a.y += q.y; a.z += q.z; a.w += q.w;
        }
        v[e] = a.x; v[e + 1] = a.y; v[e + 2] = a.z; v[e + 3] = a.w;
      }
      // BN template of epi_slice = 128: one thread per column (no cross-thread reductions)
      if constexpr (En <= 32) epi_slice<128, En>(ep, gs, n0 + r * R, b0 + b, v, tile_n * C + r, inv, nullptr, &pre);
      else epi_slice<128, En>(ep, gs, n0 + r * R, b0 + b, v, tile_n * C + r, inv);
    }
  }
  epi_bar();  // my receive buffer is free again: every peer may push its next tile
  if (threadIdx.x == 64)
    for (int p = 0; p < C; ++p) mbar_arrive_cluster_relaxed(mapa_shared(consumed_saddr, p));
}

// Rows delivered by the peer transport (GemmShape::xwait): spin on every shard's flag word, then
// order the async-proxy (TMA) reads that follow after the acquiring loads.
GH_DEV void wait_peer_rows(const GemmShape& gs) {
  if (!gs.xwait) return;
  for (int j = 0; j < gs.xwait_n; ++j) flag_wait_sys(gs.xwait + j, gs.xwait_val);
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

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
  uint64_t* ready = tempty + 2;              // all C partials of the tile published (count C)
  uint64_t* consumed = ready + 1;            // all C peers finished reading my partial (count C)
  uint32_t* tmem_slot = (uint32_t*)(consumed + 1);
  float* inv_smem = (float*)(consumed + 4);  // [kMaxInvCols] fused-RMSNorm scales

  const int warp = threadIdx.x >> 5;
  const int KB = gs.kb_total;
  const int C = (int)cluster_nctarank();
  const int rank = (int)cluster_ctarank();
  const int cid = (int)cluster_id_x(), ncl = (int)cluster_count_x();
  const int n_tiles_total = gs.n_tiles * gs.b_tiles;
  const int kbA = rank * KB / C, kbB = (rank + 1) * KB / C;  // this CTA's k-range of every tile
  const int nkb = kbB - kbA;
  const int my_tiles = cid < n_tiles_total ? (n_tiles_total - 1 - cid) / ncl + 1 : 0;
  unsigned long long* trace = gs.trace ? gs.trace + blockIdx.x * 16 : nullptr;
  if (trace && threadIdx.x == 0) trace[0] = globaltimer();

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmW);
    prefetch_tmap(&tmX);
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 4); }
    mbar_init(ready, C);      // one arrival per CTA of the cluster
    mbar_init(consumed, C);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<L::kTmemCols>(tmem_slot);
  tc_fence_before();
  if (C > 1) cluster_sync_all();  // peers' barriers are initialised before any remote arrive
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_launch_dependents();

  if (warp == 0) {
    // ---------------- TMA producer: k-blocks [kbA, kbB) of each of this cluster's tiles
    if (elect_one()) {
      const bool hint = !(gs.flags & GEMM_DBG_NO_HINT);
      const bool load_x = !(gs.flags & GEMM_DBG_NO_X);
      const uint64_t pol_w = hint ? policy_evict_first() : 0;  // weights stream through once
      const uint64_t pol_x = hint ? policy_evict_last() : 0;   // activations are re-read by every tile
      const int total = my_tiles * nkb;
      const int pre = min(S, total);
      // Weights do not depend on the previous kernel: the first S stages of weights are requested
      // before griddepcontrol.wait (overlapping the predecessor's tail), activations after it.
      for (int i = 0; i < pre; ++i) {
        const int tile = cid + (i / nkb) * ncl, kb = kbA + i % nkb;
        mbar_arrive_expect_tx(&full[i], load_x ? L::kStageBytes : L::kABytes);
        uint8_t* sa = smem + i * L::kStageBytes;
        if (hint) tma_load_2d(sa, &tmW, 0, ((tile / gs.b_tiles) * KB + kb) * kBlockM, &full[i], pol_w);
        else tma_load_2d_nohint(sa, &tmW, 0, ((tile / gs.b_tiles) * KB + kb) * kBlockM, &full[i]);
      }
      if (trace) trace[1] = globaltimer();
      griddep_wait();
      wait_peer_rows(gs);
      if (trace) trace[2] = globaltimer();
      for (int i = 0; i < pre && load_x; ++i) {
        const int tile = cid + (i / nkb) * ncl, kb = kbA + i % nkb;
        uint8_t* sb = smem + i * L::kStageBytes + L::kABytes;
        if (hint) tma_load_2d(sb, &tmX, kb * kBlockK, (tile % gs.b_tiles) * BN, &full[i], pol_x);
        else tma_load_2d_nohint(sb, &tmX, kb * kBlockK, (tile % gs.b_tiles) * BN, &full[i]);
      }
      for (int i = pre; i < total; ++i) {
        const int tile = cid + (i / nkb) * ncl, kb = kbA + i % nkb;
        const int tile_n = tile / gs.b_tiles, tile_b = tile % gs.b_tiles;
        const int s = i % S;
        mbar_wait(&empty[s], ((i / S) & 1) ^ 1);
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
      prefetch_l2_share(gs.pf, gs.pf_bytes, blockIdx.x, gridDim.x);
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: one accumulator buffer per tile, alternating
    const uint32_t idesc = umma_idesc_bf16(kBlockM, BN);
    const bool no_mma = gs.flags & GEMM_DBG_NO_MMA;
    int i = 0;
    for (int j = 0; j < my_tiles; ++j) {
      if (trace && j == 0 && elect_one()) { mbar_wait(&full[0], 0); trace[3] = globaltimer(); }
      __syncwarp();
      const int acc = j & 1;
      mbar_wait(&tempty[acc], ((j >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * L::kAccCols;
      for (int k = 0; k < nkb; ++k, ++i) {
        const int s = i % S;
        mbar_wait(&full[s], (i / S) & 1);
        tc_fence_after();
        if (elect_one()) {
          if (no_mma) {
            mbar_arrive(&empty[s]);
            if (k == nkb - 1) mbar_arrive(&tfull[acc]);
          } else {
            const uint32_t sa = smem_u32(smem + s * L::kStageBytes);
            const uint64_t da = umma_desc_sw128(sa);
            const uint64_t db = umma_desc_sw128(sa + L::kABytes);
#pragma unroll
            for (int kk = 0; kk < kBlockK / 16; ++kk)
              // +32 bytes along K inside the 128-byte swizzle atom = +2 in the >>4 address field
              umma_bf16(d_tmem, da + (uint64_t)(kk * 2), db + (uint64_t)(kk * 2), idesc,
                        (k > 0 || kk > 0) ? 1u : 0u);
            umma_commit(&empty[s]);
            if (k == nkb - 1) umma_commit(&tfull[acc]);
          }
        }
        __syncwarp();
      }
    }
    if (trace && elect_one()) trace[4] = globaltimer();
  } else {
    // ---------------- epilogue warps 2..5
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row = q * 32 + (threadIdx.x & 31);
    const bool skip = gs.flags & GEMM_DBG_NO_EPI;
    griddep_wait();          // residual / positions belong to earlier kernels
    wait_peer_rows(gs);
    if (ep.ss_in) {          // overlaps the mainloop: the epilogue warps are idle until tile 0
      compute_inv_rms(ep, gs, inv_smem);
      epi_bar();
    }
    const uint32_t red_saddr = smem_u32(esm);
    float* red = (float*)esm;
    for (int j = 0; j < my_tiles; ++j) {
      const int tile = cid + j * ncl;
      const int tile_n = tile / gs.b_tiles, tile_b = tile % gs.b_tiles;
      const int n0 = tile_n * kBlockM, b0 = tile_b * BN;
      const int acc = j & 1;
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * L::kAccCols;
      mbar_wait(&tfull[acc], (j >> 1) & 1);
      tc_fence_after();
      const bool tr = trace && threadIdx.x == 64 && j == my_tiles - 1;
      if (tr) trace[7] = globaltimer();
      {
        // drain TMEM and push every value to the CTA that owns its rows, release TMEM
        if (tr) trace[8] = globaltimer();
        if (j > 0) mbar_wait_cluster(consumed, (j - 1) & 1);  // every owner has read tile j-1
        if (tr) trace[9] = globaltimer();
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 16) {
          uint32_t r[16];
          tmem_ld16(taddr + c0, r);
          tmem_ld_wait();
          float v16[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) v16[e] = __uint_as_float(r[e]);
          switch (C) {
            case 1: push_partial<BN, 1>(red_saddr, rank, row, v16, c0); break;
            case 2: push_partial<BN, 2>(red_saddr, rank, row, v16, c0); break;
            case 4: push_partial<BN, 4>(red_saddr, rank, row, v16, c0); break;
            default: push_partial<BN, 8>(red_saddr, rank, row, v16, c0); break;
          }
        }
        tc_fence_before();
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(&tempty[acc]);
        epi_bar();  // the four warps' pushes happen before thread 64's cluster fence
        if (threadIdx.x == 64) {
          fence_acq_rel_cluster();
          for (int p = 0; p < C; ++p) mbar_arrive_cluster_relaxed(mapa_shared(smem_u32(ready), p));
        }
        if (tr) trace[10] = globaltimer();
        unsigned long long* rt = tr ? trace : nullptr;
        const uint32_t rp = j & 1;
        if (!skip) {
          if constexpr (BN > 128) {
            switch (C) {
              case 4: reduce_and_store_wide<BN, 4>(ep, gs, red, rank, n0, b0, tile_n, smem_u32(consumed), inv_smem, ready, rp); break;
              default: break;  // the planner pairs a wide tile only with C = 4 (64-row runs spill)
            }
          } else {
            switch (C) {
              case 1:
                if constexpr (BN <= 64) reduce_and_store<BN, 1>(ep, gs, red, rank, n0, b0, tile_n, smem_u32(consumed), rt, inv_smem, ready, rp);
                break;
              case 2: reduce_and_store<BN, 2>(ep, gs, red, rank, n0, b0, tile_n, smem_u32(consumed), rt, inv_smem, ready, rp); break;
              case 4: reduce_and_store<BN, 4>(ep, gs, red, rank, n0, b0, tile_n, smem_u32(consumed), rt, inv_smem, ready, rp); break;
              case 8:
                if constexpr (BN >= 32) reduce_and_store<BN, 8>(ep, gs, red, rank, n0, b0, tile_n, smem_u32(consumed), rt, inv_smem, ready, rp);
                break;
            }
          }
        } else {
          mbar_wait_cluster(ready, rp);
        }
        if (tr) trace[12] = globaltimer();
        if (skip) {
          epi_bar();
          if (threadIdx.x == 64)
            for (int p = 0; p < C; ++p) mbar_arrive_cluster_relaxed(mapa_shared(smem_u32(consumed), p));
        }
        if (tr && ep.tp_n <= 1) trace[13] = globaltimer();
      }
    }
    if (my_tiles > 0) mbar_wait_cluster(consumed, (my_tiles - 1) & 1);  // peers done with my smem
    if (trace && threadIdx.x == 64) trace[14] = globaltimer();
  }
  if (trace && threadIdx.x == 64) trace[5] = globaltimer();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_free<L::kTmemCols>(tmem_base);
  if (trace && threadIdx.x == 0) trace[6] = globaltimer();
}

}  // namespace gh
