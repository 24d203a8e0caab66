// attention_gqa.cuh — Tier-2 decode attention F2 for grouped-query attention, sm_100a.
//
// With G = H / H_kv query heads per KV head (70B: G = 8) the per-query-head kernel of
// attention.cuh streams every KV block G times.  Here one work unit = (prompt b, KV head g): the
// K/V tiles of the unit are streamed ONCE and all G query heads are scored against each tile, so
// the kernel moves the algorithmic bytes of SURVEY.md §8d instead of G times them.
//
// Same pipeline as attention.cuh (persistent CTA per SM, 1 TMA producer warp + 8 consumer warps,
// cp.async.bulk K/V stages of 64 positions, per-unit header carrying q of the G heads, the new
// k / v and the G residual slices, online softmax in the exp2 domain, fused KV append), with the
// consumers organised as NG = G / HPW head groups of 8 / NG warps: a warp keeps HPW (= 2) query heads in
// registers, reads each 16-byte K / V chunk from shared memory once and applies it to its HPW
// heads, and covers 64 / (8 / NG) positions of every stage.  The last warp to finish a unit merges
// the 8 partial states (per head: the 8 / NG warps of its group) and writes the G outputs.
#pragma once
#include "attention.cuh"
#include "common.cuh"
#include "params.hpp"

namespace gh {

template <typename T, int DH, int G>
struct GqaCfg {
  static constexpr int HPW = 2;                        // query heads per warp (register budget)
  static constexpr int NG = G / HPW;                   // head groups
  static constexpr int WG = 8 / NG;                    // warps per head group
  static constexpr int kVec = 16 / sizeof(T);
  static constexpr int kChunks = DH / kVec;
  static constexpr int kLpp = (kChunks % 8 == 0) ? 8 : (kChunks % 4 == 0) ? 4 : (kChunks % 2 == 0) ? 2 : 1;
  static constexpr int kCpl = kChunks / kLpp;
  static constexpr int kPg = 32 / kLpp;                // positions per warp pass
  static constexpr int kW = 8;                         // consumer warps
  static constexpr int kTpos = (kW * kPg > 64) ? kW * kPg : 64;  // positions per stage
  static constexpr int kPasses = kTpos / (WG * kPg);  // position passes of a warp per stage
  static constexpr int kTileBytes = kTpos * DH * (int)sizeof(T);
  // header: q of G heads | new k | new v | x slices of G heads | {L, b, g, slot}
  static constexpr int kHdrBytes = (2 * G + 2) * DH * (int)sizeof(T) + 16;
  static constexpr int kStageBytes = ((2 * kTileBytes + kHdrBytes + 127) / 128) * 128;
  static constexpr int kNB = 2;                        // combine buffers (units in flight)
  static constexpr int kCombPerUnit = kW * HPW * (DH + 2);  // floats
  static constexpr int kStages = ((227 * 1024 - 2048 - kNB * kCombPerUnit * 4) / kStageBytes) > 5
                                     ? 5 : ((227 * 1024 - 2048 - kNB * kCombPerUnit * 4) / kStageBytes);
  static constexpr int kThreads = 32 * (1 + kW);
  static constexpr int kEl = kCpl * kVec;
  static constexpr int kCombOffset = kStages * kStageBytes;
  static constexpr int kCombBytes = kNB * kCombPerUnit * 4;
  static constexpr int kCtlOffset = kCombOffset + ((kCombBytes + 127) / 128) * 128;
  static constexpr int kBarOffset = kCtlOffset + 128;
  static constexpr int kSmem = kBarOffset + 2 * kStages * 8 + 16;
  static_assert(kStages >= 2, "GQA attention stages");
  static_assert(G % HPW == 0 && NG <= kW && kW % NG == 0 && kPasses >= 1, "GQA group shape");
};

// (9 warps per CTA: a sub-partition holds 3 warps' registers, i.e. at most 168 per thread, which
// is why a warp keeps HPW = 2 query heads)
template <typename T, int DH, int G>
__global__ void __launch_bounds__(GqaCfg<T, DH, G>::kThreads, 1)
    attn_gqa_kernel(const AttnArgs a) {
  using C = GqaCfg<T, DH, G>;
  constexpr int HPW = C::HPW, WG = C::WG;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = (uint64_t*)(smem + C::kBarOffset);
  uint64_t* empty = full + C::kStages;
  float* comb = (float*)(smem + C::kCombOffset);
  int* comb_cnt = (int*)(smem + C::kCtlOffset);
  volatile int* comb_seq = comb_cnt + C::kNB;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_units = a.B * a.Hkv;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], C::kW); }
    for (int i = 0; i < C::kNB; ++i) { comb_cnt[i] = 0; comb_seq[i] = 0; }
    fence_barrier_init();
  }
  __syncthreads();
  griddep_launch_dependents();
  griddep_wait();

  const T* fwd = (const T*)a.msg_fwd;
  T* bwd = (T*)a.msg_bwd;
  T* arena = (T*)a.arena;
  const long ld_fwd = 2L * a.D + 2L * a.Dkv;
  const long ld_bwd = 2L * a.D;
  const uint32_t hdr_bytes = (uint32_t)((2 * G + 2) * DH * sizeof(T));

  if (warp == 0) {
    // ------------------------------------------------ producer
    if (elect_one()) {
      const uint64_t pol = policy_evict_first();
      uint32_t it = 0;
      int u = blockIdx.x;
      int L = 0, sl = 0;
      if (u < n_units) { L = a.pos[u / a.Hkv]; sl = (int)a.slot[u / a.Hkv]; }
      while (u < n_units) {
        const int b = u / a.Hkv, g = u % a.Hkv;
        const int un = next_unit(a, u);
        int Ln = 0, sln = 0;
        if (un < n_units) { Ln = a.pos[un / a.Hkv]; sln = (int)a.slot[un / a.Hkv]; }
        const int nch = L > 0 ? (L + C::kTpos - 1) / C::kTpos : 1;
        for (int c = 0; c < nch; ++c, ++it) {
          const int s = it % C::kStages;
          mbar_wait(&empty[s], ((it / C::kStages) & 1) ^ 1);
          const int np = max(0, min(C::kTpos, L - c * C::kTpos));
          const uint32_t bytes = (uint32_t)np * DH * sizeof(T);
          uint8_t* sk = smem + s * C::kStageBytes;
          uint8_t* hdr = sk + 2 * C::kTileBytes;
          if (c == 0) {
            int* meta = (int*)(hdr + (2 * G + 2) * DH * sizeof(T));
            meta[0] = L; meta[1] = b; meta[2] = g; meta[3] = sl;
          }
          mbar_arrive_expect_tx(&full[s], 2 * bytes + (c == 0 ? hdr_bytes : 0u));
          if (np > 0) load_kv_chunk<T, DH>(a, arena, sl, g, c * C::kTpos, np, sk, sk + C::kTileBytes, &full[s], pol);
          if (c == 0) {
            const T* row = fwd + (long)b * ld_fwd;
            const uint32_t gq = (uint32_t)(G * DH * sizeof(T));
            bulk_g2s(hdr, row + a.D + (long)g * G * DH, gq, &full[s], pol);                        // q of the group
            bulk_g2s(hdr + gq, row + 2L * a.D + (long)g * DH, DH * sizeof(T), &full[s], pol);      // new k
            bulk_g2s(hdr + gq + DH * sizeof(T), row + 2L * a.D + a.Dkv + (long)g * DH, DH * sizeof(T), &full[s],
                     pol);                                                                         // new v
            bulk_g2s(hdr + gq + 2 * DH * sizeof(T), row + (long)g * G * DH, gq, &full[s], pol);    // x slices
          }
        }
        u = un;
        L = Ln;
        sl = sln;
      }
      units_done(a);
      {  // end of this CTA's units: a header-only stage with L = -1
        const int s = it % C::kStages;
        mbar_wait(&empty[s], ((it / C::kStages) & 1) ^ 1);
        *(int*)(smem + s * C::kStageBytes + 2 * C::kTileBytes + hdr_bytes) = -1;
        mbar_arrive(&full[s]);
      }
      prefetch_l2_share(a.pf, a.pf_bytes, blockIdx.x, gridDim.x);
    }
    return;
  }

  // -------------------------------------------------- consumers
  const int cw = warp - 1;
  const int ng = cw / WG;             // my head group: query heads ng*HPW .. +HPW of the unit
  const int wi = cw % WG;             // my index inside the group
  const int grp = lane / C::kLpp;
  const int sub = lane % C::kLpp;
  uint32_t it = 0;

  for (int ui = 0;; ++ui) {
    const int s0 = it % C::kStages;
    mbar_wait(&full[s0], (it / C::kStages) & 1);
    const uint8_t* hdr = smem + s0 * C::kStageBytes + 2 * C::kTileBytes;
    const T* hq = (const T*)hdr;                  // [G][DH]
    const T* hk = hq + G * DH;
    const T* hv = hk + DH;
    const T* hx = hv + DH;                        // [G][DH]
    const int* meta = (const int*)(hdr + (2 * G + 2) * DH * sizeof(T));
    const int L = meta[0];
    if (L < 0) return;  // end of the CTA's units
    const int b = meta[1], g = meta[2], slot = meta[3];
    const int nch = L > 0 ? (L + C::kTpos - 1) / C::kTpos : 1;

    float q[HPW][C::kEl], o[HPW][C::kEl], m[HPW], l[HPW];
#pragma unroll
    for (int hh = 0; hh < HPW; ++hh) {
#pragma unroll
      for (int j = 0; j < C::kCpl; ++j) {
        uint4 c = *(const uint4*)(hq + (ng * HPW + hh) * DH + (sub + j * C::kLpp) * C::kVec);
        chunk_to_f32<T>(c, q[hh] + j * C::kVec);
      }
#pragma unroll
      for (int e = 0; e < C::kEl; ++e) { q[hh][e] *= a.scale_log2; o[hh][e] = 0.f; }
      m[hh] = -INFINITY;
      l[hh] = 0.f;
    }

    if (wi == 0) {
      // new token: scores of my heads with the new key (group 0 lanes keep the mass); the first
      // warp also appends k / v to the arena
      T* kdst = arena + kv_offset(a, slot, g, L, DH);
      T* vdst = kdst + a.kv_stride;
      float vf[C::kEl], kf[C::kEl];
#pragma unroll
      for (int j = 0; j < C::kCpl; ++j) {
        const int off = (sub + j * C::kLpp) * C::kVec;
        uint4 kc = *(const uint4*)(hk + off);
        uint4 vc = *(const uint4*)(hv + off);
        if (cw == 0 && grp == 0) {
          *(uint4*)(kdst + off) = kc;
          *(uint4*)(vdst + off) = vc;
        }
        chunk_to_f32<T>(kc, kf + j * C::kVec);
        chunk_to_f32<T>(vc, vf + j * C::kVec);
      }
#pragma unroll
      for (int hh = 0; hh < HPW; ++hh) {
        float part = 0.f;
#pragma unroll
        for (int e = 0; e < C::kEl; ++e) part = fmaf(q[hh][e], kf[e], part);
#pragma unroll
        for (int o2 = C::kLpp / 2; o2 > 0; o2 >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o2);
        m[hh] = part;
        if (grp == 0) {
          l[hh] = 1.f;
#pragma unroll
          for (int e = 0; e < C::kEl; ++e) o[hh][e] = vf[e];
        }
      }
    }

    if (cw == C::kW - 1) {
      // residual pass-through of the unit's G slices: bwd.x[(g*G + i)*DH ..] = fwd.x[...]
      const int n16 = G * C::kChunks;
      for (int i = lane; i < n16; i += 32)
        *((uint4*)(bwd + (long)b * ld_bwd + (long)g * G * DH) + i) = ((const uint4*)hx)[i];
    }

    for (int c = 0; c < nch; ++c, ++it) {
      const int s = it % C::kStages;
      const int np = max(0, min(C::kTpos, L - c * C::kTpos));
      if (c > 0) mbar_wait(&full[s], (it / C::kStages) & 1);
      const T* sk = (const T*)(smem + s * C::kStageBytes);
      const T* sv = (const T*)(smem + s * C::kStageBytes + C::kTileBytes);

      float sc[C::kPasses][HPW];
      float mx[HPW];
#pragma unroll
      for (int hh = 0; hh < HPW; ++hh) mx[hh] = -INFINITY;
#pragma unroll
      for (int ps = 0; ps < C::kPasses; ++ps) {
        const int r = ps * WG * C::kPg + wi * C::kPg + grp;
        float kf[C::kEl];
        if (r < np) {
#pragma unroll
          for (int j = 0; j < C::kCpl; ++j) {
            uint4 kc = *(const uint4*)(sk + r * DH + (sub + j * C::kLpp) * C::kVec);
            chunk_to_f32<T>(kc, kf + j * C::kVec);
          }
        }
#pragma unroll
        for (int hh = 0; hh < HPW; ++hh) {
          float part = 0.f;
          if (r < np) {
            float pp[2] = {0.f, 0.f};
#pragma unroll
            for (int e = 0; e < C::kEl; ++e) pp[e & 1] = fmaf(q[hh][e], kf[e], pp[e & 1]);
            part = pp[0] + pp[1];
          }
#pragma unroll
          for (int o2 = C::kLpp / 2; o2 > 0; o2 >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o2);
          sc[ps][hh] = (r < np) ? part : -INFINITY;
          mx[hh] = fmaxf(mx[hh], sc[ps][hh]);
        }
      }
      float mn[HPW];
#pragma unroll
      for (int hh = 0; hh < HPW; ++hh) {
#pragma unroll
        for (int o2 = C::kLpp; o2 < 32; o2 <<= 1) mx[hh] = fmaxf(mx[hh], __shfl_xor_sync(0xffffffffu, mx[hh], o2));
        mn[hh] = fmaxf(m[hh], mx[hh]);
        if (mx[hh] != -INFINITY) {
          const float corr = (m[hh] == -INFINITY) ? 0.f : exp2f(m[hh] - mn[hh]);
          l[hh] *= corr;
#pragma unroll
          for (int e = 0; e < C::kEl; ++e) o[hh][e] *= corr;
          m[hh] = mn[hh];
        }
      }
#pragma unroll
      for (int ps = 0; ps < C::kPasses; ++ps) {
        const int r = ps * WG * C::kPg + wi * C::kPg + grp;
        if (r < np) {
          float vf[C::kEl];
#pragma unroll
          for (int j = 0; j < C::kCpl; ++j) {
            uint4 vc = *(const uint4*)(sv + r * DH + (sub + j * C::kLpp) * C::kVec);
            chunk_to_f32<T>(vc, vf + j * C::kVec);
          }
#pragma unroll
          for (int hh = 0; hh < HPW; ++hh) {
            const float p = exp2f(sc[ps][hh] - m[hh]);
            l[hh] += p;
#pragma unroll
            for (int e = 0; e < C::kEl; ++e) o[hh][e] = fmaf(p, vf[e], o[hh][e]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }

    // merge the lane groups of this warp (m is warp-uniform per head)
#pragma unroll
    for (int hh = 0; hh < HPW; ++hh)
#pragma unroll
      for (int o2 = C::kLpp; o2 < 32; o2 <<= 1) {
        l[hh] += __shfl_xor_sync(0xffffffffu, l[hh], o2);
#pragma unroll
        for (int e = 0; e < C::kEl; ++e) o[hh][e] += __shfl_xor_sync(0xffffffffu, o[hh][e], o2);
      }
    // publish [warp][head][DH + 2] into combine buffer ui % kNB; the last warp merges
    const int cbi = ui % C::kNB;
    while (comb_seq[cbi] != ui / C::kNB) { }
    float* cbuf = comb + cbi * C::kCombPerUnit;
#pragma unroll
    for (int hh = 0; hh < HPW; ++hh) {
      float* cwbuf = cbuf + (cw * HPW + hh) * (DH + 2);
      if (grp == 0) {
#pragma unroll
        for (int j = 0; j < C::kCpl; ++j)
#pragma unroll
          for (int e = 0; e < C::kVec; ++e) cwbuf[(sub + j * C::kLpp) * C::kVec + e] = o[hh][j * C::kVec + e];
      }
      if (lane == 0) { cwbuf[DH] = m[hh]; cwbuf[DH + 1] = l[hh]; }
    }
    __syncwarp();
    int last = 0;
    if (lane == 0) {
      __threadfence_block();
      last = atomicAdd(&comb_cnt[cbi], 1) == C::kW - 1;
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
      __threadfence_block();
      for (int hq = 0; hq < G; ++hq) {  // query head hq of the unit: head group hq / HPW, slot hq % HPW
        const int gg = hq / HPW, hh = hq % HPW;
        float M = -INFINITY;
#pragma unroll
        for (int k = 0; k < C::kW; ++k)
          if (k < WG) M = fmaxf(M, cbuf[((gg * WG + k) * HPW + hh) * (DH + 2) + DH]);
        float den = 0.f;
        float f[C::kW];
#pragma unroll
        for (int k = 0; k < C::kW; ++k) {
          f[k] = 0.f;
          if (k < WG) {
            const float mw = cbuf[((gg * WG + k) * HPW + hh) * (DH + 2) + DH];
            f[k] = (mw == -INFINITY) ? 0.f : exp2f(mw - M);
            den += cbuf[((gg * WG + k) * HPW + hh) * (DH + 2) + DH + 1] * f[k];
          }
        }
        const float inv = 1.f / den;
        T* orow = bwd + (long)b * ld_bwd + a.D + (long)(g * G + hq) * DH;
        for (int d = lane; d < DH; d += 32) {
          float acc = 0.f;
#pragma unroll
          for (int k = 0; k < C::kW; ++k)
            if (k < WG) acc += cbuf[((gg * WG + k) * HPW + hh) * (DH + 2) + d] * f[k];
          St<T>::store(orow, d, acc * inv);
        }
      }
      __syncwarp();
      if (lane == 0) {
        comb_cnt[cbi] = 0;
        __threadfence_block();
        comb_seq[cbi] = ui / C::kNB + 1;
      }
    }
  }
}

}  // namespace gh

namespace gh {

// ====================================================================== tensor-core GQA (bf16, d_h 128)
// The same unit (prompt, KV head) and pipeline, with the group's scores and P·V on the tensor
// cores (mma.sync m16n8k16 / m16n8k8, bf16 in, fp32 accumulate; the query heads are the M = 16
// rows, zero-padded above G).  K and V tiles arrive through TMA with the 128-byte swizzle (a 3-D
// tensor map over the whole KV arena: [rows = (layer, slot, K/V, kv head)][position][d_h], boxes of
// 64 positions x 64 d_h) so that the ldmatrix fragment loads are bank-conflict free.  Consumer warp
// w owns positions 8w..8w+7 of every 64-position stage: S (16 x 8) = Q (16 x 128) · K_wᵀ as 8
// MMAs, an online softmax per query head over its quad of lanes, O (16 x 128) += P (16 x 8) · V_w
// as 16 MMAs.  The 8 warps' states and the new token's (computed on CUDA cores by warp 0) are
// merged by a dedicated merge warp, so no consumer falls behind the stage ring.
GH_DEV void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
GH_DEV void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
GH_DEV void mma_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
GH_DEV void mma_1688(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t b0) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5}, {%6}, {%0, %1, %2, %3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a0), "r"(a1), "r"(b0));
}
GH_DEV void tma_load_3d(void* smem_dst, const void* tmap, int c0, int c1, int c2, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;\n" ::"r"(smem_u32(smem_dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

template <int G>
struct GqaTcCfg {
  static constexpr int DH = 128;
  static constexpr int kW = 8;                     // consumer warps, 8 positions each
  static constexpr int kTpos = 64;
  static constexpr int kBox = 64 * 64 * 2;         // one TMA box: 64 positions x 64 d_h (8 KB)
  static constexpr int kKV = 4 * kBox;             // K (2 boxes) + V (2 boxes)
  static constexpr int kHdrBytes = (2 * G + 2) * DH * 2 + 16;
  static constexpr int kStageBytes = kKV + ((kHdrBytes + 1023) / 1024) * 1024;  // boxes stay 1 KB aligned
  static constexpr int kNB = 2;
  // G >= 4: the consumer warps merge the unit themselves, warp h combining query head h, after a
  // named barrier -- one merge warp combining G heads serially was the bottleneck at short
  // contexts (70B, ctx 512: 4.1 TB/s); G < 4 keeps the dedicated merge warp
  static constexpr bool kSplitMerge = G >= 4;
  static constexpr int kCombPerUnit = (kW + 1) * G * (DH + 2);  // + the new token's state
  static constexpr int kCombBytes = kNB * kCombPerUnit * 4;
  static constexpr int kStages = ((227 * 1024 - 2048 - kCombBytes - 1024) / kStageBytes) > 6
                                     ? 6 : ((227 * 1024 - 2048 - kCombBytes - 1024) / kStageBytes);
  static constexpr int kThreads = 32 * (2 + kW);   // producer, kW consumers, merge warp
  static constexpr int kCombOffset = kStages * kStageBytes;
  static constexpr int kCtlOffset = kCombOffset + ((kCombBytes + 127) / 128) * 128;
  static constexpr int kBarOffset = kCtlOffset + 128;
  static constexpr int kSmem = kBarOffset + 2 * kStages * 8 + 16 + 1024;  // + alignment slack
  static_assert(G >= 1 && G <= 8 && kStages >= 2, "tensor-core GQA shape");
};

template <int G>
__global__ void __launch_bounds__(GqaTcCfg<G>::kThreads, 1)
    attn_gqa_tc_kernel(const __grid_constant__ CUtensorMap tmKV, const AttnArgs a) {
  using C = GqaTcCfg<G>;
  constexpr int DH = C::DH;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + C::kBarOffset);
  uint64_t* empty = full + C::kStages;
  float* comb = (float*)(smem + C::kCombOffset);
  int* comb_cnt = (int*)(smem + C::kCtlOffset);
  volatile int* comb_seq = comb_cnt + C::kNB;
  volatile int* comb_bg = comb_cnt + 2 * C::kNB;  // [kNB][2] (prompt, KV head) of the unit in the buffer

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_units = a.B * a.Hkv;

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmKV);
    for (int s = 0; s < C::kStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], C::kW); }
    for (int i = 0; i < C::kNB; ++i) { comb_cnt[i] = 0; comb_seq[i] = 0; }
    fence_barrier_init();
  }
  __syncthreads();
  griddep_launch_dependents();
  // the producer may request its first unit's cached K / V before griddepcontrol.wait
  // (a.kv_early, see attention.cuh); every other warp waits here
  if (warp != 0) griddep_wait();

  const bf16_t* fwd = (const bf16_t*)a.msg_fwd;
  bf16_t* bwd = (bf16_t*)a.msg_bwd;
  bf16_t* arena = (bf16_t*)a.arena;
  // message rows: tp head blocks (AttnArgs::tp); tp = 1 is the plain PayloadModel row
  const int tp = a.tp > 1 ? a.tp : 1;
  const int gpb = a.Hkv / tp;                 // KV heads per block
  const long wf = (2L * a.D + 2L * a.Dkv) / tp, wb = 2L * a.D / tp;
  const long Dt = a.D / tp, Dkvt = a.Dkv / tp;
  auto frow = [&](int b, int g) { return fwd + ((long)(g / gpb) * a.B + b) * wf; };
  auto brow = [&](int b, int g) { return bwd + ((long)(g / gpb) * a.B + b) * wb; };
  constexpr uint32_t hdr_bytes = (uint32_t)((2 * G + 2) * DH * 2);

  if (warp == 0) {
    // ------------------------------------------------ producer
    if (elect_one()) {
      const uint64_t pol = policy_evict_first();
      uint32_t it = 0;
      int u = blockIdx.x;
      int L = 0, sl = 0;
      // positions / slots are read before griddepcontrol.wait only by kv_early callers, which
      // promise that the preceding kernel writes neither them nor the arena
      if (a.kv_early && u < n_units) { L = a.pos[u / a.Hkv]; sl = (int)a.slot[u / a.Hkv]; }
      int pre = 0;  // stages of the first unit whose K / V were requested before the wait
      if (a.kv_early && u < n_units && L > 0) {
        const int g = u % a.Hkv;
        const int* pt = a.page_table ? a.page_table + (long)sl * a.max_pages : nullptr;
        pre = min((L + C::kTpos - 1) / C::kTpos, C::kStages);
        for (int c = 0; c < pre; ++c) {
          uint8_t* st = smem + c * C::kStageBytes;
          if (c == 0) mbar_expect_tx(&full[0], (uint32_t)C::kKV);
          else mbar_arrive_expect_tx(&full[c], (uint32_t)C::kKV);
          const int blk = pt ? pt[c] : sl, p0 = pt ? 0 : c * C::kTpos;
          const int row_k = ((a.layer_local * a.n_slots + blk) * 2 + 0) * a.Hkv + g;
          const int row_v = row_k + a.Hkv;
          tma_load_3d(st, &tmKV, 0, p0, row_k, &full[c], pol);
          tma_load_3d(st + C::kBox, &tmKV, 64, p0, row_k, &full[c], pol);
          tma_load_3d(st + 2 * C::kBox, &tmKV, 0, p0, row_v, &full[c], pol);
          tma_load_3d(st + 3 * C::kBox, &tmKV, 64, p0, row_v, &full[c], pol);
        }
      }
      griddep_wait();
      if (!a.kv_early && u < n_units) { L = a.pos[u / a.Hkv]; sl = (int)a.slot[u / a.Hkv]; }
      while (u < n_units) {
        const int b = u / a.Hkv, g = u % a.Hkv;
        // tensor-map rows (layer, slot or page, K/V, kv head); paged: one page per stage
        const int* pt = a.page_table ? a.page_table + (long)sl * a.max_pages : nullptr;
        const int nch = L > 0 ? (L + C::kTpos - 1) / C::kTpos : 1;
        for (int c = 0; c < nch; ++c, ++it) {
          const int s = it % C::kStages;
          const bool issued = (int)it < pre;
          if (issued && c > 0) continue;
          mbar_wait(&empty[s], ((it / C::kStages) & 1) ^ 1);
          uint8_t* st = smem + s * C::kStageBytes;
          uint8_t* hdr = st + C::kKV;
          if (c == 0) {
            int* meta = (int*)(hdr + hdr_bytes);
            meta[0] = L; meta[1] = b; meta[2] = g; meta[3] = sl;
          }
          const bool any = L > 0 && !issued;
          mbar_arrive_expect_tx(&full[s], (any ? (uint32_t)C::kKV : 0u) + (c == 0 ? hdr_bytes : 0u));
          if (any) {  // full 64-position boxes (rows past L are masked by the consumers)
            const int blk = pt ? pt[c] : sl, p0 = pt ? 0 : c * C::kTpos;
            const int row_k = ((a.layer_local * a.n_slots + blk) * 2 + 0) * a.Hkv + g;
            const int row_v = row_k + a.Hkv;
            tma_load_3d(st, &tmKV, 0, p0, row_k, &full[s], pol);
            tma_load_3d(st + C::kBox, &tmKV, 64, p0, row_k, &full[s], pol);
            tma_load_3d(st + 2 * C::kBox, &tmKV, 0, p0, row_v, &full[s], pol);
            tma_load_3d(st + 3 * C::kBox, &tmKV, 64, p0, row_v, &full[s], pol);
          }
          if (c == 0) {
            const bf16_t* row = frow(b, g);
            const long gl = g % gpb;
            constexpr uint32_t gq = (uint32_t)(G * DH * 2);
            bulk_g2s(hdr, row + Dt + gl * G * DH, gq, &full[s], pol);                     // q of the group
            bulk_g2s(hdr + gq, row + 2 * Dt + gl * DH, DH * 2, &full[s], pol);            // new k
            bulk_g2s(hdr + gq + DH * 2, row + 2 * Dt + Dkvt + gl * DH, DH * 2, &full[s], pol);  // new v
            bulk_g2s(hdr + gq + 2 * DH * 2, row + gl * G * DH, gq, &full[s], pol);        // x slices
          }
        }
        // the next unit is fetched only now, once this unit's stages are all requested: the
        // work-counter atomic and the dependent position / slot loads (~2 round trips) then
        // overlap the consumers draining the ring instead of delaying this unit's first loads
        const int un = next_unit(a, u);
        u = un;
        L = 0;
        sl = 0;
        if (un < n_units) { L = a.pos[un / a.Hkv]; sl = (int)a.slot[un / a.Hkv]; }
      }
      units_done(a);
      {  // end of this CTA's units: a header-only stage with L = -1
        const int s = it % C::kStages;
        mbar_wait(&empty[s], ((it / C::kStages) & 1) ^ 1);
        *(int*)(smem + s * C::kStageBytes + C::kKV + hdr_bytes) = -1;
        mbar_arrive(&full[s]);
      }
      prefetch_l2_share(a.pf, a.pf_bytes, blockIdx.x, gridDim.x);
    }
    return;
  }

  if (warp == C::kW + 1) {
    // -------------------------------------------------- merge warp (unit order): combines the kW
    // consumer states and the new token's state of every query head, writes the G output rows
    if constexpr (C::kSplitMerge) return;  // the consumers merge (see GqaTcCfg::kSplitMerge)
    for (int ui = 0;; ++ui) {
      const int cb = ui % C::kNB;
      while (*(volatile int*)&comb_cnt[cb] < C::kW)
        if (!(a.flags & 8)) __nanosleep(32);  // idle most of the time: back off (8: diagnostics, spin)
      __threadfence_block();
      const float* cbuf = comb + cb * C::kCombPerUnit;
      const int b = comb_bg[2 * cb], g = comb_bg[2 * cb + 1];
      if (b < 0) return;  // the consumers saw the end of the CTA's units
      for (int hq = 0; hq < G; ++hq) {
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w <= C::kW; ++w) M = fmaxf(M, cbuf[(w * G + hq) * (DH + 2) + DH]);
        float f[C::kW + 1];
        float den = 0.f;
#pragma unroll
        for (int w = 0; w <= C::kW; ++w) {
          const float mw = cbuf[(w * G + hq) * (DH + 2) + DH];
          f[w] = (mw == -INFINITY) ? 0.f : exp2f(mw - M);
          den += cbuf[(w * G + hq) * (DH + 2) + DH + 1] * f[w];
        }
        const float inv = 1.f / den;
        bf16_t* orow = brow(b, g) + Dt + (long)((g % gpb) * G + hq) * DH;
        for (int d = lane; d < DH; d += 32) {
          float acc = 0.f;
#pragma unroll
          for (int w = 0; w <= C::kW; ++w) acc += cbuf[(w * G + hq) * (DH + 2) + d] * f[w];
          St<bf16_t>::store(orow, d, acc * inv);
        }
      }
      __syncwarp();
      if (lane == 0) {
        comb_cnt[cb] = 0;
        __threadfence_block();
        comb_seq[cb] = ui / C::kNB + 1;
      }
    }
    return;
  }

  // -------------------------------------------------- consumers
  const int cw = warp - 1;
  const int qr = lane >> 2;            // query head (MMA row) of this lane's accumulator entries
  const int qc = (lane & 3) * 2;       // first of its two columns
  uint32_t it = 0;
  for (int ui = 0;; ++ui) {
    const int s0 = it % C::kStages;
    mbar_wait(&full[s0], (it / C::kStages) & 1);
    const uint8_t* hdr = smem + s0 * C::kStageBytes + C::kKV;
    const bf16_t* hq = (const bf16_t*)hdr;
    const bf16_t* hk = hq + G * DH;
    const bf16_t* hv = hk + DH;
    const bf16_t* hx = hv + DH;
    const int* meta = (const int*)(hdr + hdr_bytes);
    const int L = meta[0];
    if (L < 0) {  // end of units: pass the end marker to the merge warp through the next buffer
      if constexpr (C::kSplitMerge) return;
      const int cb = ui % C::kNB;
      while (comb_seq[cb] != ui / C::kNB) { }
      if (cw == 0 && lane == 0) comb_bg[2 * cb] = -1;
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        atomicAdd(&comb_cnt[cb], 1);
      }
      return;
    }
    const int b = meta[1], g = meta[2], slot = meta[3];
    const int nch = L > 0 ? (L + C::kTpos - 1) / C::kTpos : 1;

    // Q fragments (A operand, rows = query heads; rows >= G and 8..15 are zero)
    uint32_t qa[8][2];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      qa[kk][0] = qr < G ? *(const uint32_t*)(hq + qr * DH + kk * 16 + qc) : 0u;
      qa[kk][1] = qr < G ? *(const uint32_t*)(hq + qr * DH + kk * 16 + 8 + qc) : 0u;
    }
    float o[16][4];
#pragma unroll
    for (int j = 0; j < 16; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
    float m = -INFINITY, l = 0.f;  // per query head qr (quad-uniform m; l is this lane's partial)

    const int cb = ui % C::kNB;
    float* cbuf = comb + cb * C::kCombPerUnit;
    // split merge: warp cw < G keeps the new token's score for query head cw and its value
    // (d = lane + 32 i) in registers -- the header's stage is released before the merge
    float nsc = 0.f, nv[DH / 32];
    if constexpr (C::kSplitMerge) {
      if (cw < G) {
        float part = 0.f;
#pragma unroll
        for (int i = 0; i < DH / 32; ++i) {
          const int d = lane + 32 * i;
          part = fmaf(bf16_to_f32(hq[cw * DH + d].bits), bf16_to_f32(hk[d].bits), part);
          nv[i] = bf16_to_f32(hv[d].bits);
        }
        nsc = warp_sum(part) * a.scale_log2;
      }
    }
    if (cw == 0) {
      // new token: its key / value from the header; append them to the arena; its state is merged
      // as a ninth partial (m = score, l = 1, o = v) by the last warp
      bf16_t* kdst = arena + kv_offset(a, slot, g, L, DH);
      bf16_t* vdst = kdst + a.kv_stride;
      if (lane < DH / 8) {
        *((uint4*)kdst + lane) = ((const uint4*)hk)[lane];
        *((uint4*)vdst + lane) = ((const uint4*)hv)[lane];
      }
    }
    if (cw == 0 && !C::kSplitMerge) {
      while (comb_seq[cb] != ui / C::kNB) { }
      for (int h = 0; h < G; ++h) {
        float part = 0.f;
        for (int d = lane; d < DH; d += 32) part = fmaf(bf16_to_f32(hq[h * DH + d].bits), bf16_to_f32(hk[d].bits), part);
        part = warp_sum(part) * a.scale_log2;
        float* nb = cbuf + (C::kW * G + h) * (DH + 2);
        for (int d = lane; d < DH; d += 32) nb[d] = bf16_to_f32(hv[d].bits);
        if (lane == 0) { nb[DH] = part; nb[DH + 1] = 1.f; }
      }
    }
    if (cw == C::kW - 1) {
      for (int i = lane; i < G * DH / 8; i += 32)
        *((uint4*)(brow(b, g) + (long)(g % gpb) * G * DH) + i) = ((const uint4*)hx)[i];
    }

    for (int c = 0; c < nch; ++c, ++it) {
      const int s = it % C::kStages;
      const int np = max(0, min(C::kTpos, L - c * C::kTpos));
      if (c > 0) mbar_wait(&full[s], (it / C::kStages) & 1);
      const uint32_t st = smem_u32(smem + s * C::kStageBytes);
      if (cw * 8 < np && !(a.flags & 1)) {  // (flags & 1: diagnostics, K / V streaming only)
        // ---- S = Q Kᵀ for positions 8cw..8cw+7 (B fragments by ldmatrix from the swizzled boxes)
        float sacc[4] = {0.f, 0.f, 0.f, 0.f};
        const int prow = cw * 8 + (lane & 7);          // position row this lane addresses
#pragma unroll
        for (int kk = 0; kk < 8; kk += 2) {
          const int chunk = kk * 2 + (lane >> 3);       // 16-byte d_h chunk 0..15 of block lane/8
          const uint32_t addr = st + (chunk >> 3) * C::kBox + prow * 128 + (((chunk & 7) ^ (prow & 7)) << 4);
          uint32_t b0, b1, b2, b3;
          ldsm_x4(addr, b0, b1, b2, b3);
          mma_16816(sacc, qa[kk][0], 0u, qa[kk][1], 0u, b0, b1);
          mma_16816(sacc, qa[kk + 1][0], 0u, qa[kk + 1][1], 0u, b2, b3);
        }
        // ---- online softmax per query head (row qr) over this warp's 8 positions
        const int p0 = cw * 8 + qc;
        float s0 = (p0 < np) ? sacc[0] * a.scale_log2 : -INFINITY;
        float s1 = (p0 + 1 < np) ? sacc[1] * a.scale_log2 : -INFINITY;
        float mx = fmaxf(s0, s1);
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        const float mn = fmaxf(m, mx);                  // mx is finite: position 8cw < np
        const float corr = (m == -INFINITY) ? 0.f : exp2f(m - mn);
        const float e0 = exp2f(s0 - mn), e1 = exp2f(s1 - mn);
        l = l * corr + e0 + e1;
        m = mn;
#pragma unroll
        for (int j = 0; j < 16; ++j) { o[j][0] *= corr; o[j][1] *= corr; o[j][2] *= corr; o[j][3] *= corr; }
        // P as the A operand: rows 0..7 = bf16(P); rows 8..15 (no query head lives there) = the
        // rounding residual bf16(P - bf16(P)).  Accumulator rows r and r + 8 of one lane then sum
        // to (bf16(P) + residual) V, i.e. P V with P exact to ~2^-17 relative at no extra MMA:
        // the fp32-compute rule of P:514, consistent with l, which sums the same unrounded P.
        const uint32_t pa = pack_bf16x2(e0, e1);
        const uint32_t pl = pack_bf16x2(e0 - __uint_as_float(pa << 16), e1 - __uint_as_float(pa & 0xffff0000u));
        // ---- O += P Vw (V fragments by ldmatrix.trans: 4 d_h tiles of 8 per instruction)
#pragma unroll
        for (int dg = 0; dg < 4; ++dg) {
          const int chunk = dg * 4 + (lane >> 3);       // d_h chunk (8 d_h) of tile lane/8
          const uint32_t addr =
              st + 2 * C::kBox + (chunk >> 3) * C::kBox + prow * 128 + (((chunk & 7) ^ (prow & 7)) << 4);
          uint32_t v0, v1, v2, v3;
          ldsm_x4_t(addr, v0, v1, v2, v3);
          mma_1688(o[dg * 4 + 0], pa, pl, v0);
          mma_1688(o[dg * 4 + 1], pa, pl, v1);
          mma_1688(o[dg * 4 + 2], pa, pl, v2);
          mma_1688(o[dg * 4 + 3], pa, pl, v3);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }

    // publish this warp's state [warp][head][DH + 2]; the last warp merges 8 + 1 states per head
    l += __shfl_xor_sync(0xffffffffu, l, 1);
    l += __shfl_xor_sync(0xffffffffu, l, 2);
    if (cw != 0 && !C::kSplitMerge) while (comb_seq[cb] != ui / C::kNB) { }
    if (qr < G) {
      float* wb = cbuf + (cw * G + qr) * (DH + 2);
#pragma unroll
      for (int j = 0; j < 16; ++j) { wb[j * 8 + qc] = o[j][0] + o[j][2]; wb[j * 8 + qc + 1] = o[j][1] + o[j][3]; }
      if ((lane & 3) == 0) { wb[DH] = m; wb[DH + 1] = l; }
    }
    if constexpr (C::kSplitMerge) {
      // every consumer warp's state of this unit is in the buffer; warp h merges query head h.
      // Buffer ui % 2 is written again only at unit ui + 2, after the barrier of unit ui + 1,
      // which every warp passes only once it has merged unit ui.
      asm volatile("bar.sync 3, %0;" ::"n"(C::kW * 32) : "memory");
      if (cw < G) {
        const float* hb = cbuf + cw * (DH + 2);  // warp w's state of head cw at hb + w * G * (DH + 2)
        float M = nsc;
#pragma unroll
        for (int w = 0; w < C::kW; ++w) M = fmaxf(M, hb[w * G * (DH + 2) + DH]);
        float f[C::kW];
        float den = 0.f;
#pragma unroll
        for (int w = 0; w < C::kW; ++w) {
          const float mw = hb[w * G * (DH + 2) + DH];
          f[w] = (mw == -INFINITY) ? 0.f : exp2f(mw - M);
          den += hb[w * G * (DH + 2) + DH + 1] * f[w];
        }
        const float fn = exp2f(nsc - M);  // the new token (l = 1) as the last partial
        den += fn;
        const float inv = 1.f / den;
        bf16_t* orow = brow(b, g) + Dt + (long)((g % gpb) * G + cw) * DH;
#pragma unroll
        for (int i = 0; i < DH / 32; ++i) {
          const int d = lane + 32 * i;
          float acc = 0.f;
#pragma unroll
          for (int w = 0; w < C::kW; ++w) acc += hb[w * G * (DH + 2) + d] * f[w];
          acc += nv[i] * fn;
          St<bf16_t>::store(orow, d, acc * inv);
        }
      }
      continue;
    }
    if (cw == 0 && lane == 0) { comb_bg[2 * cb] = b; comb_bg[2 * cb + 1] = g; }
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      atomicAdd(&comb_cnt[cb], 1);
    }
  }
}

}  // namespace gh
