// attention.cuh — Tier-2 batched decode attention F2 for sm_100a.
//
// One work unit = (prompt b, query head h).  The KV arena is head-major so that the cached
// keys (and values) of one (slot, kv head) are one contiguous [S_max, d_h] block:
//
//   arena[layer][slot][kv ∈ {K, V}][kv_head][position][d_h]         (storage dtype)
//
// A persistent CTA per SM walks its units; warp 0 is a TMA producer that streams K and V tiles
// of TPOS positions with 1-D bulk copies (cp.async.bulk, SASS UBLKCP) into a STAGES-deep
// shared-memory ring guarded by mbarriers; warps 1..W are consumers that compute scores with
// 16-byte shared loads and warp-shuffle reductions, run an online (running-max) softmax per
// warp, and accumulate P·V in fp32 registers.  The W partial states are merged through shared
// memory at the end of each unit.  The new token's key/value come straight from the Tier-1
// message (fwd [x|q|k|v]) and are appended to the arena by the same kernel (fused append), so
// there is no ordering hazard between the append and the bulk loads (which only cover cached
// positions 0..pos-1).  Output = bwd message [x|attn].
#pragma once
#include "common.cuh"
#include "params.hpp"

namespace gh {

// K and V of positions [q0, q0 + np) of (slot sl, kv head g) into sk / sv: one bulk copy each for
// contiguous slots, one per 64-position page segment for the paged arena.
template <typename T, int DH>
GH_DEV void load_kv_chunk(const AttnArgs& a, const T* arena, int sl, int g, int q0, int np, uint8_t* sk,
                          uint8_t* sv, uint64_t* bar, uint64_t pol) {
  for (int q = 0; q < np;) {
    const int p = q0 + q;
    const int n = a.page_table ? min(np - q, kKvPagePositions - p % kKvPagePositions) : np - q;
    const T* kb = arena + kv_offset(a, sl, g, p, DH);
    const uint32_t off = (uint32_t)q * DH * sizeof(T), bytes = (uint32_t)n * DH * sizeof(T);
    bulk_g2s(sk + off, kb, bytes, bar, pol);
    bulk_g2s(sv + off, kb + a.kv_stride, bytes, bar, pol);
    q += n;
  }
}

// Persistent unit schedule: a CTA's first unit is blockIdx.x; later ones come from the launch's
// work counter (ragged contexts balance across CTAs) or, without one, stride gridDim.x.
GH_DEV int next_unit(const AttnArgs& a, int u) {
  return a.work ? (int)atomicAdd(a.work, 1u) + (int)gridDim.x : u + (int)gridDim.x;
}
// Producer after its last fetch: the last CTA to get here resets the counter for the next launch
// (no CTA fetches any more once every producer has counted itself out).
GH_DEV void units_done(const AttnArgs& a) {
  if (a.work && atomicAdd(a.work + 1, 1u) == gridDim.x - 1) {
    atomicExch(a.work, 0u);
    atomicExch(a.work + 1, 0u);
  }
}

template <typename T, int DH, int W = 8>
struct AttnCfg {
  static constexpr int kVec = 16 / sizeof(T);          // elements per 16-byte chunk
  static constexpr int kChunks = DH / kVec;            // 16-byte chunks per row
  static constexpr int kLpp = (kChunks % 8 == 0) ? 8 : (kChunks % 4 == 0) ? 4 : (kChunks % 2 == 0) ? 2 : 1;
  static constexpr int kCpl = kChunks / kLpp;          // chunks per lane
  static constexpr int kPg = 32 / kLpp;                // positions per warp pass
  static constexpr int kW = W;                         // consumer warps
  static constexpr int kTpos = (kW * kPg > 64) ? kW * kPg : 64;  // positions per stage
  static constexpr int kPasses = kTpos / (kW * kPg);
  static constexpr int kTileBytes = kTpos * DH * (int)sizeof(T);
  // per-stage header (first stage of a unit): q, new k, new v and the unit's d_h-slice of the
  // residual x (bulk-copied from the fwd message) + {L, b, h, slot}
  static constexpr int kHdrBytes = 4 * DH * (int)sizeof(T) + 16;
  static constexpr int kStageBytes = ((2 * kTileBytes + kHdrBytes + 127) / 128) * 128;
  static constexpr int kStages = (196608 / kStageBytes) > 6 ? 6 : (196608 / kStageBytes);
  static constexpr int kThreads = 32 * (2 + kW);       // producer, kW consumers, merge warp
  static constexpr int kEl = kCpl * kVec;              // elements per lane
  static constexpr int kNB = 4;                        // combine buffers (units in flight)
  static constexpr int kCombOffset = kStages * kStageBytes;
  static constexpr int kCombBytes = kNB * kW * (DH + 2) * 4;
  static constexpr int kCtlOffset = kCombOffset + ((kCombBytes + 127) / 128) * 128;  // 2*kNB ints
  static constexpr int kBarOffset = kCtlOffset + 128;
  static constexpr int kSmem = kBarOffset + 2 * kStages * 8 + 16;
  static_assert(kChunks * kVec == DH, "d_head must be a multiple of 16 bytes");
};

// 16-byte chunk -> kVec floats
template <typename T> GH_DEV void chunk_to_f32(const uint4& c, float* f);
template <> GH_DEV void chunk_to_f32<float>(const uint4& c, float* f) {
  f[0] = __uint_as_float(c.x); f[1] = __uint_as_float(c.y);
  f[2] = __uint_as_float(c.z); f[3] = __uint_as_float(c.w);
}
template <> GH_DEV void chunk_to_f32<bf16_t>(const uint4& c, float* f) {
  const uint32_t w[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}

// out = f * g * s packed back into a 16-byte chunk of the storage type
template <typename T> GH_DEV void pack_f32(const float* f, const float* g, float s, uint4& o);
template <> GH_DEV void pack_f32<float>(const float* f, const float* g, float s, uint4& o) {
  o.x = __float_as_uint(f[0] * s * g[0]); o.y = __float_as_uint(f[1] * s * g[1]);
  o.z = __float_as_uint(f[2] * s * g[2]); o.w = __float_as_uint(f[3] * s * g[3]);
}
template <> GH_DEV void pack_f32<bf16_t>(const float* f, const float* g, float s, uint4& o) {
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    w[i] = (uint32_t)f32_to_bf16(f[2 * i] * s * g[2 * i]) |
           ((uint32_t)f32_to_bf16(f[2 * i + 1] * s * g[2 * i + 1]) << 16);
  o = make_uint4(w[0], w[1], w[2], w[3]);
}

template <typename T, int DH, int W>
__global__ void __launch_bounds__(AttnCfg<T, DH, W>::kThreads, 1)
    attn_decode_kernel(const AttnArgs a) {
  using C = AttnCfg<T, DH, W>;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = (uint64_t*)(smem + C::kBarOffset);
  uint64_t* empty = full + C::kStages;
  float* comb = (float*)(smem + C::kCombOffset);
  int* comb_cnt = (int*)(smem + C::kCtlOffset);       // [kNB] warps that published unit i
  volatile int* comb_seq = comb_cnt + C::kNB;          // [kNB] units combined from this buffer
  volatile int* comb_bh = comb_cnt + 2 * C::kNB;       // [kNB][2] (prompt, head) of the unit in the buffer

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_units = a.B * a.H;
  const int group = a.H / a.Hkv;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], C::kW); }
    for (int i = 0; i < C::kNB; ++i) { comb_cnt[i] = 0; comb_seq[i] = 0; }
    fence_barrier_init();
  }
  __syncthreads();
  griddep_launch_dependents();
  // griddepcontrol.wait (the fwd message, and the arena when a.kv_early == 0, are visible after
  // it) is taken per role below: the producer may stream the first unit's cached keys first

  const T* fwd = (const T*)a.msg_fwd;
  T* bwd = (T*)a.msg_bwd;
  T* arena = (T*)a.arena;
  const long ld_fwd = 2L * a.D + 2L * a.Dkv;
  const long ld_bwd = 2L * a.D;

  if (warp == 0) {
    // ------------------------------------------------ producer
    if (elect_one()) {
      const uint64_t pol = policy_evict_first();
      uint32_t it = 0;
      int u = blockIdx.x;
      int L = 0, sl = 0;
      // positions / slots are read before griddepcontrol.wait only by kv_early callers (whose
      // predecessor writes neither them nor the arena)
      if (a.kv_early && u < n_units) { L = a.pos[u / a.H]; sl = (int)a.slot[u / a.H]; }
      // early start: the first unit's cached K / V (independent of the predecessor) fill the
      // free stages before griddepcontrol.wait; stage 0's arrive (with the header) comes after it
      int pre = 0;
      if (a.kv_early && u < n_units) {
        const int kvh = (u % a.H) / group;
        pre = min(L > 0 ? (L + C::kTpos - 1) / C::kTpos : 1, C::kStages);
        for (int c = 0; c < pre; ++c) {
          const int np = max(0, min(C::kTpos, L - c * C::kTpos));
          const uint32_t bytes = (uint32_t)np * DH * sizeof(T);
          uint8_t* sk = smem + c * C::kStageBytes;
          if (c == 0) mbar_expect_tx(&full[0], 2 * bytes);
          else mbar_arrive_expect_tx(&full[c], 2 * bytes);
          if (np > 0) load_kv_chunk<T, DH>(a, arena, sl, kvh, c * C::kTpos, np, sk, sk + C::kTileBytes, &full[c], pol);
        }
      }
      griddep_wait();
      if (!a.kv_early && u < n_units) { L = a.pos[u / a.H]; sl = (int)a.slot[u / a.H]; }
      while (u < n_units) {
        const int b = u / a.H, h = u % a.H, kvh = h / group;
        // next unit's position / slot, one unit ahead (hides the dependent global loads)
        const int un = next_unit(a, u);
        int Ln = 0, sln = 0;
        if (un < n_units) { Ln = a.pos[un / a.H]; sln = (int)a.slot[un / a.H]; }
        const int nch = L > 0 ? (L + C::kTpos - 1) / C::kTpos : 1;
        for (int c = 0; c < nch; ++c, ++it) {
          const int s = it % C::kStages;
          const bool issued = (int)it < pre;  // K / V already requested before the wait
          if (issued && c > 0) continue;
          mbar_wait(&empty[s], ((it / C::kStages) & 1) ^ 1);
          const int np = max(0, min(C::kTpos, L - c * C::kTpos));
          const uint32_t bytes = issued ? 0u : (uint32_t)np * DH * sizeof(T);
          uint8_t* sk = smem + s * C::kStageBytes;
          uint8_t* hdr = sk + 2 * C::kTileBytes;
          if (c == 0) {  // unit header: metadata (plain store, released by the arrive) + q/k/v/x copies
            int* meta = (int*)(hdr + 4 * DH * sizeof(T));
            meta[0] = L; meta[1] = b; meta[2] = h; meta[3] = sl;
          }
          mbar_arrive_expect_tx(&full[s], 2 * bytes + (c == 0 ? 4 * DH * (uint32_t)sizeof(T) : 0u));
          if (np > 0 && !issued)
            load_kv_chunk<T, DH>(a, arena, sl, kvh, c * C::kTpos, np, sk, sk + C::kTileBytes, &full[s], pol);
          if (c == 0) {
            const T* row = fwd + (long)b * ld_fwd;
            bulk_g2s(hdr, row + a.D + (long)h * DH, DH * sizeof(T), &full[s], pol);
            bulk_g2s(hdr + DH * sizeof(T), row + 2L * a.D + (long)kvh * DH, DH * sizeof(T), &full[s], pol);
            bulk_g2s(hdr + 2 * DH * sizeof(T), row + 2L * a.D + a.Dkv + (long)kvh * DH, DH * sizeof(T), &full[s], pol);
            bulk_g2s(hdr + 3 * DH * sizeof(T), row + (long)h * DH, DH * sizeof(T), &full[s], pol);
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
        *(int*)(smem + s * C::kStageBytes + 2 * C::kTileBytes + 4 * DH * sizeof(T)) = -1;
        mbar_arrive(&full[s]);
      }
      prefetch_l2_share(a.pf, a.pf_bytes, blockIdx.x, gridDim.x);
    }
    return;
  }

  if (warp == C::kW + 1) {
    // -------------------------------------------------- merge warp: combines the kW published
    // partial states of each unit (in unit order) and writes the output row, so that no consumer
    // warp falls behind the stage ring while merging
    if (a.flags & 3) return;
    griddep_wait();
    for (int ui = 0;; ++ui) {
      const int cb = ui % C::kNB;
      while (*(volatile int*)&comb_cnt[cb] < C::kW)
        if (!(a.flags & 8)) __nanosleep(32);  // idle most of the time: back off (8: diagnostics, spin)
      __threadfence_block();
      const float* cbuf = comb + cb * C::kW * (DH + 2);
      const int b = comb_bh[2 * cb], h = comb_bh[2 * cb + 1];
      if (b < 0) return;  // the consumers saw the end of the CTA's units
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < C::kW; ++w) M = fmaxf(M, cbuf[w * (DH + 2) + DH]);
      float den = 0.f;
      float f[C::kW];
#pragma unroll
      for (int w = 0; w < C::kW; ++w) {
        const float mw = cbuf[w * (DH + 2) + DH];
        f[w] = (mw == -INFINITY) ? 0.f : exp2f(mw - M);
        den += cbuf[w * (DH + 2) + DH + 1] * f[w];
      }
      const float inv = 1.f / den;
      T* orow = bwd + (long)b * ld_bwd + a.D + (long)h * DH;
      for (int d = lane; d < DH; d += 32) {
        float acc = 0.f;
#pragma unroll
        for (int w = 0; w < C::kW; ++w) acc += cbuf[w * (DH + 2) + d] * f[w];
        St<T>::store(orow, d, acc * inv);
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
  griddep_wait();  // they write the arena and the bwd message
  const int cw = warp - 1;
  const int grp = lane / C::kLpp;
  const int sub = lane % C::kLpp;
  uint32_t it = 0;

  for (int ui = 0;; ++ui) {
    // unit header (first stage of the unit)
    const int s0 = it % C::kStages;
    mbar_wait(&full[s0], (it / C::kStages) & 1);
    const uint8_t* hdr = smem + s0 * C::kStageBytes + 2 * C::kTileBytes;
    const T* hq = (const T*)hdr;
    const T* hk = hq + DH;
    const T* hv = hk + DH;
    const int* meta = (const int*)(hdr + 4 * DH * sizeof(T));
    const int L = meta[0];
    if (L < 0) {  // end of units: pass the end marker to the merge warp through the next buffer
      if (!(a.flags & 3)) {
        const int cb = ui % C::kNB;
        while (comb_seq[cb] != ui / C::kNB) { }
        if (cw == 0 && lane == 0) comb_bh[2 * cb] = -1;
        __syncwarp();
        if (lane == 0) {
          __threadfence_block();
          atomicAdd(&comb_cnt[cb], 1);
        }
      }
      return;
    }
    const int b = meta[1], h = meta[2], kvh = h / group, slot = meta[3];
    const int nch = L > 0 ? (L + C::kTpos - 1) / C::kTpos : 1;

    float q[C::kEl], o[C::kEl];
#pragma unroll
    for (int j = 0; j < C::kCpl; ++j) {
      uint4 c = *(const uint4*)(hq + (sub + j * C::kLpp) * C::kVec);
      chunk_to_f32<T>(c, q + j * C::kVec);
    }
#pragma unroll
    for (int e = 0; e < C::kEl; ++e) { q[e] *= a.scale_log2; o[e] = 0.f; }
    float m = -INFINITY;  // warp-uniform running max (log2 domain)
    float l = 0.f;        // per-group partial sum

    if (cw == 0) {
      // new token: score from the header, append k/v to the arena (group 0 lanes)
      T* kdst = arena + kv_offset(a, slot, kvh, L, DH);
      T* vdst = kdst + a.kv_stride;
      float part = 0.f;
      float vf[C::kEl];
#pragma unroll
      for (int j = 0; j < C::kCpl; ++j) {
        const int off = (sub + j * C::kLpp) * C::kVec;
        uint4 kc = *(const uint4*)(hk + off);
        uint4 vc = *(const uint4*)(hv + off);
        if (grp == 0 && (h % group) == 0) {  // one writer per kv head
          *(uint4*)(kdst + off) = kc;
          *(uint4*)(vdst + off) = vc;
        }
        float kf[C::kVec];
        chunk_to_f32<T>(kc, kf);
        chunk_to_f32<T>(vc, vf + j * C::kVec);
#pragma unroll
        for (int e = 0; e < C::kVec; ++e) part = fmaf(q[j * C::kVec + e], kf[e], part);
      }
#pragma unroll
      for (int o2 = C::kLpp / 2; o2 > 0; o2 >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o2);
      m = part;  // identical in every group; only group 0 keeps mass
      if (grp == 0) {
        l = 1.f;
#pragma unroll
        for (int e = 0; e < C::kEl; ++e) o[e] = vf[e];
      }
    }

    if (cw == (C::kW > 1 ? 1 : 0) && lane < C::kChunks) {
      // pass the residual stream through, one d_h slice per unit: bwd.x[h*DH .. +DH) = fwd.x[...]
      const uint4* xs = (const uint4*)(hk + 2 * DH);
      *((uint4*)(bwd + (long)b * ld_bwd + (long)h * DH) + lane) = xs[lane];
    }

    for (int c = 0; c < nch; ++c, ++it) {
      const int s = it % C::kStages;
      const int np = max(0, min(C::kTpos, L - c * C::kTpos));
      if (c > 0) mbar_wait(&full[s], (it / C::kStages) & 1);
      if (a.flags & 1) {  // diagnostics: streaming only
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        continue;
      }
      const T* sk = (const T*)(smem + s * C::kStageBytes);
      const T* sv = (const T*)(smem + s * C::kStageBytes + C::kTileBytes);

      float sc[C::kPasses];
      float mx = -INFINITY;
#pragma unroll
      for (int ps = 0; ps < C::kPasses; ++ps) {
        const int r = ps * C::kW * C::kPg + cw * C::kPg + grp;
        float part = 0.f;
        if (r < np) {
          uint4 kc[C::kCpl];
#pragma unroll
          for (int j = 0; j < C::kCpl; ++j) kc[j] = *(const uint4*)(sk + r * DH + (sub + j * C::kLpp) * C::kVec);
          float pp[4] = {0.f, 0.f, 0.f, 0.f};  // four independent FMA chains
#pragma unroll
          for (int j = 0; j < C::kCpl; ++j) {
            float kf[C::kVec];
            chunk_to_f32<T>(kc[j], kf);
#pragma unroll
            for (int e = 0; e < C::kVec; ++e) pp[e & 3] = fmaf(q[j * C::kVec + e], kf[e], pp[e & 3]);
          }
          part = (pp[0] + pp[1]) + (pp[2] + pp[3]);
        }
#pragma unroll
        for (int o2 = C::kLpp / 2; o2 > 0; o2 >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o2);
        sc[ps] = (r < np) ? part : -INFINITY;
        mx = fmaxf(mx, sc[ps]);
      }
#pragma unroll
      for (int o2 = C::kLpp; o2 < 32; o2 <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o2));
      if (mx != -INFINITY) {
        const float mn = fmaxf(m, mx);
        const float corr = (m == -INFINITY) ? 0.f : exp2f(m - mn);
        l *= corr;
#pragma unroll
        for (int e = 0; e < C::kEl; ++e) o[e] *= corr;
#pragma unroll
        for (int ps = 0; ps < C::kPasses; ++ps) {
          const int r = ps * C::kW * C::kPg + cw * C::kPg + grp;
          if (r < np) {
            const float p = exp2f(sc[ps] - mn);
            l += p;
#pragma unroll
            for (int j = 0; j < C::kCpl; ++j) {
              uint4 vc = *(const uint4*)(sv + r * DH + (sub + j * C::kLpp) * C::kVec);
              float vf[C::kVec];
              chunk_to_f32<T>(vc, vf);
#pragma unroll
              for (int e = 0; e < C::kVec; ++e) o[j * C::kVec + e] = fmaf(p, vf[e], o[j * C::kVec + e]);
            }
          }
        }
        m = mn;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (a.flags & 3) continue;  // diagnostics: 1 = streaming only, 2 = no merge / output

    // merge the groups of this warp (m is warp-uniform)
#pragma unroll
    for (int o2 = C::kLpp; o2 < 32; o2 <<= 1) {
      l += __shfl_xor_sync(0xffffffffu, l, o2);
#pragma unroll
      for (int e = 0; e < C::kEl; ++e) o[e] += __shfl_xor_sync(0xffffffffu, o[e], o2);
    }
    // publish this warp's state to combine buffer ui % kNB for the merge warp (no CTA barrier: the
    // consumer warps move on to the next unit)
    const int cb = ui % C::kNB;
    while (comb_seq[cb] != ui / C::kNB) { }  // the merge of unit ui - kNB has left this buffer
    float* cbuf = comb + cb * C::kW * (DH + 2);
    float* cwbuf = cbuf + cw * (DH + 2);
    if (grp == 0) {
#pragma unroll
      for (int j = 0; j < C::kCpl; ++j)
#pragma unroll
        for (int e = 0; e < C::kVec; ++e) cwbuf[(sub + j * C::kLpp) * C::kVec + e] = o[j * C::kVec + e];
    }
    if (lane == 0) { cwbuf[DH] = m; cwbuf[DH + 1] = l; }
    if (cw == 0 && lane == 0) { comb_bh[2 * cb] = b; comb_bh[2 * cb + 1] = h; }
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      atomicAdd(&comb_cnt[cb], 1);
    }
  }
}

}  // namespace gh
