// common.cuh — device helpers shared by every sm_100a kernel of the two-tier decode path:
// storage-type traits (fp32 / bf16), the deterministic synthetic-weight generator, and thin
// inline-PTX wrappers for mbarrier, TMA / bulk copies and tcgen05.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#define GH_DEV __device__ __forceinline__
#define GH_HD __host__ __device__ __forceinline__

namespace gh {

constexpr int kNumSMs = 148;

// ------------------------------------------------------------------ storage types
// fp32 storage (C1 tiny model) or bf16 storage (7B/13B/70B shapes).  Compute is fp32.
struct bf16_t { uint16_t bits; };

// ---- temperature sampling (Gumbel-max, argmax_rows_kernel over the written logits):
// token = argmax_r(logit_r / T + g_r), g_r = -log(-log(u_r))
// with u_r a counter-based uniform of (seed, position, r); T = 0 rows stay greedy.  The scores
// use separately rounded fp32 multiply / add and the noise is computed in double and rounded
// once, so a numpy restatement (oracle/sampling.py) reproduces every decision bit for bit.
GH_HD uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
GH_HD uint64_t sample_key(uint32_t seed, int pos) { return splitmix64(((uint64_t)seed << 32) | (uint32_t)pos); }
GH_DEV float gumbel_noise(uint64_t key, int r) {
  const uint64_t h = splitmix64(key + (uint64_t)r);
  const double u = ((double)(h >> 11) + 0.5) * 0x1p-53;
  return (float)(-log(-log(u)));
}
GH_DEV float sample_score(float logit, float inv_t, uint64_t key, int r) {
  return __fadd_rn(__fmul_rn(logit, inv_t), gumbel_noise(key, r));
}

GH_HD float bf16_to_f32(uint16_t b) {
  union { uint32_t u; float f; } v; v.u = (uint32_t)b << 16; return v.f;
}
// Round-to-nearest-even (finite inputs); identical to the oracle's restatement.
GH_HD uint16_t f32_to_bf16(float f) {
#ifdef __CUDA_ARCH__
  uint16_t r;  // one cvt.rn (the bit manipulation below costs ~10 instructions per element)
  asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(r) : "f"(f));
  return r;
#endif
  union { uint32_t u; float f; } v; v.f = f;
  uint32_t u = v.u;
  if ((u & 0x7f800000u) == 0x7f800000u) return (uint16_t)((u >> 16) | ((u & 0xffff) ? 0x40 : 0));
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

#ifdef __CUDACC__
// Two floats -> packed bf16x2 (lo in bits 0..15) with one cvt.rn (round-to-nearest-even: the same
// bits as f32_to_bf16 for every finite input).
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
#endif

template <typename T> struct St;
template <> struct St<float> {
  static constexpr int kBytes = 4;
  static GH_HD float load(const float* p, size_t i) { return p[i]; }
  static GH_HD void store(float* p, size_t i, float v) { p[i] = v; }
  static GH_HD float from_f32(float v) { return v; }
};
template <> struct St<bf16_t> {
  static constexpr int kBytes = 2;
  static GH_HD float load(const bf16_t* p, size_t i) { return bf16_to_f32(p[i].bits); }
  static GH_HD void store(bf16_t* p, size_t i, float v) { p[i].bits = f32_to_bf16(v); }
};

// ------------------------------------------------------------------ synthetic weights
// value(seed, tensor, idx) = Irwin-Hall(4) approximation of N(0,1) times `k`, built only from
// integer hashing, one int->float conversion and one multiply so that the CPU oracle's
// restatement is bit-identical (no transcendental, no FMA contraction).
GH_HD uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
GH_HD uint64_t tensor_base(uint64_t seed, uint64_t tensor) {
  return mix64(seed ^ (tensor * 0xD1B54A32D192ED03ull));
}
// k = sqrt(3) * std / 2^24 (computed in double on the host, rounded to float)
GH_DEV float randn_scaled(uint64_t base, uint64_t idx, float k) {
  uint64_t h0 = mix64(base + 2 * idx);
  uint64_t h1 = mix64(base + 2 * idx + 1);
  int64_t s = (int64_t)(h0 >> 40) + (int64_t)((h0 >> 16) & 0xFFFFFF) +
              (int64_t)(h1 >> 40) + (int64_t)((h1 >> 16) & 0xFFFFFF);
  int64_t c = s - (int64_t)2 * (1 << 24);  // centred, |c| < 2^25
  return __fmul_rn(__ll2float_rn(c), k);
}

// Tensor ids of the synthetic model.
enum : uint64_t { kTidEmbed = 1, kTidCls = 2 };
GH_HD uint64_t tid_layer(uint64_t layer, uint64_t which) { return 64 + layer * 16 + which; }
enum : uint64_t { kWq = 0, kWk = 1, kWv = 2, kWo = 3, kW1 = 4, kW3 = 5, kW2 = 6 };
GH_HD uint64_t tid_kv(uint64_t layer, uint64_t slot, uint64_t kv) {
  return (1ull << 40) | (layer << 24) | (slot << 1) | kv;
}

// ------------------------------------------------------------------ misc device helpers
GH_DEV unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
GH_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
GH_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
GH_DEV bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}\n"
      : "=r"(pred));
  return pred != 0;
}

// ------------------------------------------------------------------ programmatic dependent launch
// Every decode-path kernel is launched with programmatic stream serialization: it lets its
// dependents launch as soon as all of its CTAs have started (griddep_launch_dependents), and
// waits for its predecessor's completion + memory visibility (griddep_wait) only before it reads
// data the predecessor produced (weights and its own prologue overlap the predecessor's tail).
// Both are no-ops when the kernel was launched without the attribute.
GH_DEV void griddep_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
GH_DEV void griddep_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// ------------------------------------------------------------------ mbarrier
GH_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
GH_DEV void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
GH_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}
// raise the expected transaction bytes of the current phase without arriving
GH_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}
GH_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
GH_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// ------------------------------------------------------------------ thread-block clusters / DSMEM
GH_DEV uint32_t cluster_ctarank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
GH_DEV uint32_t cluster_nctarank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r)); return r; }
GH_DEV uint32_t cluster_id_x() { uint32_t r; asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r)); return r; }
GH_DEV uint32_t cluster_count_x() { uint32_t r; asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r)); return r; }
// shared::cta address -> shared::cluster address of the same variable in CTA `rank`
GH_DEV uint32_t mapa_shared(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// (volatile keeps it after the preceding mbarrier wait; no memory clobber so that a batch of
// these loads can be issued back to back before their results are consumed)
GH_DEV void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAITC_%=;\n\t}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}
GH_DEV void mbar_arrive_cluster_relaxed(uint32_t caddr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(caddr) : "memory");
}
GH_DEV void fence_acq_rel_cluster() { asm volatile("fence.acq_rel.cluster;" ::: "memory"); }
GH_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// spin (acquire, gpu scope) until *flag >= target
GH_DEV void flag_wait(const unsigned int* flag, unsigned int target) {
  unsigned int v;
  for (;;) {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (v >= target) break;
    __nanosleep(64);  // polls go to L2: back off
  }
}

// System-scope flag between GPUs: acquire spin on a local flag word that a peer's copy engine
// (cuStreamWriteValue32 after its copy) advances to a sequence number.
GH_DEV void flag_wait_sys(const unsigned int* flag, unsigned int target) {
  unsigned int v;
  for (;;) {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if ((int)(v - target) >= 0) break;  // sequence numbers (wrap-safe)
    __nanosleep(32);
  }
}

// ------------------------------------------------------------------ bulk / tensor copies (TMA)
// 1-D bulk copy global -> shared, completion signalled on an mbarrier (SASS: UBLKCP).
GH_DEV void bulk_g2s(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar,
                     uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;\n" ::"r"(smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
GH_DEV uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
GH_DEV uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
// 2-D tiled TMA load (SASS: UTMALDG)
GH_DEV void tma_load_2d(void* smem_dst, const void* tmap, int c0, int c1, uint64_t* bar,
                        uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(smem_u32(smem_dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
GH_DEV void tma_load_2d_nohint(void* smem_dst, const void* tmap, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(smem_dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// Bulk L2 prefetch (no completion tracking): part `part` of `nparts` equal shares of [base, +bytes).
GH_DEV void prefetch_l2_share(const void* base, unsigned long long bytes, int part, int nparts) {
  if (!base || bytes == 0) return;
  const unsigned long long share = ((bytes + nparts - 1) / nparts + 4095) & ~4095ull;
  const unsigned long long lo = share * part;
  const unsigned long long hi = lo + share < bytes ? lo + share : bytes;
  for (unsigned long long o = lo; o < hi; o += 32768) {
    const uint32_t n = (uint32_t)((hi - o < 32768 ? hi - o : 32768) & ~15ull);
    if (n) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"((const char*)base + o), "r"(n) : "memory");
  }
}
GH_DEV void prefetch_tmap(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(tmap) : "memory");
}

// ------------------------------------------------------------------ tcgen05
GH_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
GH_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
template <uint32_t kCols>
GH_DEV void tmem_alloc(uint32_t* smem_dst) {  // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                   smem_u32(smem_dst)),
               "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
}
template <uint32_t kCols>
GH_DEV void tmem_free(uint32_t taddr) {  // whole warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "n"(kCols));
}
// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (bf16 in, fp32 accumulate)
GH_DEV void umma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                      uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// Arrive on an mbarrier once all previously issued tcgen05.mma of this thread complete.
GH_DEV void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
          smem_u32(bar))
      : "memory");
}
// ---- CTA-pair (cta_group::2) variants: the two CTAs of a cluster pair share one M = 256 MMA.
// Both CTAs' allocator warps allocate together (same column count, same smem slot offset).
template <uint32_t kCols>
GH_DEV void tmem_alloc_pair(uint32_t* smem_dst) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(smem_dst)),
               "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
}
template <uint32_t kCols>
GH_DEV void tmem_free_pair(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "n"(kCols));
}
// Issued by the leader CTA only: A rows 0..127 / B rows 0..N/2-1 come from the leader's shared
// memory, A rows 128..255 / B rows N/2..N-1 from the peer's at the same offsets; D rows 0..127
// land in the leader's TMEM and rows 128..255 in the peer's.
GH_DEV void umma_bf16_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// Arrive on the mbarrier at the same offset in every CTA of `mask` once the leader's previously
// issued pair MMAs complete.
GH_DEV void umma_commit_pair(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
// TMA into this CTA's shared memory whose completion is signalled on the LEADER's mbarrier
// (`leader_bar` is a shared::cluster address, see mapa_shared).
GH_DEV void tma_load_2d_pair(void* smem_dst, const void* tmap, int c0, int c1, uint32_t leader_bar,
                             uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(smem_u32(smem_dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(leader_bar), "l"(policy)
      : "memory");
}

// 32 lanes x 32b, 16 consecutive columns per thread
GH_DEV void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
GH_DEV void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row atoms of 128 B (SBO = 1024 B).
GH_DEV uint64_t umma_desc_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);  // start address
  d |= (uint64_t)1 << 16;                       // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;             // SBO
  d |= (uint64_t)1 << 46;                       // version (sm100)
  d |= (uint64_t)2 << 61;                       // SWIZZLE_128B
  return d;
}
// Instruction descriptor: bf16 x bf16 -> f32, both K-major, M x N.
GH_HD uint32_t umma_idesc_bf16(uint32_t M, uint32_t N) {
  return (1u << 4)            // D = f32
         | (1u << 7)          // A = bf16
         | (1u << 10)         // B = bf16
         | ((N >> 3) << 17)   // N
         | ((M >> 4) << 24);  // M
}

}  // namespace gh
