// params.hpp — plain-old-data launch parameters shared by host code and the sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gh {

enum EpiKind : int {
  EPI_STORE = 0,         // out[b, n] = acc
  EPI_STORE_RESID = 1,   // out[b, n] = acc + resid[b, n]
  EPI_QKV_ROPE = 2,      // msg_fwd[b, D + n] = rope(acc) for q/k rows, acc for v rows
  EPI_SWIGLU = 3,        // rows interleaved (gate_f, up_f): out[b, f] = silu(gate) * up
  EPI_LOGITS_ARGMAX = 4  // logits[b, n] = acc (optional); per-tile (max, argmax) over n
};

struct EpiParams {
  int kind;
  void* out;            // output base (storage type T_out: bf16 except logits fp32)
  long ldo;             // output row stride (elements)
  const void* resid;    // residual base (same storage type as out)
  long ldr;
  const float2* rope;   // [max_seq][d_head/2] (cos, sin)
  const int* pos;       // [B]
  int d_head;
  int rope_rows;        // leading output rows (q and k) that receive RoPE
  float* logits;        // [B][ldl] fp32 (optional)
  long ldl;
  float2* part;         // [n_tiles * C][Bt] (max value, argmax index as float bits); C = cluster size
  // fused RMSNorm (bf16 tcgen05 path): the GEMM input X is the raw activation; column b of the
  // accumulator is scaled by 1/sqrt(sum_s ss_in[s][b] / ss_dim + ss_eps) (norm weight folded
  // into W).  ss_in holds per-slice sums of squares written by the producer of X.
  const float* ss_in;   // [ss_in_slices][Bt] or nullptr
  int ss_in_slices;
  int ss_dim;
  float ss_eps;
  // per-slice sums of squares of the rounded outputs of this GEMM (STORE_RESID) for the next
  // fused norm: ss_out[n_tile * C + r][Bt]; nullptr = none
  float* ss_out;
  // QKV_ROPE: copy x[b][n] (row stride xcopy_ld) into the fwd message x slot for n < xcopy_rows
  const void* xcopy_src;
  long xcopy_ld;
  int xcopy_rows;
  // Tier-1 tensor parallelism: all-reduce of the tp_n ranks' fp32 partial outputs
  // inside the epilogue (W_o and W_2, STORE_RESID).  The owner of each output slice stores its
  // partial as {value, tp_seq} words into every peer's receive buffer tp_dst[p]
  // ([tp_n][slice][row][BN] uint2; p == tp_rank is the local one, which the peers write), polls the
  // peers' words of the same slice until they carry tp_seq, and sums the tp_n partials in rank
  // order, then adds the residual.  tp_n <= 1: no exchange.
  int tp_n;
  int tp_rank;
  unsigned int tp_seq;
  float* tp_dst[4];
  int tp_dbg;           // diagnostics (wrong results): 1 = no waiting for the peers, 2 = no peer stores,
                        // 4 = no all-reduce at all
};
constexpr int kMaxTp = 4;

struct GemmShape {
  int N, K, Bt;         // weight rows, reduction length, batch
  int n_tiles, b_tiles; // 128-row weight tiles x BN-column batch tiles
  int kb_total;         // KB = ceil(K / 64)
  int stages;           // TMA -> MMA pipeline depth (shared-memory ring)
  int BN;               // pair kernel: batch columns per tile (multiple of 32, <= 256)
  int flags;            // diagnostics (GEMM_DBG_*), 0 in production
  unsigned long long* trace;  // diagnostics: per-CTA globaltimer stamps [grid][8] (nullptr = off)
  // L2 prefetch of the NEXT kernel's leading weight bytes, issued by each CTA's producer once
  // its own loads are all in flight (fills the HBM idle time of this kernel's tail)
  const void* pf;
  unsigned long long pf_bytes;
  // pair kernel, stream-K: fp32 partial workspace [pairs][256 columns][256 rows] and one flag
  // per (pair, CTA) (zero between launches)
  float* sk_ws;
  unsigned int* sk_flags;
  int sk_split;         // 1: stream-K k-block ranges; 0: contiguous whole-tile ranges
  // Tier-1 of the split over the peer transport: the activation rows (and the residual) arrive
  // from xwait_n Tier-2 GPUs, each publishing sequence number xwait_val in its flag word
  // xwait[j] after its copy (nullptr: the rows belong to earlier kernels only)
  const unsigned int* xwait;
  int xwait_n;
  unsigned int xwait_val;
};
enum GemmDbg : int { GEMM_DBG_NO_MMA = 1, GEMM_DBG_NO_X = 2, GEMM_DBG_NO_HINT = 4, GEMM_DBG_NO_EPI = 8, GEMM_DBG_SK_TILES = 16,
                     GEMM_DBG_NO_STORE = 32 };

struct AttnArgs {
  const void* msg_fwd;  // [B][2D + 2Dkv]
  void* msg_bwd;        // [B][2D]
  void* arena;          // layer base
  const uint32_t* slot; // [B]
  const int* pos;       // [B]  (cached positions before the new token)
  long slot_stride;     // elements per slot (= 2 * Hkv * S * DH)
  long kv_stride;       // elements between K and V blocks (= Hkv * S * DH)
  long head_stride;     // elements per kv head (= S * DH)
  int B, H, Hkv, D, Dkv;
  float scale_log2;     // log2(e) / sqrt(DH)
  int flags;            // diagnostics: 1 = consumers release stages without computing
  const void* pf;       // L2 prefetch of the next kernel's leading weight bytes (see GemmShape)
  unsigned long long pf_bytes;
  int layer_local;      // layer index inside the Tier-2's arena (tensor-core GQA path)
  int n_slots;
  const CUtensorMap* kv_tmap;  // host-side: 3-D map of the whole arena (nullptr = no TMA path)
  // Paged arena (nullptr = contiguous slots): page_table[slot * max_pages + p] is the page holding
  // positions [64p, 64p + 64) of the slot; slot_stride / kv_stride / head_stride then describe a
  // page (2 * Hkv * 64 * DH / Hkv * 64 * DH / 64 * DH) and n_slots is the number of pages.
  const int* page_table;
  int max_pages;
  // Dynamic unit schedule (nullptr = static stride gridDim.x): work[0] hands out units after each
  // CTA's first, work[1] counts finished producers; the last one zeroes both for the next launch.
  unsigned int* work;
  // 1: the kernel's predecessor writes neither the arena nor pos / slot (the QKV GEMM or a stream
  // wait), so the first unit's cached keys / values may be requested before griddepcontrol.wait
  int kv_early;
  // Tier-1 tensor parallelism over tp ranks (1 = none): the messages are the PayloadModel rows cut
  // into tp head blocks, block r = the columns of Tier-1 rank r:
  //   fwd [tp][B][(2D + 2Dkv)/tp] = [x_r | q_r | k_r | v_r],   bwd [tp][B][2D/tp] = [x_r | attn_r]
  // (tp = 1: the plain [x|q|k|v] / [x|attn] rows).  Same bytes per token.
  int tp;
};
// Positions per KV page of the paged arena (one 64-position TMA box / attention stage).
constexpr int kKvPagePositions = 64;

// Element offset (from the layer base) of position `pos` of (slot, kv head) in either layout.
__host__ __device__ inline long kv_offset(const AttnArgs& a, int slot, int head, int pos, int DH) {
  if (a.page_table) {
    const int pg = a.page_table[(long)slot * a.max_pages + pos / kKvPagePositions];
    return (long)pg * a.slot_stride + (long)head * a.head_stride + (long)(pos % kKvPagePositions) * DH;
  }
  return (long)slot * a.slot_stride + (long)head * a.head_stride + (long)pos * DH;
}

}  // namespace gh
