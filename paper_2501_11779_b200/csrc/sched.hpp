// sched.hpp — the batch-state scheduler of the two-tier decode path (host only, no CUDA).
//
// Glinthawk's dispatcher keeps "a set of batch-state objects, each holding the prompts of one
// in-flight batch" and refills a batch's free entries from the request queue as prompts finish
// (P:471-479); the planner sizes the pool with in-flight batches and KV oversubscription
// (optimizer.cpp:194-207, 42-45).  This class is that dispatcher's decision logic:
//
//  * lanes: IF in-flight batches x B rows; lane (ib, row) is bound to one context slot for life;
//    in the tier split row r belongs to Tier-2 shard j of gh_shard_plan(B, K') (analytic.cpp:119)
//  * per-shard page pools (paged arena: 64-position pages, GH_KV_PAGE_POSITIONS), admission maps
//    a request's positions (all of them, or only its prompt with on-demand growth); when a pool
//    runs dry the shard's most recently admitted request is preempted -- by recompute (it
//    re-enters the queue head with its generated tokens appended to its prompt) or by swap (its
//    context goes to host memory and comes back into a lane of the same shard)
//  * every step each lane gets an input: an idle lane a dummy token at position 0, a busy lane its
//    prompt token (host) or the token its previous step generated (device feedback)
//  * chunked prefill (chunk > 1, "the Dispatcher decides which tokens are placed in empty
//    slots of batches"): the idle lanes of an in-flight batch's shard carry further prompt tokens
//    of that shard's busy lanes still reading their prompts -- up to chunk tokens of one request
//    per step, at consecutive positions of the request's own slot (a prefill-row engine appends
//    every row's key and value before attention, so the rows see each other exactly as one token
//    per step would); the request's own lane takes the chunk's last token, so its output and the
//    device feedback stay on its own row
//
// Decisions depend only on prompt lengths, max_new, the page accounting and the step count,
// never on token values, so every rank of a tier split runs the same scheduler and takes the same
// decisions (SPMD); token values are only needed to record outputs and to rebuild a preempted
// request's prompt, and they are supplied a step late (resolve) so the host never waits for the
// step it just queued.
#pragma once
#include <stdint.h>

#include <deque>
#include <string>
#include <vector>

namespace gh {

struct SchedConfig {
  uint32_t batch = 0;        // rows per in-flight batch (B)
  uint32_t inflight = 1;     // in-flight batches (IF)
  uint32_t kp = 0;           // Tier-2 shards per batch (0: colocated, one pool)
  uint32_t pages = 0;        // KV pages per shard pool (0: contiguous slots of max_seq_len)
  uint32_t max_seq = 0;      // positions per slot (max_seq_len)
  uint32_t max_new = 1;      // tokens generated per request (default; submit may override)
  bool on_demand = false;    // paged: map the prompt only, grow a page at a time
  bool swap = false;         // preemption by swap (else recompute)
  bool shortest = false;     // admission order: shortest prompt first (else FIFO)
  uint32_t chunk = 1;        // prompt tokens of one request per step (> 1: chunked prefill into idle lanes)
};

// input of one lane for the next step
enum LaneSrc : int32_t { kIdle = 0, kHost = 1, kDevice = 2 };
struct LaneInput {
  int32_t src, tok, pos;
  uint32_t home;    // the lane whose slot this row appends to and attends over (itself, or the
                    // lane whose prompt chunk it carries)
};
// KV action on a lane's slot, applied (before the step) by the rank holding the lane's shard
enum KvOp : int32_t { kMap = 0, kUnmap = 1, kSwapOut = 2, kSwapIn = 3 };
struct KvAction {
  int32_t op;
  uint32_t lane;
  uint32_t n;       // positions (map: [0, n) backed; swap: [0, n) copied)
  uint64_t buf;     // swap buffer id
};

class Sched {
 public:
  static constexpr uint32_t kPage = 64;
  // returns "" or the validation error
  std::string init(const SchedConfig& c);
  // "" or the reason the request can never be served (longer than a slot / a page pool)
  std::string submit(const int32_t* prompt, uint32_t len, float temperature, uint32_t seed, uint64_t* id,
                     uint32_t max_new = 0);  // max_new 0: the configured one
  // the next step: inputs of every lane (IF * B) and the KV actions to apply first.  Returns an
  // error string (infeasible request) or "".
  std::string plan(std::vector<LaneInput>& in, std::vector<KvAction>& acts);
  void commit();                       // the planned step was issued
  void resolve(const int32_t* next);   // next tokens (IF * B) of the oldest unresolved step
  bool done() const;
  uint32_t unresolved() const { return (uint32_t)pending_.size(); }
  // per-lane sampling state (changed since the last call -> true)
  bool sampling(std::vector<float>& inv_temp, std::vector<uint32_t>& seed);
  const std::vector<int32_t>* result(uint64_t id) const;
  uint64_t steps = 0, preemptions = 0, swaps = 0, admitted = 0, finished = 0, tokens = 0;
  uint64_t lane_steps = 0;             // busy lanes summed over steps (tokens processed, prompt or generated)
  uint64_t context_sum = 0;            // positions attended, summed over busy lane-steps
  uint32_t lane_shard(uint32_t lane) const { return shard_of_[lane % c_.batch]; }
  uint32_t lanes() const { return c_.batch * c_.inflight; }
  uint32_t peak_pages = 0;             // the largest number of pages of one pool in use (tests)

 private:
  struct Req {
    std::vector<int32_t> prompt;       // grows by the generated tokens on recompute preemption
    uint32_t orig_len = 0;             // the submitted prompt's length (output k sits at orig_len + k)
    uint32_t max_new = 0;              // tokens to generate
    bool recompute = false;            // preempted by recompute: re-read prompt + outputs on admission
    std::vector<int32_t> out;          // generated tokens (values resolved a step late)
    uint32_t n_out = 0;                // generated so far (resolved or not)
    uint32_t resolved = 0;             // out[0, resolved) hold values
    float temp = 0.f;
    uint32_t seed = 0;
    // swap preemption: positions saved, shard holding the buffer, buffer id
    bool swapped = false;
    uint32_t swap_t = 0, swap_shard = 0;
    uint64_t swap_buf = 0;
    bool done = false;
  };
  struct Lane {
    int64_t req = -1;
    uint32_t t = 0;                    // position of the next input token
    uint64_t seq = 0;                  // admission order
    uint32_t mapped = 0;               // pages held
    bool fed_back = false;             // the previous step of this lane produced its next input
    bool freed = false;                // its request finished at the last commit: return the pages
    uint32_t fed = 1;                  // prompt / output tokens fed by the planned step (chunked prefill)
  };
  uint32_t pages_for(uint32_t n) const { return (n + kPage - 1) / kPage; }
  bool paged() const { return c_.pages > 0; }
  bool try_map(uint32_t lane, uint32_t n, std::vector<KvAction>& acts);
  void unmap(uint32_t lane, std::vector<KvAction>& acts);
  void release(uint32_t lane, std::vector<KvAction>& acts);
  bool admissible(const Req& r, uint32_t lane) const;
  uint32_t admit_need(const Req& r) const;
  void admit(uint32_t lane, std::vector<KvAction>& acts);
  void preempt(uint32_t lane, std::vector<KvAction>& acts);
  std::string grow(std::vector<KvAction>& acts);

  SchedConfig c_;
  std::vector<uint32_t> shard_of_;     // row -> shard
  std::vector<uint32_t> free_;         // per shard: free pages
  std::vector<uint32_t> unmapped_;     // per shard: lanes holding no page
  // admission order: the k-th lane of every (in-flight batch, shard) group before any group's
  // (k+1)-th, so a partly filled pool spreads its requests over the batches and Tier-2 shards
  // (equal Tier-2 load) and leaves idle lanes beside each for chunked prefill
  std::vector<uint32_t> admit_order_;
  std::vector<Req> reqs_;
  std::deque<uint64_t> queue_;
  std::vector<Lane> lanes_;
  uint64_t admit_seq_ = 0, swap_ids_ = 0;
  bool sampling_dirty_ = false;
  // outputs of committed steps awaiting their token values: (request, output index, lane)
  struct Emit { uint64_t req; uint32_t idx; uint32_t lane; };
  std::deque<std::vector<Emit>> pending_;
  std::vector<Emit> cur_;              // outputs of the planned (not yet committed) step
  void chunk_prefill(std::vector<LaneInput>& in, std::vector<KvAction>& acts);
};

}  // namespace gh
