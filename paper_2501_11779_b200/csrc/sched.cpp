// sched.cpp — batch-state scheduler; see sched.hpp.
#include "sched.hpp"

#include <algorithm>

namespace gh {

std::string Sched::init(const SchedConfig& c) {
  if (c.batch == 0 || c.inflight == 0) return "batch and inflight must be >= 1";
  if (c.kp > c.batch) return "more Tier-2 shards than rows";
  if (c.max_new == 0) return "max_new must be >= 1";
  if (c.on_demand && c.pages == 0) return "on-demand paging needs a paged KV arena";
  c_ = c;
  if (c_.chunk == 0) c_.chunk = 1;
  const uint32_t ns = std::max(1u, c.kp);
  shard_of_.assign(c.batch, 0);
  for (uint32_t j = 0, row = 0; j < ns; ++j) {  // balanced shards, low shards first (analytic.cpp:119)
    const uint32_t n = c.batch / ns + (j < c.batch % ns ? 1 : 0);
    for (uint32_t i = 0; i < n; ++i) shard_of_[row++] = j;
  }
  free_.assign(ns, c.pages);
  lanes_.assign((size_t)c.batch * c.inflight, Lane{});
  unmapped_.assign(ns, 0);
  for (uint32_t l = 0; l < lanes(); ++l) ++unmapped_[lane_shard(l)];
  std::vector<uint32_t> first(ns + 1, 0);  // first row of each shard
  for (uint32_t row = 0; row < c.batch; ++row) first[shard_of_[row] + 1] = row + 1;
  admit_order_.clear();
  for (uint32_t k = 0; k < c.batch; ++k)
    for (uint32_t ib = 0; ib < c.inflight; ++ib)
      for (uint32_t j = 0; j < ns; ++j)
        if (first[j] + k < first[j + 1]) admit_order_.push_back(ib * c.batch + first[j] + k);
  if (paged()) {
    std::vector<uint32_t> per(ns, 0);
    for (uint32_t l = 0; l < lanes(); ++l) ++per[lane_shard(l)];
    for (uint32_t j = 0; j < ns; ++j)
      if (per[j] > c.pages) return "KV page pool smaller than one page per lane";
  }
  return "";
}

std::string Sched::submit(const int32_t* prompt, uint32_t len, float temperature, uint32_t seed, uint64_t* id_out,
                          uint32_t max_new) {
  if (len == 0) return "empty prompt";
  if (max_new == 0) max_new = c_.max_new;
  const uint32_t positions = len + max_new - 1;  // every position the request ever attends
  if (c_.max_seq && positions > c_.max_seq)
    return "request needs " + std::to_string(positions) + " positions, max_seq_len is " + std::to_string(c_.max_seq);
  if (paged()) {  // it must fit its shard's pool beside one dummy page per other lane
    uint32_t most = 0;
    std::vector<uint32_t> per(free_.size(), 0);
    for (uint32_t l = 0; l < lanes(); ++l) most = std::max(most, ++per[lane_shard(l)]);
    if (pages_for(positions) > c_.pages - (most - 1))
      return "request needs " + std::to_string(pages_for(positions)) + " KV pages, a shard's pool can give " +
             std::to_string(c_.pages - (most - 1)) + " (binding constraint: memory)";
  }
  Req r;
  r.prompt.assign(prompt, prompt + len);
  r.orig_len = len;
  r.max_new = max_new;
  r.temp = temperature;
  r.seed = seed;
  reqs_.push_back(std::move(r));
  const uint64_t id = reqs_.size() - 1;
  if (c_.shortest) {  // stable: after every queued request of the same or a shorter prompt
    auto it = std::upper_bound(queue_.begin(), queue_.end(), len,
                               [&](uint32_t l, uint64_t q) { return l < reqs_[q].prompt.size(); });
    queue_.insert(it, id);
  } else {
    queue_.push_back(id);
  }
  *id_out = id;
  return "";
}

bool Sched::try_map(uint32_t lane, uint32_t n, std::vector<KvAction>& acts) {
  if (n > c_.max_seq && c_.max_seq) return false;
  if (!paged()) return true;  // contiguous slots hold max_seq_len positions
  Lane& L = lanes_[lane];
  const uint32_t need = pages_for(n) > L.mapped ? pages_for(n) - L.mapped : 0;
  const uint32_t sh = lane_shard(lane);
  // keep one page for every other lane of the shard that holds none (its dummy token)
  const uint32_t empty = unmapped_[sh] - (L.mapped == 0 ? 1 : 0);
  if (need + empty > free_[sh]) return false;
  if (need) {
    free_[sh] -= need;
    if (L.mapped == 0) --unmapped_[sh];
    L.mapped += need;
    acts.push_back({kMap, lane, n, 0});
    peak_pages = std::max(peak_pages, c_.pages - free_[sh]);
  }
  return true;
}

void Sched::unmap(uint32_t lane, std::vector<KvAction>& acts) {
  Lane& L = lanes_[lane];
  if (paged() && L.mapped) {
    free_[lane_shard(lane)] += L.mapped;
    ++unmapped_[lane_shard(lane)];
    L.mapped = 0;
    acts.push_back({kUnmap, lane, 0, 0});
  }
}

void Sched::release(uint32_t lane, std::vector<KvAction>& acts) {
  unmap(lane, acts);
  Lane& L = lanes_[lane];
  if (L.req >= 0 && reqs_[L.req].temp != 0.f) sampling_dirty_ = true;
  L.req = -1;
  L.t = 0;
  L.fed_back = false;
}

// A request may take this lane: a swapped one only in its own shard (its context is in that
// shard's host buffer) and, like a recompute victim, once every token it generated has a value.
bool Sched::admissible(const Req& r, uint32_t lane) const {
  if (r.swapped && r.swap_shard != lane_shard(lane)) return false;
  return r.resolved == r.n_out;
}

uint32_t Sched::admit_need(const Req& r) const {
  if (r.swapped) return r.swap_t + 1;  // the saved context plus the position it decodes next
  if (c_.on_demand) return r.orig_len + r.n_out;  // the prompt (+ the outputs it re-reads)
  return r.orig_len + r.max_new - 1;
}

void Sched::admit(uint32_t lane, std::vector<KvAction>& acts) {
  // FIFO (or shortest-first) over the requests this lane may take; the first one that may take
  // it is the only candidate (no overtaking by a smaller request that happens to fit)
  for (auto it = queue_.begin(); it != queue_.end(); ++it) {
    Req& r = reqs_[*it];
    if (!admissible(r, lane)) continue;
    if (!try_map(lane, admit_need(r), acts)) break;
    const uint64_t id = *it;
    queue_.erase(it);
    Lane& L = lanes_[lane];
    L.req = (int64_t)id;
    L.t = 0;
    L.seq = ++admit_seq_;
    L.fed_back = false;
    ++admitted;
    if (r.swapped) {  // resume at the saved position
      acts.push_back({kSwapIn, lane, r.swap_t, r.swap_buf});
      L.t = r.swap_t;
      r.swapped = false;
    } else if (r.recompute) {
      // recompute: re-read the prompt and every token generated so far (all resolved)
      r.prompt.resize(r.orig_len);
      r.prompt.insert(r.prompt.end(), r.out.begin(), r.out.begin() + r.n_out);
      r.recompute = false;
    }
    if (r.temp != 0.f) sampling_dirty_ = true;
    return;
  }
  // idle: a dummy token at position 0 of its own slot (one page)
  try_map(lane, 1, acts);
}

void Sched::preempt(uint32_t lane, std::vector<KvAction>& acts) {
  Lane& L = lanes_[lane];
  Req& r = reqs_[L.req];
  const uint64_t id = (uint64_t)L.req;
  if (c_.swap && L.t > 0) {
    r.swapped = true;
    r.swap_t = L.t;
    r.swap_shard = lane_shard(lane);
    r.swap_buf = ++swap_ids_;
    acts.push_back({kSwapOut, lane, L.t, r.swap_buf});
    ++swaps;
  } else {
    // recompute on re-admission (admit() appends the generated tokens once their values are known)
    r.recompute = true;
  }
  queue_.push_front(id);
  release(lane, acts);
  ++preemptions;
  try_map(lane, 1, acts);  // the idle lane's dummy token (its own pages just came back)
}

std::string Sched::grow(std::vector<KvAction>& acts) {
  std::vector<uint32_t> order;
  for (uint32_t l = 0; l < lanes(); ++l)
    if (lanes_[l].req >= 0) order.push_back(l);
  std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return lanes_[a].seq < lanes_[b].seq; });
  for (uint32_t lane : order) {
    Lane& L = lanes_[lane];
    if (L.req < 0 || pages_for(L.t + 1) <= L.mapped) continue;
    while (!try_map(lane, L.t + 1, acts)) {
      const uint32_t sh = lane_shard(lane);
      int64_t victim = -1;
      for (uint32_t o = 0; o < lanes(); ++o)
        if (lanes_[o].req >= 0 && lane_shard(o) == sh && (victim < 0 || lanes_[o].seq > lanes_[victim].seq))
          victim = o;
      if (victim < 0) return "KV page pool cannot back a single request";
      preempt((uint32_t)victim, acts);
      if ((uint32_t)victim == lane) break;
    }
  }
  return "";
}

std::string Sched::plan(std::vector<LaneInput>& in, std::vector<KvAction>& acts) {
  acts.clear();
  // finished requests gave their lanes back at commit; admissions first (spread order)
  for (uint32_t l : admit_order_)
    if (lanes_[l].req < 0) {
      if (lanes_[l].freed) {  // its request finished at the last commit
        unmap(l, acts);
        lanes_[l].freed = false;
      }
      admit(l, acts);
    }
  if (c_.on_demand) {
    std::string e = grow(acts);
    if (!e.empty()) return e;
  }
  bool busy = false;
  for (auto& L : lanes_) busy |= L.req >= 0;
  if (!busy && !queue_.empty() && pending_.empty()) {
    const Req& r = reqs_[queue_.front()];
    return "request " + std::to_string(queue_.front()) + " needs " + std::to_string(admit_need(r)) +
           " positions, more than a KV page pool can back";
  }
  in.resize(lanes());
  cur_.clear();
  for (uint32_t l = 0; l < lanes(); ++l) {
    Lane& L = lanes_[l];
    L.fed = 1;
    in[l] = {kIdle, 0, 0, l};
    if (L.req < 0) continue;
    const Req& r = reqs_[L.req];
    const uint32_t plen = (uint32_t)r.prompt.size();
    if (L.t < plen) in[l] = {kHost, r.prompt[L.t], (int32_t)L.t, l};
    else if (L.fed_back) in[l] = {kDevice, 0, (int32_t)L.t, l};
    else in[l] = {kHost, r.out[L.t - r.orig_len], (int32_t)L.t, l};
  }
  if (c_.chunk > 1) chunk_prefill(in, acts);
  return "";
}

void Sched::chunk_prefill(std::vector<LaneInput>& in, std::vector<KvAction>& acts) {
  const uint32_t B = c_.batch, ns = std::max(1u, c_.kp);
  std::vector<uint32_t> idle, reading;
  for (uint32_t ib = 0; ib < c_.inflight; ++ib)
    for (uint32_t j = 0; j < ns; ++j) {
      idle.clear();
      reading.clear();
      for (uint32_t row = 0; row < B; ++row) {
        if (shard_of_[row] != j) continue;
        const uint32_t l = ib * B + row;
        const Lane& L = lanes_[l];
        if (L.req < 0) idle.push_back(l);
        else if (L.t + 1 < reqs_[L.req].prompt.size()) reading.push_back(l);  // >= 2 prompt tokens left
      }
      if (idle.empty() || reading.empty()) continue;
      std::sort(reading.begin(), reading.end(), [&](uint32_t a, uint32_t b) { return lanes_[a].seq < lanes_[b].seq; });
      size_t next_idle = 0;
      for (uint32_t l : reading) {  // oldest admission first
        Lane& L = lanes_[l];
        const Req& r = reqs_[L.req];
        uint32_t extra = std::min<uint32_t>({c_.chunk - 1, (uint32_t)r.prompt.size() - L.t - 1,
                                             (uint32_t)(idle.size() - next_idle)});
        // on-demand paging: the chunk's positions must be backed (the whole request is otherwise)
        while (extra && c_.on_demand && !try_map(l, L.t + extra + 1, acts)) --extra;
        if (!extra) continue;
        for (uint32_t k = 0; k < extra; ++k)  // borrowed rows: the chunk's leading tokens
          in[idle[next_idle++]] = {kHost, r.prompt[L.t + k], (int32_t)(L.t + k), l};
        in[l] = {kHost, r.prompt[L.t + extra], (int32_t)(L.t + extra), l};  // its own row: the last
        L.fed = extra + 1;
        if (next_idle == idle.size()) break;
      }
    }
}

void Sched::commit() {
  ++steps;
  for (uint32_t l = 0; l < lanes(); ++l) {
    Lane& L = lanes_[l];
    if (L.req < 0) continue;
    Req& r = reqs_[L.req];
    const uint32_t plen = (uint32_t)r.prompt.size();
    const uint32_t n = L.fed;  // tokens fed at positions [t, t + n); the lane's own row held the last
    lane_steps += n;
    context_sum += (uint64_t)n * L.t + (uint64_t)n * (n + 1) / 2;
    L.t += n - 1;
    L.fed = 1;
    if (L.t + 1 >= plen) {  // this step's output is the request's next token
      cur_.push_back({(uint64_t)L.req, r.n_out, l});
      ++r.n_out;
      r.out.resize(r.n_out);
      ++tokens;
      L.fed_back = true;
    } else {
      L.fed_back = false;
    }
    ++L.t;
    if (r.n_out == r.max_new) {  // done: the lane (and its slot) goes to the next request
      r.done = true;
      ++finished;
      if (r.temp != 0.f) sampling_dirty_ = true;
      L.req = -1;
      L.t = 0;
      L.fed_back = false;
      L.freed = true;      // pages are returned by the next plan (before any admission)
    }
  }
  pending_.push_back(cur_);
  cur_.clear();
}

void Sched::resolve(const int32_t* next) {
  if (pending_.empty()) return;
  for (const Emit& e : pending_.front()) {
    Req& r = reqs_[e.req];
    r.out[e.idx] = next ? next[e.lane] : 0;
    r.resolved = std::max(r.resolved, e.idx + 1);
  }
  pending_.pop_front();
}

bool Sched::done() const {
  if (!queue_.empty()) return false;
  for (auto& L : lanes_)
    if (L.req >= 0) return false;
  return true;
}

bool Sched::sampling(std::vector<float>& inv_temp, std::vector<uint32_t>& seed) {
  if (!sampling_dirty_) return false;
  sampling_dirty_ = false;
  inv_temp.assign(lanes(), 0.f);
  seed.assign(lanes(), 0u);
  for (uint32_t l = 0; l < lanes(); ++l)
    if (lanes_[l].req >= 0) {
      const Req& r = reqs_[lanes_[l].req];
      inv_temp[l] = r.temp > 0.f ? 1.0f / r.temp : 0.f;
      seed[l] = r.seed;
    }
  return true;
}

const std::vector<int32_t>* Sched::result(uint64_t id) const {
  if (id >= reqs_.size() || !reqs_[id].done || reqs_[id].resolved < reqs_[id].n_out) return nullptr;
  return &reqs_[id].out;
}

}  // namespace gh
