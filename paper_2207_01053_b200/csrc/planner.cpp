// planner.cpp — protea_plan: profile-driven packing of clients onto GPU slots.
//
// PAPER.md §3.2: the VCE schedules "the clients in the round in a FIFO
// fashion with as many clients running concurrently as the available system
// resources can hold; ... once a client has finished training, the resources
// get freed and another client in the round will be spawned".  §3.4 Eq. (1)
// turns a client's measured VRAM into its GPU share.  §5:
// memory does not predict compute, so the multi-GPU split balances FLOPs.
//
// Integer-only (a float margin would make ceil(2600*1.10) = 2861, SURVEY
// finding 5).  Steps:
//  0 validate; slot = align256(ceil(peak * margin / 1000)); slot > max C -> NO_CAPACITY
//  1 LPT: sort (flops desc, id asc); GPU with min (load, g) among C_g >= slot
//  2 per GPU replay in lock-step iterations: strict head-of-line FIFO, lowest-
//    offset first-fit, release in ascending id at each event, gaps coalesced
//  3 output ascending id; makespan_g = max release
#include <algorithm>
#include <map>
#include <string>
#include <vector>

#include "common.h"

namespace protea {
void set_global_error(const std::string& msg);
}

using namespace protea;

extern "C" protea_status protea_plan(const protea_profile* profiles, size_t n, const protea_cluster* cluster,
                                     const protea_plan_opts* opts, protea_assignment* out,
                                     uint64_t* makespan_steps) {
  if (!profiles || !cluster || !opts || !out || !makespan_steps || n == 0 || cluster->n_gpus == 0 ||
      !cluster->capacity) {
    set_global_error("protea_plan: null argument, n == 0 or no GPU");
    return PROTEA_ERR_INVALID;
  }
  const uint32_t G = cluster->n_gpus;
  std::vector<uint64_t> cap(cluster->capacity, cluster->capacity + G);
  for (uint32_t g = 0; g < G; ++g)
    if (cap[g] == 0) {
      set_global_error("protea_plan: GPU " + std::to_string(g) + " has zero capacity");
      return PROTEA_ERR_INVALID;
    }
  if (opts->margin_permille < 1000 || (opts->policy != PROTEA_POLICY_PROFILED && opts->policy != PROTEA_POLICY_STATIC) ||
      (opts->order != PROTEA_ORDER_ASC_ID && opts->order != PROTEA_ORDER_DESC_STEPS)) {
    set_global_error("protea_plan: bad options (margin_permille >= 1000, policy, order)");
    return PROTEA_ERR_INVALID;
  }
  // unsigned __int128 keeps total capacity / 1024*slot exact for any u64 input
  unsigned __int128 total_cap = 0;
  uint64_t maxcap = 0;
  for (uint64_t c : cap) {
    total_cap += c;
    maxcap = std::max(maxcap, c);
  }
  std::vector<size_t> idx(n);
  std::map<int64_t, size_t> byid;
  std::vector<uint64_t> slot(n);
  for (size_t i = 0; i < n; ++i) {
    const protea_profile& p = profiles[i];
    if (!byid.emplace(p.client_id, i).second) {
      set_global_error("protea_plan: duplicate client id " + std::to_string(p.client_id));
      return PROTEA_ERR_INVALID;
    }
    if (p.steps == 0 || p.peak_bytes == 0) {
      set_global_error("protea_plan: client " + std::to_string(p.client_id) + " has zero steps or peak_bytes");
      return PROTEA_ERR_INVALID;
    }
    unsigned __int128 num = (unsigned __int128)p.peak_bytes * opts->margin_permille;
    unsigned __int128 s = (num + 999) / 1000;
    s = (s + kAlign - 1) / kAlign * kAlign;
    if (s > maxcap) {
      set_global_error("protea_plan: client " + std::to_string(p.client_id) + " needs a slot of " +
                       std::to_string((unsigned long long)s) + " B, more than any GPU holds");
      return PROTEA_ERR_NO_CAPACITY;
    }
    slot[i] = (uint64_t)s;
    idx[i] = i;
  }
  // 1. LPT partition
  std::sort(idx.begin(), idx.end(), [&](size_t a, size_t b) {
    if (profiles[a].flops != profiles[b].flops) return profiles[a].flops > profiles[b].flops;
    return profiles[a].client_id < profiles[b].client_id;
  });
  std::vector<unsigned __int128> load(G, 0);
  std::vector<std::vector<size_t>> members(G);
  for (size_t i : idx) {
    int best = -1;
    for (uint32_t g = 0; g < G; ++g)
      if (cap[g] >= slot[i] && (best < 0 || load[g] < load[best])) best = (int)g;
    load[best] += profiles[i].flops;
    members[best].push_back(i);
  }
  // 2. per-GPU admission replay
  std::vector<protea_assignment> res(n);
  for (uint32_t g = 0; g < G; ++g) {
    auto& q = members[g];
    if (opts->order == PROTEA_ORDER_ASC_ID)
      std::sort(q.begin(), q.end(), [&](size_t a, size_t b) { return profiles[a].client_id < profiles[b].client_id; });
    else
      std::sort(q.begin(), q.end(), [&](size_t a, size_t b) {
        if (profiles[a].steps != profiles[b].steps) return profiles[a].steps > profiles[b].steps;
        return profiles[a].client_id < profiles[b].client_id;
      });
    const uint64_t C = cap[g];
    std::vector<std::pair<uint64_t, uint64_t>> free_list{{0, C}};  // sorted (offset, length)
    struct Live {
      int64_t id;
      size_t i;
      uint64_t off, len, rel;
    };
    std::vector<Live> active;
    uint64_t t = 0, mk = 0;
    size_t qi = 0;
    while (true) {
      while (qi < q.size() && (opts->max_active == 0 || active.size() < opts->max_active)) {
        size_t h = q[qi];
        uint64_t s = opts->policy == PROTEA_POLICY_STATIC ? C : slot[h];
        size_t gap = free_list.size();
        for (size_t k = 0; k < free_list.size(); ++k)
          if (free_list[k].second >= s) {
            gap = k;
            break;
          }
        if (gap == free_list.size()) break;  // strict head-of-line blocking
        uint64_t o = free_list[gap].first;
        if (free_list[gap].second == s)
          free_list.erase(free_list.begin() + gap);
        else
          free_list[gap] = {o + s, free_list[gap].second - s};
        const protea_profile& p = profiles[h];
        active.push_back({p.client_id, h, o, s, t + p.steps});
        protea_assignment& a = res[h];
        a.client_id = p.client_id;
        a.gpu = (int32_t)g;
        a.offset = o;
        a.slot = s;
        a.admit = t;
        a.release = t + p.steps;
        a.q1024 = (uint32_t)(((unsigned __int128)s * 1024 + total_cap - 1) / total_cap);
        mk = std::max(mk, a.release);
        ++qi;
      }
      if (active.empty() && qi == q.size()) break;
      if (active.empty()) {
        set_global_error("protea_plan: head client can never be admitted on GPU " + std::to_string(g));
        return PROTEA_ERR_PLAN;
      }
      uint64_t tmin = UINT64_MAX;
      for (auto& a : active) tmin = std::min(tmin, a.rel);
      t = tmin;
      std::vector<Live> done, keep;
      for (auto& a : active) (a.rel == t ? done : keep).push_back(a);
      std::sort(done.begin(), done.end(), [](const Live& a, const Live& b) { return a.id < b.id; });
      for (auto& d : done) {
        free_list.push_back({d.off, d.len});
        std::sort(free_list.begin(), free_list.end());
        std::vector<std::pair<uint64_t, uint64_t>> merged;
        for (auto& f : free_list) {
          if (!merged.empty() && merged.back().first + merged.back().second == f.first)
            merged.back().second += f.second;
          else
            merged.push_back(f);
        }
        free_list.swap(merged);
      }
      active.swap(keep);
    }
    makespan_steps[g] = mk;
  }
  std::vector<size_t> order(n);
  for (size_t i = 0; i < n; ++i) order[i] = i;
  std::sort(order.begin(), order.end(),
            [&](size_t a, size_t b) { return profiles[a].client_id < profiles[b].client_id; });
  for (size_t i = 0; i < n; ++i) out[i] = res[order[i]];
  return PROTEA_OK;
}
