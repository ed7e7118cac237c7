// Ring and token-level load-balanced causal schedules as flat task tables,
// plus the schedule validator.
//
// Semantics follow the reference exactly (bit-exact tables are a parity
// requirement): build_ring_schedule (schedule.cpp:60-77),
// build_balanced_schedule (schedule.cpp:79-108), validate (:121-258).
// The representation differs: a Schedule is a pair of flat int32 arrays so it
// can cross the C ABI and drive the device executor without conversion.
#include "schedule_impl.h"

#include <algorithm>
#include <map>
#include <string>
#include <utility>

#include "capi_internal.h"

namespace da {

FlatSchedule make_ring(int P) {
  FlatSchedule s;
  s.workers = P;
  s.steps = P;
  for (int p = 1; p <= P; ++p) s.tasks.push_back({0, kLocal, p, p, p, 0});
  for (int t = 1; t < P; ++t) {
    for (int p = 1; p <= P; ++p) {
      if (p > t) {
        // worker p pulls kv chunk p-t (ring distance t)
        s.tasks.push_back({t, kRemote, p, p, p - t, 0});
        s.messages.push_back({t, p - t, p, kMsgKV});
      } else {
        s.tasks.push_back({t, kIdle, p, 0, 0, 0});
      }
    }
  }
  return s;
}

FlatSchedule make_balanced(int P) {
  FlatSchedule s;
  s.workers = P;
  const int half = P / 2;
  s.steps = half + 1;
  for (int p = 1; p <= P; ++p) s.tasks.push_back({0, kLocal, p, p, p, 0});
  for (int t = 1; t <= half; ++t) {
    std::vector<Task> merges;
    for (int p = 1; p <= P; ++p) {
      if (p > t) {
        s.tasks.push_back({t, kRemote, p, p, p - t, 0});
        s.messages.push_back({t, p - t, p, kMsgKV});
      } else if (P % 2 == 0 && t == half) {
        // the distance-P/2 pairs are already covered by direct workers
        s.tasks.push_back({t, kIdle, p, 0, 0, 0});
      } else {
        // helper p computes the wrap-around owner's query on its own kv
        const int owner = p + P - t;
        s.tasks.push_back({t, kRemote, p, owner, p, 0});
        s.messages.push_back({t, owner, p, kMsgQ});
        s.messages.push_back({t, p, owner, kMsgPartial});
        merges.push_back({t, kMerge, owner, 0, 0, p});
      }
    }
    s.tasks.insert(s.tasks.end(), merges.begin(), merges.end());
  }
  return s;
}

FlatSchedule make_balanced_split(int P) {
  if (P % 2 == 1) return make_balanced(P);
  FlatSchedule s;
  s.workers = P;
  const int half = P / 2;
  s.steps = half + 1;
  for (int p = 1; p <= P; ++p) s.tasks.push_back({0, kLocal, p, p, p, 0});
  for (int t = 1; t <= half; ++t) {
    std::vector<Task> merges;
    for (int p = 1; p <= P; ++p) {
      if (p > t) {
        if (t == half) {
          // direct pair (p, p - P/2) on the high half of kv chunk p - P/2
          s.tasks.push_back({t, kRemote, p, p, p - t, kPartHigh});
          s.messages.push_back({t, p - t, p, kMsgKVHalf});
        } else {
          s.tasks.push_back({t, kRemote, p, p, p - t, kPartWhole});
          s.messages.push_back({t, p - t, p, kMsgKV});
        }
      } else {
        const int owner = p + P - t;
        s.tasks.push_back({t, kRemote, p, owner, p, t == half ? kPartLow : kPartWhole});
        s.messages.push_back({t, owner, p, kMsgQ});
        s.messages.push_back({t, p, owner, kMsgPartial});
        merges.push_back({t, kMerge, owner, 0, 0, p});
      }
    }
    s.tasks.insert(s.tasks.end(), merges.begin(), merges.end());
  }
  return s;
}

static const char* kind_name(int k) {
  switch (k) {
    case kMsgKV: return "kv";
    case kMsgQ: return "q";
    case kMsgPartial: return "partial";
    case kMsgGradKV: return "grad_kv";
    case kMsgKVHalf: return "kv_half";
  }
  return "?";
}

std::vector<std::string> validate_flat(const FlatSchedule& s) {
  std::vector<std::string> errs;
  if (s.workers < 1) {
    errs.push_back("schedule has no workers");
    return errs;
  }
  const int P = s.workers;
  // (q, kv) -> times each half of the kv rows was covered (low, high)
  std::map<std::pair<int, int>, std::pair<int, int>> pairs;
  auto cover = [&](int q, int kv, int part) {
    auto& c = pairs[{q, kv}];
    if (part != kPartHigh) ++c.first;
    if (part != kPartLow) ++c.second;
  };
  struct Pending {
    int step, owner, helper;
    bool merged;
  };
  std::vector<Pending> helpers;
  std::vector<Message> open = s.messages;
  std::vector<bool> used(open.size(), false);
  auto take = [&](int step, int from, int to, int kind) {
    for (size_t i = 0; i < open.size(); ++i) {
      const Message& m = open[i];
      if (!used[i] && m.step <= step && m.from == from && m.to == to && m.kind == kind) {
        used[i] = true;
        return true;
      }
    }
    return false;
  };
  const std::string st = "step ";
  for (int t = 0; t < s.steps; ++t) {
    std::vector<int> slots(P + 1, 0);
    for (const Task& k : s.tasks) {
      if (k.step != t) continue;
      if (k.worker < 1 || k.worker > P) {
        errs.push_back(st + std::to_string(t) + ": worker id out of range");
        continue;
      }
      if (k.kind == kLocal) {
        ++slots[k.worker];
        cover(k.worker, k.worker, kPartWhole);
      } else if (k.kind == kIdle) {
        ++slots[k.worker];
      } else if (k.kind == kRemote) {
        ++slots[k.worker];
        if (k.kv_owner >= k.query_owner)
          errs.push_back(st + std::to_string(t) + ": remote task with non-causal pair (q=" +
                         std::to_string(k.query_owner) + ", kv=" + std::to_string(k.kv_owner) +
                         ")");
        const int part = k.helper;
        if (part != kPartWhole && part != kPartLow && part != kPartHigh)
          errs.push_back(st + std::to_string(t) + ": remote task with unknown kv part " +
                         std::to_string(part));
        cover(k.query_owner, k.kv_owner, part);
        if (k.worker == k.query_owner) {
          if (!take(t, k.kv_owner, k.worker, part == kPartWhole ? kMsgKV : kMsgKVHalf))
            errs.push_back(st + std::to_string(t) + ": worker " + std::to_string(k.worker) +
                           " computes on kv chunk " + std::to_string(k.kv_owner) +
                           " that was never sent");
        } else {
          if (k.worker != k.kv_owner)
            errs.push_back(st + std::to_string(t) + ": helper must use its own kv chunk");
          if (!take(t, k.query_owner, k.worker, kMsgQ))
            errs.push_back(st + std::to_string(t) + ": helper " + std::to_string(k.worker) +
                           " computes on query chunk " + std::to_string(k.query_owner) +
                           " that was never sent");
          helpers.push_back({t, k.query_owner, k.worker, false});
        }
      } else if (k.kind == kMerge) {
        auto it = std::find_if(helpers.begin(), helpers.end(), [&](const Pending& h) {
          return !h.merged && h.owner == k.worker && h.helper == k.helper && h.step <= t;
        });
        if (it == helpers.end()) {
          errs.push_back(st + std::to_string(t) + ": merge at worker " + std::to_string(k.worker) +
                         " from helper " + std::to_string(k.helper) + " has no pending partial");
        } else {
          it->merged = true;
          if (!take(t, k.helper, k.worker, kMsgPartial))
            errs.push_back(st + std::to_string(t) + ": merged partial was never sent");
        }
      } else {
        errs.push_back(st + std::to_string(t) + ": unknown task kind");
      }
    }
    for (int p = 1; p <= P; ++p)
      if (slots[p] != 1)
        errs.push_back(st + std::to_string(t) + ": worker " + std::to_string(p) + " holds " +
                       std::to_string(slots[p]) + " primary tasks (want exactly 1)");
  }
  for (const Pending& h : helpers)
    if (!h.merged)
      errs.push_back("helper partial (owner=" + std::to_string(h.owner) + ", helper=" +
                     std::to_string(h.helper) + ", step=" + std::to_string(h.step) +
                     ") is never merged");
  for (int p = 1; p <= P; ++p)
    for (int r = 1; r <= p; ++r) {
      auto it = pairs.find({p, r});
      const int lo = it == pairs.end() ? 0 : it->second.first;
      const int hi = it == pairs.end() ? 0 : it->second.second;
      const int n = std::max(lo, hi);
      if (n == 0)
        errs.push_back("pair (q=" + std::to_string(p) + ", kv=" + std::to_string(r) +
                       ") is never computed");
      else if (std::min(lo, hi) == 0)
        errs.push_back("pair (q=" + std::to_string(p) + ", kv=" + std::to_string(r) +
                       ") is only partly computed (" + (lo ? "low" : "high") + " half)");
      else if (n > 1)
        errs.push_back("pair (q=" + std::to_string(p) + ", kv=" + std::to_string(r) +
                       ") computed " + std::to_string(n) + " times");
    }
  for (const auto& kv : pairs)
    if (kv.first.second > kv.first.first)
      errs.push_back("non-causal pair (q=" + std::to_string(kv.first.first) +
                     ", kv=" + std::to_string(kv.first.second) + ") computed");
  for (size_t i = 0; i < open.size(); ++i)
    if (!used[i])
      errs.push_back("message (step=" + std::to_string(open[i].step) + ", " +
                     std::to_string(open[i].from) + "->" + std::to_string(open[i].to) + ", " +
                     kind_name(open[i].kind) + ") is never consumed");
  return errs;
}

static FlatSchedule with_grad_kv(FlatSchedule s) {
  // a GradKV message follows every direct task, in task order
  std::vector<Message> grads;
  for (const Task& k : s.tasks)
    if (k.kind == kRemote && k.worker == k.query_owner)
      grads.push_back({k.step, k.worker, k.kv_owner, kMsgGradKV});
  s.messages.insert(s.messages.end(), grads.begin(), grads.end());
  return s;
}

FlatSchedule make_ring_backward(int P) { return with_grad_kv(make_ring(P)); }
FlatSchedule make_balanced_backward(int P) { return with_grad_kv(make_balanced(P)); }
FlatSchedule make_balanced_split_backward(int P) {
  return with_grad_kv(make_balanced_split(P));
}

std::vector<std::string> validate_backward_flat(const FlatSchedule& s) {
  FlatSchedule fwd = s;
  std::vector<Message> grads;
  fwd.messages.clear();
  for (const Message& m : s.messages) (m.kind == kMsgGradKV ? grads : fwd.messages).push_back(m);
  std::vector<std::string> errs = validate_flat(fwd);
  std::vector<bool> used(grads.size(), false);
  for (const Task& k : s.tasks) {
    if (!(k.kind == kRemote && k.worker == k.query_owner)) continue;
    bool found = false;
    for (size_t i = 0; i < grads.size() && !found; ++i) {
      const Message& g = grads[i];
      if (!used[i] && g.from == k.worker && g.to == k.kv_owner && g.step >= k.step) {
        used[i] = true;
        found = true;
      }
    }
    if (!found)
      errs.push_back("step " + std::to_string(k.step) + ": gradient of pair (q=" +
                     std::to_string(k.query_owner) + ", kv=" + std::to_string(k.kv_owner) +
                     ") is never returned to its kv owner");
  }
  for (size_t i = 0; i < grads.size(); ++i)
    if (!used[i])
      errs.push_back("message (step=" + std::to_string(grads[i].step) + ", " +
                     std::to_string(grads[i].from) + "->" + std::to_string(grads[i].to) +
                     ", grad_kv) is never consumed");
  return errs;
}

}  // namespace da

extern "C" {

da_status da_schedule_build(int workers, int kind, int32_t* steps_out, int32_t* tasks,
                            int64_t* n_tasks, int32_t* messages, int64_t* n_messages) {
  if (workers < 1)
    return da::set_error(DA_ERR_CONFIG, kind == DA_SCHEDULE_RING
                                            ? "ring schedule needs at least 1 worker"
                                            : "balanced schedule needs at least 1 worker");
  da::FlatSchedule s;
  switch (kind) {
    case DA_SCHEDULE_RING: s = da::make_ring(workers); break;
    case DA_SCHEDULE_BALANCED: s = da::make_balanced(workers); break;
    case DA_SCHEDULE_RING_BWD: s = da::make_ring_backward(workers); break;
    case DA_SCHEDULE_BALANCED_BWD: s = da::make_balanced_backward(workers); break;
    case DA_SCHEDULE_BALANCED_SPLIT: s = da::make_balanced_split(workers); break;
    case DA_SCHEDULE_BALANCED_SPLIT_BWD: s = da::make_balanced_split_backward(workers); break;
    default: return da::set_error(DA_ERR_CONFIG, "unknown schedule kind");
  }
  if (steps_out) *steps_out = s.steps;
  if (tasks) {
    for (size_t i = 0; i < s.tasks.size(); ++i) {
      const da::Task& k = s.tasks[i];
      int32_t* o = tasks + 6 * i;
      o[0] = k.step; o[1] = k.kind; o[2] = k.worker; o[3] = k.query_owner; o[4] = k.kv_owner;
      o[5] = k.helper;
    }
  }
  if (messages) {
    for (size_t i = 0; i < s.messages.size(); ++i) {
      const da::Message& m = s.messages[i];
      int32_t* o = messages + 4 * i;
      o[0] = m.step; o[1] = m.from; o[2] = m.to; o[3] = m.kind;
    }
  }
  if (n_tasks) *n_tasks = static_cast<int64_t>(s.tasks.size());
  if (n_messages) *n_messages = static_cast<int64_t>(s.messages.size());
  return DA_OK;
}

static int64_t validate_impl(int workers, int32_t steps, const int32_t* tasks, int64_t n_tasks,
                             const int32_t* messages, int64_t n_messages, bool backward) {
  if (n_tasks < 0 || n_messages < 0 || (n_tasks > 0 && !tasks) || (n_messages > 0 && !messages)) {
    da::set_error(DA_ERR_CONFIG, "da_schedule_validate: bad buffers");
    return -1;
  }
  da::FlatSchedule s;
  s.workers = workers;
  s.steps = steps;
  for (int64_t i = 0; i < n_tasks; ++i) {
    const int32_t* o = tasks + 6 * i;
    s.tasks.push_back({o[0], o[1], o[2], o[3], o[4], o[5]});
  }
  for (int64_t i = 0; i < n_messages; ++i) {
    const int32_t* o = messages + 4 * i;
    s.messages.push_back({o[0], o[1], o[2], o[3]});
  }
  const auto errs = backward ? da::validate_backward_flat(s) : da::validate_flat(s);
  if (!errs.empty()) {
    std::string all;
    for (const auto& e : errs) all += (all.empty() ? "" : "\n") + e;
    da::set_error(DA_ERR_SCHEDULE, all);
  }
  return static_cast<int64_t>(errs.size());
}

int64_t da_schedule_validate(int workers, int32_t steps, const int32_t* tasks, int64_t n_tasks,
                             const int32_t* messages, int64_t n_messages) {
  return validate_impl(workers, steps, tasks, n_tasks, messages, n_messages, false);
}

int64_t da_schedule_validate_backward(int workers, int32_t steps, const int32_t* tasks,
                                      int64_t n_tasks, const int32_t* messages,
                                      int64_t n_messages) {
  return validate_impl(workers, steps, tasks, n_tasks, messages, n_messages, true);
}

}  // extern "C"
