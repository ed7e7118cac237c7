// Flat schedule representation shared by the schedule builders, the
// validator and the device executor (runtime.cu).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace da {

// TaskKind order of schedule.hpp:21
enum : int32_t { kLocal = 0, kRemote = 1, kMerge = 2, kIdle = 3 };
// PayloadKind order of schedule.hpp:45; KVHalf is the split-schedule extension
enum : int32_t { kMsgKV = 0, kMsgQ = 1, kMsgPartial = 2, kMsgGradKV = 3, kMsgKVHalf = 4 };

// Row part of a RemoteAttn task's kv chunk (carried in Task::helper, which the
// reference only uses for RescaleMerge): the whole chunk, or the low / high
// half of its rows (low = rows [0, c/2), high = [c/2, c)).
enum : int32_t { kPartWhole = 0, kPartLow = 1, kPartHigh = 2 };

struct Task {
  int32_t step, kind, worker, query_owner, kv_owner, helper;
};

struct Message {
  int32_t step, from, to, kind;
};

struct FlatSchedule {
  int workers = 0;
  int steps = 0;
  std::vector<Task> tasks;  // step-major; per step: P primaries by worker, then merges
  std::vector<Message> messages;
};

FlatSchedule make_ring(int P);
FlatSchedule make_balanced(int P);
// Balanced schedule with the even-P last step split (extension):
// at t = P/2 the reference leaves helpers 1..P/2 idle because owner p + P/2's
// direct pair (p + P/2, p) is the helper's own pair. Here helper p computes that
// pair on the LOW half of its kv rows (Q in, Partial out, merged by the owner)
// and the owner computes it on the HIGH half (KVHalf message). Identical to
// make_balanced for odd P.
FlatSchedule make_balanced_split(int P);
std::vector<std::string> validate_flat(const FlatSchedule& s);

// Backward schedules (extension: the reference's backward is ring-only,
// runtime.hpp:110). Task tables are the forward ones; message semantics:
//   KV        kv owner -> direct worker           (k, v)
//   GradKV    direct worker -> kv owner           (dk, dv contribution)
//   Q         query owner -> helper               (q, dO, lse, D bundle)
//   Partial   helper -> query owner               (dq contribution, folded by the
//                                                  RescaleMerge task in helper order)
// Ring backward = the reference run_backward order (runtime.cpp:605-651).
FlatSchedule make_ring_backward(int P);
FlatSchedule make_balanced_backward(int P);
// make_balanced_split's table with the backward messages (GradKV of the high
// half for the split direct pairs): no worker idles at t = P/2 in the backward
// either. Identical to make_balanced_backward for odd P.
FlatSchedule make_balanced_split_backward(int P);
// validate_flat's invariants plus: every direct pair (p, r) returns a GradKV
// p -> r no earlier than its step, and no other GradKV exists.
std::vector<std::string> validate_backward_flat(const FlatSchedule& s);

}  // namespace da
