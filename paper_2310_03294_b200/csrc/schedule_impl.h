// Flat schedule representation shared by the schedule builders, the
// validator and the device executor (runtime.cu).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace da {

// TaskKind order of schedule.hpp:21
enum : int32_t { kLocal = 0, kRemote = 1, kMerge = 2, kIdle = 3 };
// PayloadKind order of schedule.hpp:45
enum : int32_t { kMsgKV = 0, kMsgQ = 1, kMsgPartial = 2, kMsgGradKV = 3 };

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
std::vector<std::string> validate_flat(const FlatSchedule& s);

}  // namespace da
