// Per-rank sequence-parallel runtime (one process per GPU) in C++.
//
// Each rank holds ONE contiguous chunk and runs the reference worker's
// operation order (runtime.cpp:390-487 forward, 653-716 backward; per step:
// the primary task, then the merges in helper order) from the same flat
// schedule tables as the rest of the library (schedule.cpp).
//
// Protocol. A pass is a fixed sequence of PHASES, identical on every rank:
//   operands(0), operands(1), results(0), operands(2), results(1), ...
// operands(t) carries the messages step t consumes (KV / KVHalf / Q, and for
// the backward the (q, dO, lse, D) bundle), posted one step ahead (prefetch
// depth 1 into double-buffered slots: the reference's residency bound of 2,
// runtime.cpp:280-284, 427-431); results(t) carries what step t produces
// (Partial, GradKV, dq partials), right after its kernels. The phase lists
// are built by one pure function (program()) from the schedule, so sender
// and receiver derive every message from the same table; da_rank_protocol()
// exposes them and the CPU tests check that every send has exactly one
// matching receive in the same phase, in the same order.
//
// Transports, chosen at creation (da_rank_options.transport):
//   NCCL  each phase is one ncclGroupStart/Send/Recv/GroupEnd on a
//         high-priority side stream, after an event from the compute stream
//         (north_star: K/V prefetched with NCCL send/recv over NVLink on a
//         side stream). Identical phase order on all ranks makes the groups
//         deadlock-free. NCCL is dlopen'ed (libnccl.so.2 — in a torch
//         process the already-loaded copy), so the library loads without it.
//   IPC   the receiver's side stream pulls straight from the sender's HBM
//         (CUDA IPC mapping; copy engines, no SM), ordered by 32-bit device
//         counters (csrc/peer.cu): flags[dst] "ready" bumped on the sender's
//         compute stream after the producer of the n-th message to dst;
//         flags[world + src] "done" bumped on the receiver's side stream
//         after the n-th pull from src. Works for ranks that share one GPU.
//   NONE  no transfer: every receive slot is filled ONCE from the rank's own
//         buffer of the same kind and then reused, so the same kernels run on
//         local data — the no-communication arm that exposed communication is
//         measured against (analyzer.cpp:60-64). Results are not attention.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <array>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "capi_internal.h"
#include "kernels.h"
#include "schedule_impl.h"

extern "C" da_status da_stream_write_u32(void* stream, void* addr, uint32_t value);
extern "C" da_status da_stream_wait_u32_geq(void* stream, const void* addr, uint32_t value);

namespace da {
namespace {

// buffers a rank sends (per pass)
enum Key : int {
  kK = 0, kV, kQ, kPart, kKHi, kVHi,                    // forward
  kDOut, kLse, kDVec, kGK0, kGV0, kGK1, kGV1, kGQ0, kGQ1,  // backward
  kGKH, kGVH,                                              // backward split step: a half's GradKV
  kNumKeys
};

// receive slots (resolved to device addresses by the executor)
enum Slot : int {
  kSlotKV = 0, kSlotKVH, kSlotQ, kSlotPart, kSlotBundle, kSlotGrad, kSlotGQ, kSlotGradH
};

struct XSend {
  int dst;  // 0-based rank
  Key key;
};
struct XRecv {
  int src;  // 0-based rank
  Key key;
  Slot slot;
  int index;  // slot parity (t % 2) or the helper's worker id for partials
  int part;   // byte offset selector inside a multi-tensor slot (0..3)
};
struct Phase {
  std::vector<XSend> sends;
  std::vector<XRecv> recvs;
  bool empty() const { return sends.empty() && recvs.empty(); }
};

struct Plan {
  int action = 0;  // 0 idle, 1 local, 2 direct, 3 help
  int peer = 0;    // 1-based
  int part = kPartWhole;
  int gradkv_part = kPartWhole;  // backward: row part of the GradKV this worker receives
  std::vector<int> kv_sends, kvh_sends, q_sends, merges, gradkv_from, gradkv_to;
};

std::vector<Plan> plans_for(const FlatSchedule& s, int worker) {
  std::vector<Plan> plans(s.steps);
  for (const Task& k : s.tasks) {
    if (k.worker != worker) continue;
    Plan& p = plans[k.step];
    if (k.kind == kLocal) {
      p.action = 1;
    } else if (k.kind == kRemote) {
      p.action = k.query_owner == worker ? 2 : 3;
      p.peer = k.query_owner == worker ? k.kv_owner : k.query_owner;
      p.part = k.helper;
    } else if (k.kind == kMerge) {
      p.merges.push_back(k.helper);
    }
  }
  for (const Message& m : s.messages) {
    Plan& p = plans[m.step];
    if (m.from == worker && m.kind == kMsgKV) p.kv_sends.push_back(m.to);
    if (m.from == worker && m.kind == kMsgKVHalf) p.kvh_sends.push_back(m.to);
    if (m.from == worker && m.kind == kMsgQ) p.q_sends.push_back(m.to);
    if (m.to == worker && m.kind == kMsgGradKV) {
      p.gradkv_from.push_back(m.from);
      for (const Task& k : s.tasks)  // the sender's direct task of that step: its row part
        if (k.step == m.step && k.kind == kRemote && k.worker == m.from && k.query_owner == m.from)
          p.gradkv_part = k.helper;
    }
    if (m.from == worker && m.kind == kMsgGradKV) p.gradkv_to.push_back(m.to);
  }
  return plans;
}

// Split steps as the executors implement them (make_balanced_split): a direct
// task takes the high half of the kv rows (KVHalf payload), a helper the low
// half of its own rows, and all of a worker's half tasks and half GradKVs sit
// in one step (the half buffers and receive slots are single, not parity-
// buffered like the whole-chunk ones).
da_status check_parts(const std::vector<Plan>& plans) {
  int split_steps = 0;
  for (const Plan& p : plans) {
    if ((p.action == 2 && p.part == kPartLow) || (p.action == 3 && p.part == kPartHigh))
      return set_error(DA_ERR_UNSUPPORTED,
                       "split step: direct tasks take the high half, helpers the low half");
    if (p.part != kPartWhole || !p.kvh_sends.empty() || p.gradkv_part != kPartWhole) ++split_steps;
  }
  if (split_steps > 1)
    return set_error(DA_ERR_UNSUPPORTED, "split step: at most one split step per worker");
  return DA_OK;
}

// The pass as phases: [operands(0)], then per step t: operands(t+1), results(t).
struct Program {
  std::vector<Plan> plans;
  std::vector<Phase> operands;  // [t]
  std::vector<Phase> results;   // [t]
};

da_status forward_program(const FlatSchedule& s, int worker, Program* out) {
  Program pg;
  pg.plans = plans_for(s, worker);
  if (check_parts(pg.plans) != DA_OK) return DA_ERR_UNSUPPORTED;
  const int T = static_cast<int>(pg.plans.size());
  pg.operands.resize(T);
  pg.results.resize(T);
  for (int t = 0; t < T; ++t) {
    const Plan& p = pg.plans[t];
    Phase& op = pg.operands[t];
    for (int dst : p.kv_sends) op.sends.insert(op.sends.end(), {{dst - 1, kK}, {dst - 1, kV}});
    for (int dst : p.kvh_sends)
      op.sends.insert(op.sends.end(), {{dst - 1, kKHi}, {dst - 1, kVHi}});
    for (int dst : p.q_sends) op.sends.push_back({dst - 1, kQ});
    if (p.action == 2 && p.part == kPartHigh) {
      op.recvs.push_back({p.peer - 1, kKHi, kSlotKVH, 0, 0});
      op.recvs.push_back({p.peer - 1, kVHi, kSlotKVH, 0, 1});
    } else if (p.action == 2) {
      op.recvs.push_back({p.peer - 1, kK, kSlotKV, t % 2, 0});
      op.recvs.push_back({p.peer - 1, kV, kSlotKV, t % 2, 1});
    } else if (p.action == 3) {
      op.recvs.push_back({p.peer - 1, kQ, kSlotQ, t % 2, 0});
    }
    Phase& res = pg.results[t];
    if (p.action == 3) res.sends.push_back({p.peer - 1, kPart});
    for (int hw : p.merges) res.recvs.push_back({hw - 1, kPart, kSlotPart, hw, 0});
  }
  *out = std::move(pg);
  return DA_OK;
}

da_status backward_program(const FlatSchedule& s, int worker, Program* out) {
  Program pg;
  pg.plans = plans_for(s, worker);
  if (check_parts(pg.plans) != DA_OK) return DA_ERR_UNSUPPORTED;
  const int T = static_cast<int>(pg.plans.size());
  pg.operands.resize(T);
  pg.results.resize(T);
  for (int t = 0; t < T; ++t) {
    const Plan& p = pg.plans[t];
    // a direct pair's GradKV leaves with its task's results (the table's
    // GradKV message must sit at that step and go to the kv owner)
    const bool direct = p.action == 2;
    if (p.gradkv_to.size() != (direct ? 1u : 0u) || (direct && p.gradkv_to[0] != p.peer))
      return set_error(DA_ERR_SCHEDULE,
                       "GradKV must leave at its direct task's step, to the kv owner");
    if (p.gradkv_from.size() > 1)
      return set_error(DA_ERR_SCHEDULE, "at most one GradKV per worker and step is supported");
    Phase& op = pg.operands[t];
    for (int dst : p.kv_sends) op.sends.insert(op.sends.end(), {{dst - 1, kK}, {dst - 1, kV}});
    for (int dst : p.kvh_sends)
      op.sends.insert(op.sends.end(), {{dst - 1, kKHi}, {dst - 1, kVHi}});
    for (int dst : p.q_sends)
      op.sends.insert(op.sends.end(),
                      {{dst - 1, kQ}, {dst - 1, kDOut}, {dst - 1, kLse}, {dst - 1, kDVec}});
    if (p.action == 2 && p.part == kPartHigh) {
      op.recvs.push_back({p.peer - 1, kKHi, kSlotKVH, 0, 0});
      op.recvs.push_back({p.peer - 1, kVHi, kSlotKVH, 0, 1});
    } else if (p.action == 2) {
      op.recvs.push_back({p.peer - 1, kK, kSlotKV, t % 2, 0});
      op.recvs.push_back({p.peer - 1, kV, kSlotKV, t % 2, 1});
    } else if (p.action == 3) {
      op.recvs.push_back({p.peer - 1, kQ, kSlotBundle, t % 2, 0});
      op.recvs.push_back({p.peer - 1, kDOut, kSlotBundle, t % 2, 1});
      op.recvs.push_back({p.peer - 1, kLse, kSlotBundle, t % 2, 2});
      op.recvs.push_back({p.peer - 1, kDVec, kSlotBundle, t % 2, 3});
    }
    Phase& res = pg.results[t];
    const Key gk = (t % 2) ? kGK1 : kGK0, gv = (t % 2) ? kGV1 : kGV0;
    const Key gq = (t % 2) ? kGQ1 : kGQ0;
    if (p.action == 2 && p.part == kPartHigh)
      res.sends.insert(res.sends.end(), {{p.peer - 1, kGKH}, {p.peer - 1, kGVH}});
    else if (p.action == 2)
      res.sends.insert(res.sends.end(), {{p.peer - 1, gk}, {p.peer - 1, gv}});
    if (p.action == 3) res.sends.push_back({p.peer - 1, gq});
    // receive slots alternate by step parity: results(t) are folded during
    // step t+1 (after its kernel is queued), while results(t+1) may land
    for (int src : p.gradkv_from) {
      if (p.gradkv_part == kPartHigh) {  // the split step's half: one slot (one such step)
        res.recvs.push_back({src - 1, kGKH, kSlotGradH, 0, 0});
        res.recvs.push_back({src - 1, kGVH, kSlotGradH, 0, 1});
      } else {
        res.recvs.push_back({src - 1, gk, kSlotGrad, t % 2, 0});
        res.recvs.push_back({src - 1, gv, kSlotGrad, t % 2, 1});
      }
    }
    for (int hw : p.merges) res.recvs.push_back({hw - 1, gq, kSlotGQ, 2 * hw + t % 2, 0});
  }
  *out = std::move(pg);
  return DA_OK;
}

struct PubRecord {
  cudaIpcMemHandle_t handle;
  uint64_t offset;
  uint64_t base;
  int32_t valid;
  int32_t pad;
};

struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
  // grows the buffer; callers check the status (DA_ERR_CUDA on OOM, never a null kernel arg)
  cudaError_t ensure(size_t b) {
    if (b <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    const cudaError_t e = cudaMalloc(&p, b);
    if (e == cudaSuccess) bytes = b;
    return e;
  }
  ~Buf() {
    if (p) cudaFree(p);
  }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

// in-flight exchange: the compute stream waits on it before using received
// data or rewriting a sent buffer
struct Work {
  cudaEvent_t done = nullptr;
  std::vector<std::pair<int, uint32_t>> expect;  // IPC: peers' done counters to await
};

// NCCL entry points resolved at run time
struct Nccl {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*init_rank_config)(ncclComm_t*, int, ncclUniqueId, int, ncclConfig_t*) = nullptr;
  ncclResult_t (*destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) =
      nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  ncclResult_t (*async_error)(ncclComm_t, ncclResult_t*) = nullptr;
  bool ok = false;
};

const Nccl& nccl() {
  static Nccl n = [] {
    Nccl x;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h == nullptr) return x;
    auto sym = [&](const char* name) { return dlsym(h, name); };
    x.get_unique_id = reinterpret_cast<decltype(x.get_unique_id)>(sym("ncclGetUniqueId"));
    x.init_rank_config =
        reinterpret_cast<decltype(x.init_rank_config)>(sym("ncclCommInitRankConfig"));
    x.destroy = reinterpret_cast<decltype(x.destroy)>(sym("ncclCommDestroy"));
    x.group_start = reinterpret_cast<decltype(x.group_start)>(sym("ncclGroupStart"));
    x.group_end = reinterpret_cast<decltype(x.group_end)>(sym("ncclGroupEnd"));
    x.send = reinterpret_cast<decltype(x.send)>(sym("ncclSend"));
    x.recv = reinterpret_cast<decltype(x.recv)>(sym("ncclRecv"));
    x.error_string = reinterpret_cast<decltype(x.error_string)>(sym("ncclGetErrorString"));
    x.async_error = reinterpret_cast<decltype(x.async_error)>(sym("ncclCommGetAsyncError"));
    x.ok = x.get_unique_id && x.init_rank_config && x.destroy && x.group_start && x.group_end &&
           x.send && x.recv && x.error_string;
    return x;
  }();
  return n;
}

}  // namespace
}  // namespace da

struct da_rank {
  int rank = 0, world = 1;
  da_rank_options opts{};
  da_allgather_fn ag = nullptr;
  void* ctx = nullptr;
  cudaStream_t side = nullptr;
  // IPC
  int* flags = nullptr;                 // [2 * world]
  std::vector<int*> rflags;             // peers' flags (mapped)
  std::vector<uint32_t> sent, pulled;   // per peer
  std::map<std::pair<int, std::string>, char*> opened;   // (rank, IPC handle) -> mapped base
  std::vector<std::array<char*, da::kNumKeys>> remote;  // [rank][key]
  // NCCL
  ncclComm_t comm = nullptr;
  // this pass's own buffers per key (sends; the NONE transport's slot fill)
  std::array<const void*, da::kNumKeys> local{};
  std::array<size_t, da::kNumKeys> key_bytes{};
  std::set<void*> filled;  // NONE: receive slots already filled
  // wall-clock trace of the last pass of each kind: CUDA
  // events recorded around every task and message phase, resolved on demand
  bool trace_on = false;
  int trace_pass = 0;  // 0 forward, 1 backward (pass being recorded)
  cudaEvent_t trace_origin[2] = {nullptr, nullptr};
  struct PendingRec {
    da_trace_rec rec;
    cudaEvent_t e0, e1;  // e1 == e0 for instants
  };
  std::vector<PendingRec> pending[2];
  std::vector<cudaEvent_t> trace_events[2];  // every event of the pass, owned once (records share them)
  std::vector<da_trace_rec> resolved[2];
  bool trace_ready[2] = {false, false};
  // forward state (the rematerialisation hook: saved O / LSE, never recomputed)
  const void *q = nullptr, *k = nullptr, *v = nullptr;
  void* out = nullptr;
  float* lse = nullptr;
  int64_t h_q = 0, h_kv = 0, rows = 0;
  bool have_forward = false;
  // work buffers
  da::Buf acc, part, kv_slot[2], q_slot[2], k_lo, v_lo, k_hi, v_hi, kvh, flag;
  std::map<int, da::Buf> part_recv, gq_recv;
  da::Buf d_vec, bundle[2], g_send[2], q_send[2], g_recv[2];
  da::Buf gh_send, gh_recv, dkv_lo;  // split backward: a half's dk | dv (send / receive), low half's
};

namespace da {
namespace {

da_status ck(cudaError_t e, const char* where) {
  return e == cudaSuccess ? DA_OK : cuda_error(e, where);
}

da_status nk(ncclResult_t e, const char* where) {
  if (e == ncclSuccess) return DA_OK;
  return set_error(DA_ERR_NCCL, std::string(where) + ": " + nccl().error_string(e));
}

#define DA_TRY(x)                    \
  do {                               \
    const da_status s_ = (x);        \
    if (s_ != DA_OK) return s_;      \
  } while (0)

// NCCL's asynchronous errors (a failed peer, a broken connection) surface
// here after every pass instead of as a silent hang later
da_status nccl_async_check(da_rank* r) {
  if (r->comm == nullptr || nccl().async_error == nullptr) return DA_OK;
  ncclResult_t st = ncclSuccess;
  DA_TRY(nk(nccl().async_error(r->comm, &st), "ncclCommGetAsyncError"));
  return nk(st, "NCCL asynchronous error");
}

// NVTX range for the host-side enqueue of a pass / step (visible in nsys)
struct NvtxScope {
  explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
  ~NvtxScope() { nvtxRangePop(); }
};

// ---- tracing (no-ops unless da_rank_set_trace enabled it)
cudaEvent_t trace_event(da_rank* r, cudaStream_t st) {
  if (!r->trace_on) return nullptr;
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
  cudaEventRecord(e, st);
  r->trace_events[r->trace_pass].push_back(e);
  return e;
}

void trace_free(da_rank* r, int pass) {
  for (cudaEvent_t e : r->trace_events[pass]) cudaEventDestroy(e);
  r->trace_events[pass].clear();
  r->pending[pass].clear();
  r->trace_origin[pass] = nullptr;  // owned by trace_events
}

void trace_push(da_rank* r, int kind, int code, int step, int peer, int phase, cudaEvent_t e0,
                cudaEvent_t e1) {
  if (!r->trace_on || e0 == nullptr) return;
  da_trace_rec rec{};
  rec.kind = kind;
  rec.code = code;
  rec.step = step;
  rec.peer = peer;
  rec.phase = phase;
  r->pending[r->trace_pass].push_back({rec, e0, e1 ? e1 : e0});
}

void trace_begin(da_rank* r, int pass, cudaStream_t st) {
  trace_free(r, pass);
  r->resolved[pass].clear();
  r->trace_ready[pass] = false;
  r->trace_pass = pass;
  if (r->trace_on) r->trace_origin[pass] = trace_event(r, st);
}

using AddrRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
AddrRangeFn addr_range_fn() {
  static AddrRangeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<AddrRangeFn>(nullptr);
    return reinterpret_cast<AddrRangeFn>(p);
  }();
  return fn;
}

// IPC: publishes this pass's sendable buffers (nullptr = none) to every peer.
da_status publish(da_rank* r) {
  std::vector<PubRecord> mine(kNumKeys);
  for (int key = 0; key < kNumKeys; ++key) {
    PubRecord& rec = mine[key];
    std::memset(&rec, 0, sizeof(rec));
    if (r->local[key] == nullptr) continue;
    CUdeviceptr base = 0;
    size_t size = 0;
    const AddrRangeFn range = addr_range_fn();
    if (range == nullptr ||
        range(&base, &size, reinterpret_cast<CUdeviceptr>(r->local[key])) != CUDA_SUCCESS)
      return set_error(DA_ERR_CUDA, "da_rank: cuMemGetAddressRange failed");
    DA_TRY(ck(cudaIpcGetMemHandle(&rec.handle, reinterpret_cast<void*>(base)),
              "cudaIpcGetMemHandle"));
    rec.offset = reinterpret_cast<uint64_t>(r->local[key]) - base;
    rec.base = base;
    rec.valid = 1;
  }
  std::vector<PubRecord> all(static_cast<size_t>(kNumKeys) * r->world);
  if (r->ag(r->ctx, mine.data(), sizeof(PubRecord) * kNumKeys, all.data()) != 0)
    return set_error(DA_ERR_CONFIG, "da_rank: allgather callback failed");
  for (int src = 0; src < r->world; ++src) {
    if (src == r->rank) continue;
    for (int key = 0; key < kNumKeys; ++key) {
      const PubRecord& rec = all[static_cast<size_t>(src) * kNumKeys + key];
      if (!rec.valid) {
        r->remote[src][key] = nullptr;
        continue;
      }
      const std::string hkey(reinterpret_cast<const char*>(&rec.handle), sizeof(rec.handle));
      auto it = r->opened.find({src, hkey});
      char* mapped = nullptr;
      if (it == r->opened.end()) {
        void* p = nullptr;
        DA_TRY(ck(cudaIpcOpenMemHandle(&p, rec.handle, cudaIpcMemLazyEnablePeerAccess),
                  "cudaIpcOpenMemHandle"));
        mapped = static_cast<char*>(p);
        r->opened[{src, hkey}] = mapped;
      } else {
        mapped = it->second;
      }
      r->remote[src][key] = mapped + rec.offset;
    }
  }
  return DA_OK;
}

// Begins a pass: records this pass's buffers, publishes them (IPC).
da_status begin_pass(da_rank* r) {
  if (r->world > 1 && r->opts.transport == DA_TRANSPORT_IPC) return publish(r);
  return DA_OK;
}

// Receive-slot address of an XRecv (the executor's buffers).
using SlotFn = void* (*)(da_rank*, const XRecv&);

// Runs one phase: sends + receives of data produced (in stream order) on `cur`.
da_status exchange(da_rank* r, const Phase& ph, void* (*slot)(da_rank*, const XRecv&),
                   cudaStream_t cur, Work* w, int phase) {
  w->expect.clear();
  w->done = nullptr;
  if (ph.empty()) return DA_OK;
  const int tr = r->opts.transport;
  cudaEvent_t t_issue = nullptr;  // trace: the phase is posted (sender side)
  if (r->trace_on && tr != DA_TRANSPORT_NONE) {
    t_issue = trace_event(r, cur);
    for (const XSend& x : ph.sends) trace_push(r, 1, x.key, phase / 2, x.dst, phase, t_issue, t_issue);
  }
  if (tr == DA_TRANSPORT_NONE) {  // fill each slot once from the local buffer of that kind
    for (const XRecv& x : ph.recvs) {
      void* dst = slot(r, x);
      if (r->filled.count(dst)) continue;
      if (r->local[x.key] == nullptr)
        return set_error(DA_ERR_STATE, "da_rank: no local buffer for a no-comm slot");
      DA_TRY(ck(cudaMemcpyAsync(dst, r->local[x.key], r->key_bytes[x.key],
                                cudaMemcpyDeviceToDevice, cur),
                "no-comm fill"));
      r->filled.insert(dst);
    }
    return DA_OK;
  }
  if (tr == DA_TRANSPORT_IPC) {
    for (const XSend& s : ph.sends) {
      ++r->sent[s.dst];
      DA_TRY(da_stream_write_u32(cur, r->flags + s.dst, r->sent[s.dst]));
      w->expect.emplace_back(s.dst, r->sent[s.dst]);
    }
    if (ph.recvs.empty()) return DA_OK;
  }
  cudaEvent_t ready;
  DA_TRY(ck(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming), "event"));
  DA_TRY(ck(cudaEventRecord(ready, cur), "event record"));
  DA_TRY(ck(cudaStreamWaitEvent(r->side, ready, 0), "side wait"));
  cudaEventDestroy(ready);
  if (tr == DA_TRANSPORT_IPC) {
    for (const XRecv& x : ph.recvs) {
      const char* src = r->remote[x.src][x.key];
      if (src == nullptr)
        return set_error(DA_ERR_STATE, "da_rank: pulled buffer was not published");
      ++r->pulled[x.src];
      DA_TRY(da_stream_wait_u32_geq(r->side, r->rflags[x.src] + r->rank, r->pulled[x.src]));
      DA_TRY(ck(cudaMemcpyAsync(slot(r, x), src, r->key_bytes[x.key], cudaMemcpyDeviceToDevice,
                                r->side),
                "pull"));
      DA_TRY(da_stream_write_u32(r->side, r->flags + r->world + x.src, r->pulled[x.src]));
    }
  } else {  // NCCL: one group per phase, identical phase order on every rank
    const Nccl& n = nccl();
    DA_TRY(nk(n.group_start(), "ncclGroupStart"));
    for (const XSend& s : ph.sends)
      DA_TRY(nk(n.send(r->local[s.key], r->key_bytes[s.key], ncclUint8, s.dst, r->comm, r->side),
                "ncclSend"));
    for (const XRecv& x : ph.recvs)
      DA_TRY(nk(n.recv(slot(r, x), r->key_bytes[x.key], ncclUint8, x.src, r->comm, r->side),
                "ncclRecv"));
    DA_TRY(nk(n.group_end(), "ncclGroupEnd"));
  }
  if (t_issue != nullptr && !ph.recvs.empty()) {  // trace: the phase's data has landed
    cudaEvent_t t_arrive = trace_event(r, r->side);
    for (const XRecv& x : ph.recvs) trace_push(r, 2, x.key, phase / 2, x.src, phase, t_issue, t_arrive);
  }
  DA_TRY(ck(cudaEventCreateWithFlags(&w->done, cudaEventDisableTiming), "event"));
  return ck(cudaEventRecord(w->done, r->side), "event record");
}

da_status wait_work(da_rank* r, Work* w, cudaStream_t cur) {
  if (w->done) {
    DA_TRY(ck(cudaStreamWaitEvent(cur, w->done, 0), "wait transfers"));
    cudaEventDestroy(w->done);
    w->done = nullptr;
  }
  for (const auto& e : w->expect)
    DA_TRY(da_stream_wait_u32_geq(cur, r->rflags[e.first] + r->world + r->rank, e.second));
  w->expect.clear();
  return DA_OK;
}

da_status fwd_chunk(const void* q, const void* k, const void* v, int64_t h_q, int64_t h_kv,
                    int64_t rows_q, int64_t rows_kv, const float* acc_in, float* acc_out,
                    int mask, cudaStream_t st) {
  da_fwd_args a{};
  a.q = q;
  a.k = k;
  a.v = v;
  a.h_q = h_q;
  a.h_kv = h_kv;
  a.rows_q = rows_q;
  a.rows_kv = rows_kv;
  a.d = 128;
  const int64_t nr = h_q * rows_q;
  if (acc_in) {
    a.o_in = acc_in;
    a.m_in = acc_in + nr * 128;
    a.l_in = acc_in + nr * 129;
  }
  a.o_acc = acc_out;
  a.m_acc = acc_out + nr * 128;
  a.l_acc = acc_out + nr * 129;
  a.mask = mask;
  return da_attn_fwd_chunk(&a, st);
}

da_status bwd_chunk(const void* q, const void* k, const void* v, const void* d_out,
                    const float* lse, const float* d_vec, int64_t h_q, int64_t h_kv, int64_t rows,
                    int64_t rows_kv, float* dq, float* dk, float* dv, bool accumulate_kv, int mask,
                    bool deterministic, cudaStream_t st) {
  da_bwd_args a{};
  a.q = q;
  a.k = k;
  a.v = v;
  a.d_out = d_out;
  a.lse = lse;
  a.d_vec = d_vec;
  a.h_q = h_q;
  a.h_kv = h_kv;
  a.rows_q = rows;
  a.rows_kv = rows_kv;
  a.d = 128;
  a.dq_acc = dq;
  a.dk_acc = dk;
  a.dv_acc = dv;
  a.accumulate_kv = accumulate_kv ? 1 : 0;
  a.mask = mask;
  a.deterministic = deterministic ? 1 : 0;
  return da_attn_bwd_chunk(&a, st);
}

cudaError_t pack_rows(const void* src, void* dst, int64_t h, int64_t rows, int64_t r0, int64_t n,
                      cudaStream_t st) {
  const size_t pitch = static_cast<size_t>(rows) * 256, width = static_cast<size_t>(n) * 256;
  return cudaMemcpy2DAsync(dst, width, static_cast<const char*>(src) + r0 * 256, pitch, width, h,
                           cudaMemcpyDeviceToDevice, st);
}

void count(da_counters& c, int kind, int64_t scalars) {
  switch (kind) {
    case kMsgKV: c.kv_scalars += scalars; ++c.kv_messages; break;
    case kMsgQ: c.q_scalars += scalars; ++c.q_messages; break;
    case kMsgPartial: c.partial_scalars += scalars; ++c.partial_messages; break;
    case kMsgGradKV: c.grad_scalars += scalars; ++c.grad_messages; break;
  }
}

FlatSchedule forward_table(int kind, int P, bool* ok) {
  *ok = true;
  if (kind == DA_SCHEDULE_RING) return make_ring(P);
  if (kind == DA_SCHEDULE_BALANCED) return make_balanced(P);
  if (kind == DA_SCHEDULE_BALANCED_SPLIT) return make_balanced_split(P);
  *ok = false;
  return FlatSchedule{};
}

FlatSchedule backward_table(int kind, int P, bool* ok) {
  *ok = true;
  if (kind == DA_SCHEDULE_RING_BWD || kind == DA_SCHEDULE_RING) return make_ring_backward(P);
  if (kind == DA_SCHEDULE_BALANCED_BWD || kind == DA_SCHEDULE_BALANCED)
    return make_balanced_backward(P);
  if (kind == DA_SCHEDULE_BALANCED_SPLIT_BWD || kind == DA_SCHEDULE_BALANCED_SPLIT)
    return make_balanced_split_backward(P);
  *ok = false;
  return FlatSchedule{};
}

// receive-slot resolution of the two passes
void* fwd_slot(da_rank* r, const XRecv& x) {
  const size_t kv_b = static_cast<size_t>(r->h_kv) * r->rows * 256;
  const size_t half_b = r->key_bytes[kKHi];
  switch (x.slot) {
    case kSlotKV: return r->kv_slot[x.index].as<char>() + x.part * kv_b;
    case kSlotKVH: return r->kvh.as<char>() + x.part * half_b;
    case kSlotQ: return r->q_slot[x.index].p;
    case kSlotPart: return r->part_recv[x.index].p;
    default: return nullptr;
  }
}

void* bwd_slot(da_rank* r, const XRecv& x) {
  const int64_t nq = r->h_q * r->rows, nkv = r->h_kv * r->rows;
  const size_t kv_b = static_cast<size_t>(nkv) * 256, q_b = static_cast<size_t>(nq) * 256;
  const size_t g_kv = static_cast<size_t>(nkv) * 128 * 4;
  const size_t bundle_off[4] = {0, q_b, 2 * q_b, 2 * q_b + static_cast<size_t>(nq) * 4};
  switch (x.slot) {
    case kSlotKV: return r->kv_slot[x.index].as<char>() + x.part * kv_b;
    case kSlotBundle: return r->bundle[x.index].as<char>() + bundle_off[x.part];
    case kSlotGrad: return r->g_recv[x.index].as<char>() + x.part * g_kv;
    case kSlotGQ: return r->gq_recv[x.index].p;
    case kSlotKVH: return r->kvh.as<char>() + x.part * r->key_bytes[kKHi];
    case kSlotGradH: return r->gh_recv.as<char>() + x.part * r->key_bytes[kGKH];
    default: return nullptr;
  }
}

}  // namespace
}  // namespace da

using namespace da;

extern "C" {

da_status da_rank_create_ex(int rank, int world, da_allgather_fn fn, void* ctx,
                            const da_rank_options* opts, da_rank** out) {
  if (out == nullptr || fn == nullptr) return set_error(DA_ERR_CONFIG, "da_rank_create: null");
  if (world < 1 || rank < 0 || rank >= world)
    return set_error(DA_ERR_CONFIG, "da_rank_create: bad rank / world");
  std::unique_ptr<da_rank> r(new da_rank());
  r->rank = rank;
  r->world = world;
  if (opts) r->opts = *opts;
  const int tr = r->opts.transport;
  if (tr != DA_TRANSPORT_IPC && tr != DA_TRANSPORT_NCCL && tr != DA_TRANSPORT_NONE)
    return set_error(DA_ERR_CONFIG, "da_rank_create: unknown transport");
  r->ag = fn;
  r->ctx = ctx;
  r->sent.assign(world, 0);
  r->pulled.assign(world, 0);
  r->remote.assign(world, {});
  for (auto& a : r->remote) a.fill(nullptr);
  int lo = 0, hi = 0;  // transfers overtake kernels on the side stream
  DA_TRY(ck(cudaDeviceGetStreamPriorityRange(&lo, &hi), "stream priorities"));
  DA_TRY(ck(cudaStreamCreateWithPriority(&r->side, cudaStreamNonBlocking, hi), "side stream"));
  if (tr == DA_TRANSPORT_IPC) {
    DA_TRY(ck(cudaMalloc(&r->flags, sizeof(int) * 2 * world), "flags"));
    DA_TRY(ck(cudaMemset(r->flags, 0, sizeof(int) * 2 * world), "flags"));
    r->rflags.assign(world, r->flags);
    std::vector<PubRecord> mine(1), all(world);
    std::memset(mine.data(), 0, sizeof(PubRecord));
    DA_TRY(ck(cudaIpcGetMemHandle(&mine[0].handle, r->flags), "cudaIpcGetMemHandle(flags)"));
    mine[0].valid = 1;
    if (world > 1) {
      if (fn(ctx, mine.data(), sizeof(PubRecord), all.data()) != 0)
        return set_error(DA_ERR_CONFIG, "da_rank_create: allgather callback failed");
      for (int s = 0; s < world; ++s) {
        if (s == rank) continue;
        void* p = nullptr;
        DA_TRY(ck(cudaIpcOpenMemHandle(&p, all[s].handle, cudaIpcMemLazyEnablePeerAccess),
                  "cudaIpcOpenMemHandle(flags)"));
        r->rflags[s] = static_cast<int*>(p);
      }
    }
  } else if (tr == DA_TRANSPORT_NCCL) {
    const Nccl& n = nccl();
    if (!n.ok) return set_error(DA_ERR_NCCL, "da_rank_create: libnccl.so.2 not loadable");
    ncclUniqueId id;
    std::memset(&id, 0, sizeof(id));
    if (rank == 0) DA_TRY(nk(n.get_unique_id(&id), "ncclGetUniqueId"));
    std::vector<ncclUniqueId> ids(world);
    if (fn(ctx, &id, sizeof(id), ids.data()) != 0)
      return set_error(DA_ERR_CONFIG, "da_rank_create: allgather callback failed");
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    if (r->opts.nccl_max_ctas > 0) {
      cfg.minCTAs = 1;
      cfg.maxCTAs = r->opts.nccl_max_ctas;
    }
    DA_TRY(nk(n.init_rank_config(&r->comm, world, ids[0], rank, &cfg), "ncclCommInitRankConfig"));
  }
  *out = r.release();
  return DA_OK;
}

da_status da_rank_create(int rank, int world, da_allgather_fn fn, void* ctx, da_rank** out) {
  da_rank_options o{};
  o.transport = DA_TRANSPORT_IPC;
  return da_rank_create_ex(rank, world, fn, ctx, &o, out);
}

void da_rank_destroy(da_rank* r) {
  if (r == nullptr) return;
  cudaDeviceSynchronize();
  for (int pass = 0; pass < 2; ++pass) trace_free(r, pass);
  if (r->comm) nccl().destroy(r->comm);
  for (auto& kv : r->opened) cudaIpcCloseMemHandle(kv.second);
  for (int s = 0; s < static_cast<int>(r->rflags.size()); ++s)
    if (r->rflags[s] != r->flags) cudaIpcCloseMemHandle(r->rflags[s]);
  if (r->flags) cudaFree(r->flags);
  if (r->side) cudaStreamDestroy(r->side);
  delete r;
}

static da_status rank_forward_flat(da_rank* r, const FlatSchedule& sch, const void* q,
                                   const void* k, const void* v, int64_t h_q, int64_t h_kv,
                                   int64_t rows, void* out, float* lse, da_counters* counters,
                                   void* stream) {
  NvtxScope range("da_rank_forward");
  DA_TRY(nccl_async_check(r));
  if (h_q < 1 || h_kv < 1 || h_q % h_kv != 0 || rows < 1)
    return set_error(DA_ERR_SHAPE, "da_rank_forward: bad shape");
  const int P = r->world, w = r->rank + 1;
  if (sch.workers != P)
    return set_error(DA_ERR_SCHEDULE, "schedule worker count does not match the world size");
  const auto errs = validate_flat(sch);
  if (!errs.empty()) return set_error(DA_ERR_SCHEDULE, "invalid schedule: " + errs.front());
  Program pg;
  DA_TRY(forward_program(sch, w, &pg));
  const auto& plans = pg.plans;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  r->h_q = h_q;
  r->h_kv = h_kv;
  r->rows = rows;
  r->have_forward = false;
  const int64_t nq = h_q * rows, nkv = h_kv * rows;
  const size_t acc_f = static_cast<size_t>(nq) * 130;  // o | m | l
  const size_t kv_b = static_cast<size_t>(nkv) * 256, q_b = static_cast<size_t>(nq) * 256;
  DA_TRY(ck(r->acc.ensure(acc_f * 4), "da_rank workspace"));
  DA_TRY(ck(r->part.ensure(acc_f * 4), "da_rank workspace"));
  for (int i = 0; i < 2; ++i) {
    DA_TRY(ck(r->kv_slot[i].ensure(2 * kv_b), "da_rank workspace"));
    DA_TRY(ck(r->q_slot[i].ensure(q_b), "da_rank workspace"));
  }
  DA_TRY(ck(r->flag.ensure(sizeof(int)), "da_rank workspace"));
  const int64_t lo = rows / 2, hi = rows - lo;
  bool split = false;
  for (const Plan& p : plans) split = split || p.part != kPartWhole || !p.kvh_sends.empty();
  if (split) {
    DA_TRY(ck(r->k_lo.ensure(static_cast<size_t>(h_kv) * (lo > 0 ? lo : 1) * 256),
              "da_rank workspace"));
    DA_TRY(ck(r->v_lo.ensure(static_cast<size_t>(h_kv) * (lo > 0 ? lo : 1) * 256),
              "da_rank workspace"));
    DA_TRY(ck(r->k_hi.ensure(static_cast<size_t>(h_kv) * hi * 256), "da_rank workspace"));
    DA_TRY(ck(r->v_hi.ensure(static_cast<size_t>(h_kv) * hi * 256), "da_rank workspace"));
    DA_TRY(ck(r->kvh.ensure(2 * static_cast<size_t>(h_kv) * hi * 256), "da_rank workspace"));
    cudaError_t e = cudaSuccess;
    if (lo > 0) e = pack_rows(k, r->k_lo.p, h_kv, rows, 0, lo, st);
    if (e == cudaSuccess && lo > 0) e = pack_rows(v, r->v_lo.p, h_kv, rows, 0, lo, st);
    if (e == cudaSuccess) e = pack_rows(k, r->k_hi.p, h_kv, rows, lo, hi, st);
    if (e == cudaSuccess) e = pack_rows(v, r->v_hi.p, h_kv, rows, lo, hi, st);
    DA_TRY(ck(e, "da_rank_forward split pack"));
  }
  for (const Plan& p : plans)
    for (int hw : p.merges) DA_TRY(ck(r->part_recv[hw].ensure(acc_f * 4), "da_rank workspace"));
  r->local.fill(nullptr);
  r->key_bytes.fill(0);
  r->local[kK] = k;
  r->local[kV] = v;
  r->local[kQ] = q;
  r->local[kPart] = r->part.p;
  r->key_bytes[kK] = r->key_bytes[kV] = kv_b;
  r->key_bytes[kQ] = q_b;
  r->key_bytes[kPart] = acc_f * 4;
  if (split) {
    r->local[kKHi] = r->k_hi.p;
    r->local[kVHi] = r->v_hi.p;
    r->key_bytes[kKHi] = r->key_bytes[kVHi] = static_cast<size_t>(h_kv) * hi * 256;
  }
  if (P > 1) DA_TRY(begin_pass(r));

  da_counters c{};
  float* acc = r->acc.as<float>();
  bool have_acc = false;
  Work pending, part_work;
  bool part_pending = false;
  int held = 0;
  const int T = static_cast<int>(plans.size());
  trace_begin(r, 0, st);
  if (P > 1) DA_TRY(exchange(r, pg.operands[0], fwd_slot, st, &pending, 0));
  for (int t = 0; t < T; ++t) {
    const Plan& p = plans[t];
    Work next;
    const bool has_next = t + 1 < T;
    if (has_next && P > 1)  // prefetch: overlaps this step's compute
      DA_TRY(exchange(r, pg.operands[t + 1], fwd_slot, st, &next, 2 * (t + 1)));
    DA_TRY(wait_work(r, &pending, st));
    const int cur_held = (p.action >= 2 ? 1 : 0) + (has_next && plans[t + 1].action >= 2 ? 1 : 0);
    held = cur_held > held ? cur_held : held;
    cudaEvent_t te0 = p.action ? trace_event(r, st) : nullptr;
    if (p.action == 1) {
      ++c.attention_kernel_calls;
      DA_TRY(fwd_chunk(q, k, v, h_q, h_kv, rows, rows, have_acc ? acc : nullptr, acc,
                       DA_MASK_DIAGONAL, st));
      have_acc = true;
    } else if (p.action == 2) {
      ++c.attention_kernel_calls;
      const bool half = p.part == kPartHigh;
      const char* ks = half ? r->kvh.as<char>() : r->kv_slot[t % 2].as<char>();
      const char* vs = half ? ks + static_cast<size_t>(h_kv) * hi * 256 : ks + kv_b;
      count(c, kMsgKV, 2 * (half ? h_kv * hi : nkv) * 128);
      DA_TRY(fwd_chunk(q, ks, vs, h_q, h_kv, rows, half ? hi : rows, have_acc ? acc : nullptr,
                       acc, DA_MASK_FULL, st));
      have_acc = true;
    } else if (p.action == 3) {
      ++c.attention_kernel_calls;
      count(c, kMsgQ, nq * 128);
      if (part_pending) DA_TRY(wait_work(r, &part_work, st));  // previous partial has left
      part_pending = false;
      const bool low = p.part == kPartLow;
      DA_TRY(fwd_chunk(r->q_slot[t % 2].p, low ? r->k_lo.p : k, low ? r->v_lo.p : v, h_q, h_kv,
                       rows, low ? lo : rows, nullptr, r->part.as<float>(), DA_MASK_FULL, st));
    }
    if (p.action) trace_push(r, 0, p.action, t, p.action == 1 ? w : p.peer, -1, te0,
                             trace_event(r, st));
    Work res;
    if (P > 1) DA_TRY(exchange(r, pg.results[t], fwd_slot, st, &res, 2 * t + 1));
    if (p.action == 3 && p.merges.empty()) {
      part_work = res;  // the partial's send completes before r->part is rewritten
      part_pending = true;
    } else {
      DA_TRY(wait_work(r, &res, st));  // partials from this step's helpers have landed
      part_pending = false;
    }
    for (int hw : p.merges) {  // in helper order (runtime.cpp:322-328, 468-474)
      count(c, kMsgPartial, nq * 130);
      const float* b = r->part_recv[hw].as<float>();
      cudaEvent_t me0 = trace_event(r, st);
      DA_TRY(ck(launch_merge(acc, acc + nq * 128, acc + nq * 129, b, b + nq * 128, b + nq * 129,
                             acc, acc + nq * 128, acc + nq * 129, nq, st),
                "da_rank_forward merge"));
      trace_push(r, 0, 4, t, hw, -1, me0, trace_event(r, st));
    }
    pending = next;
  }
  if (part_pending) DA_TRY(wait_work(r, &part_work, st));
  DA_TRY(ck(cudaMemsetAsync(r->flag.p, 0, sizeof(int), st), "flag"));
  DA_TRY(ck(launch_finalize(acc, acc + nq * 128, acc + nq * 129, out, lse, r->flag.as<int>(), nq,
                            st),
            "da_rank_forward finalize"));
  r->q = q;
  r->k = k;
  r->v = v;
  r->out = out;
  r->lse = lse;
  r->have_forward = true;
  c.max_remote_chunks_held = held;
  if (counters) *counters = c;
  DA_TRY(nccl_async_check(r));
  if (r->opts.transport == DA_TRANSPORT_NONE) return DA_OK;  // garbage-in by design
  return da_check_degenerate(r->flag.as<int>(), stream);
}

static da_status rank_backward_flat(da_rank* r, const FlatSchedule& sch, const void* d_out,
                                    float* dq, float* dk, float* dv, da_counters* counters,
                                    void* stream) {
  NvtxScope range("da_rank_backward");
  DA_TRY(nccl_async_check(r));
  if (!r->have_forward)
    return set_error(DA_ERR_STATE, "run_backward requires forward output and logsumexp");
  if (d_out == nullptr) return set_error(DA_ERR_STATE, "run_backward requires d_out");
  const int P = r->world, w = r->rank + 1;
  if (sch.workers != P)
    return set_error(DA_ERR_SCHEDULE, "schedule worker count does not match the world size");
  const auto errs = validate_backward_flat(sch);
  if (!errs.empty()) return set_error(DA_ERR_SCHEDULE, "invalid schedule: " + errs.front());
  Program pg;
  DA_TRY(backward_program(sch, w, &pg));
  const auto& plans = pg.plans;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool det = r->opts.deterministic != 0;
  const int64_t h_q = r->h_q, h_kv = r->h_kv, rows = r->rows;
  const int64_t nq = h_q * rows, nkv = h_kv * rows;
  const size_t kv_b = static_cast<size_t>(nkv) * 256, q_b = static_cast<size_t>(nq) * 256;
  const size_t g_kv = static_cast<size_t>(nkv) * 128 * 4, g_q = static_cast<size_t>(nq) * 128 * 4;
  const size_t bundle_b = 2 * q_b + 2 * static_cast<size_t>(nq) * 4;  // q | d_out | lse | D
  DA_TRY(ck(r->d_vec.ensure(static_cast<size_t>(nq) * 4), "da_rank workspace"));
  for (int i = 0; i < 2; ++i) {
    DA_TRY(ck(r->kv_slot[i].ensure(2 * kv_b), "da_rank workspace"));
    DA_TRY(ck(r->bundle[i].ensure(bundle_b), "da_rank workspace"));
    DA_TRY(ck(r->g_send[i].ensure(2 * g_kv), "da_rank workspace"));
    DA_TRY(ck(r->q_send[i].ensure(g_q), "da_rank workspace"));
  }
  for (int i = 0; i < 2; ++i) DA_TRY(ck(r->g_recv[i].ensure(2 * g_kv), "da_rank workspace"));
  for (size_t t = 0; t < plans.size(); ++t)
    for (int hw : plans[t].merges)
      DA_TRY(ck(r->gq_recv[2 * hw + static_cast<int>(t % 2)].ensure(g_q), "da_rank workspace"));
  // split step (balanced_split backward): kv row halves lo = [0, c/2), hi = [c/2, c)
  const int64_t lo = rows / 2, hi = rows - lo;
  bool split = false;
  for (const Plan& p : plans)
    split = split || p.part != kPartWhole || !p.kvh_sends.empty() || p.gradkv_part != kPartWhole;
  const size_t half_b = static_cast<size_t>(h_kv) * hi * 256;      // bf16 k or v half
  const size_t gh_b = static_cast<size_t>(h_kv) * hi * 128 * 4;    // fp32 dk or dv half
  const size_t glo_b = static_cast<size_t>(h_kv) * (lo > 0 ? lo : 1) * 128 * 4;
  if (split) {
    DA_TRY(ck(r->k_lo.ensure(static_cast<size_t>(h_kv) * (lo > 0 ? lo : 1) * 256),
              "da_rank workspace"));
    DA_TRY(ck(r->v_lo.ensure(static_cast<size_t>(h_kv) * (lo > 0 ? lo : 1) * 256),
              "da_rank workspace"));
    DA_TRY(ck(r->k_hi.ensure(half_b), "da_rank workspace"));
    DA_TRY(ck(r->v_hi.ensure(half_b), "da_rank workspace"));
    DA_TRY(ck(r->kvh.ensure(2 * half_b), "da_rank workspace"));
    DA_TRY(ck(r->gh_send.ensure(2 * gh_b), "da_rank workspace"));
    DA_TRY(ck(r->gh_recv.ensure(2 * gh_b), "da_rank workspace"));
    DA_TRY(ck(r->dkv_lo.ensure(2 * glo_b), "da_rank workspace"));
    cudaError_t e = cudaSuccess;  // this pass's k / v (a restored layer may differ)
    if (lo > 0) e = pack_rows(r->k, r->k_lo.p, h_kv, rows, 0, lo, st);
    if (e == cudaSuccess && lo > 0) e = pack_rows(r->v, r->v_lo.p, h_kv, rows, 0, lo, st);
    if (e == cudaSuccess) e = pack_rows(r->k, r->k_hi.p, h_kv, rows, lo, hi, st);
    if (e == cudaSuccess) e = pack_rows(r->v, r->v_hi.p, h_kv, rows, lo, hi, st);
    DA_TRY(ck(e, "da_rank_backward split pack"));
  }
  DA_TRY(ck(cudaMemsetAsync(dq, 0, g_q, st), "dq zero"));
  DA_TRY(ck(cudaMemsetAsync(dk, 0, g_kv, st), "dk zero"));
  DA_TRY(ck(cudaMemsetAsync(dv, 0, g_kv, st), "dv zero"));
  DA_TRY(ck(launch_bwd_preprocess(d_out, r->out, r->d_vec.as<float>(), nq, st), "preprocess"));
  r->local.fill(nullptr);
  r->key_bytes.fill(0);
  r->local[kK] = r->k;
  r->local[kV] = r->v;
  r->local[kQ] = r->q;
  r->local[kDOut] = d_out;
  r->local[kLse] = r->lse;
  r->local[kDVec] = r->d_vec.p;
  r->local[kGK0] = r->g_send[0].p;
  r->local[kGV0] = r->g_send[0].as<char>() + g_kv;
  r->local[kGK1] = r->g_send[1].p;
  r->local[kGV1] = r->g_send[1].as<char>() + g_kv;
  r->local[kGQ0] = r->q_send[0].p;
  r->local[kGQ1] = r->q_send[1].p;
  r->key_bytes[kK] = r->key_bytes[kV] = kv_b;
  r->key_bytes[kQ] = r->key_bytes[kDOut] = q_b;
  r->key_bytes[kLse] = r->key_bytes[kDVec] = static_cast<size_t>(nq) * 4;
  for (Key key : {kGK0, kGV0, kGK1, kGV1}) r->key_bytes[key] = g_kv;
  r->key_bytes[kGQ0] = r->key_bytes[kGQ1] = g_q;
  if (split) {
    r->local[kKHi] = r->k_hi.p;
    r->local[kVHi] = r->v_hi.p;
    r->local[kGKH] = r->gh_send.p;
    r->local[kGVH] = r->gh_send.as<char>() + gh_b;
    r->key_bytes[kKHi] = r->key_bytes[kVHi] = half_b;
    r->key_bytes[kGKH] = r->key_bytes[kGVH] = gh_b;
  }
  if (P > 1) DA_TRY(begin_pass(r));

  da_counters c{};
  Work pending;
  const int T = static_cast<int>(plans.size());
  Work res_w[2];
  // waits for step tt's results phase and folds what it brought (GradKV into
  // dk / dv, helpers' dq partials into dq), in schedule order
  auto complete = [&](int tt) -> da_status {
    const Plan& pp = plans[tt];
    DA_TRY(wait_work(r, &res_w[tt % 2], st));
    cudaEvent_t fe0 =
        (!pp.gradkv_from.empty() || !pp.merges.empty()) ? trace_event(r, st) : nullptr;
    if (!pp.gradkv_from.empty() && pp.gradkv_part == kPartHigh) {  // rows [lo, rows)
      count(c, kMsgGradKV, 2 * h_kv * hi * 128);
      const float* g = r->gh_recv.as<float>();
      DA_TRY(ck(launch_add_rows(dk, g, h_kv, rows, lo, hi, st), "GradKV fold"));
      DA_TRY(ck(launch_add_rows(dv, g + h_kv * hi * 128, h_kv, rows, lo, hi, st), "GradKV fold"));
    } else if (!pp.gradkv_from.empty()) {
      count(c, kMsgGradKV, 2 * nkv * 128);
      const float* g = r->g_recv[tt % 2].as<float>();
      DA_TRY(ck(launch_add(dk, g, nkv * 128, st), "GradKV fold"));
      DA_TRY(ck(launch_add(dv, g + nkv * 128, nkv * 128, st), "GradKV fold"));
    }
    for (int hw : pp.merges) {
      c.partial_scalars += nq * 128;
      ++c.partial_messages;
      DA_TRY(ck(launch_add(dq, r->gq_recv[2 * hw + tt % 2].as<float>(), nq * 128, st),
                "dq fold"));
    }
    if (fe0)
      trace_push(r, 0, 5, tt, pp.gradkv_from.empty() ? pp.merges.front() : pp.gradkv_from.front(),
                 -1, fe0, trace_event(r, st));
    return DA_OK;
  };
  trace_begin(r, 1, st);
  if (P > 1) DA_TRY(exchange(r, pg.operands[0], bwd_slot, st, &pending, 0));
  for (int t = 0; t < T; ++t) {
    const Plan& p = plans[t];
    Work next;
    if (t + 1 < T && P > 1)
      DA_TRY(exchange(r, pg.operands[t + 1], bwd_slot, st, &next, 2 * (t + 1)));
    DA_TRY(wait_work(r, &pending, st));
    cudaEvent_t te0 = p.action ? trace_event(r, st) : nullptr;
    if (p.action == 1) {
      ++c.attention_kernel_calls;
      DA_TRY(bwd_chunk(r->q, r->k, r->v, d_out, r->lse, r->d_vec.as<float>(), h_q, h_kv, rows,
                       rows, dq, dk, dv, true, DA_MASK_DIAGONAL, det, st));
    } else if (p.action == 2 && p.part == kPartHigh) {  // split step: high half of the kv rows
      ++c.attention_kernel_calls;
      count(c, kMsgKV, 2 * h_kv * hi * 128);
      const char* ks = r->kvh.as<char>();
      float* gk = r->gh_send.as<float>();
      DA_TRY(bwd_chunk(r->q, ks, ks + half_b, d_out, r->lse, r->d_vec.as<float>(), h_q, h_kv,
                       rows, hi, dq, gk, gk + h_kv * hi * 128, false, DA_MASK_FULL, det, st));
    } else if (p.action == 3 && p.part == kPartLow) {  // split step: low half of my kv rows
      ++c.attention_kernel_calls;
      c.q_scalars += rows * (2 * 128 + 2) * h_q;
      ++c.q_messages;
      const char* b = r->bundle[t % 2].as<char>();
      float* gq = r->q_send[t % 2].as<float>();
      float* gl = r->dkv_lo.as<float>();
      DA_TRY(ck(cudaMemsetAsync(gq, 0, g_q, st), "gq zero"));
      if (lo > 0) {
        DA_TRY(bwd_chunk(b, r->k_lo.p, r->v_lo.p, b + q_b,
                         reinterpret_cast<const float*>(b + 2 * q_b),
                         reinterpret_cast<const float*>(b + 2 * q_b + nq * 4), h_q, h_kv, rows, lo,
                         gq, gl, gl + h_kv * lo * 128, false, DA_MASK_FULL, det, st));
        DA_TRY(ck(launch_add_rows(dk, gl, h_kv, rows, 0, lo, st), "low-half fold"));
        DA_TRY(ck(launch_add_rows(dv, gl + h_kv * lo * 128, h_kv, rows, 0, lo, st),
                  "low-half fold"));
      }
    } else if (p.action == 2) {
      ++c.attention_kernel_calls;
      count(c, kMsgKV, 2 * nkv * 128);
      const char* ks = r->kv_slot[t % 2].as<char>();
      float* gk = r->g_send[t % 2].as<float>();
      DA_TRY(bwd_chunk(r->q, ks, ks + kv_b, d_out, r->lse, r->d_vec.as<float>(), h_q, h_kv, rows,
                       rows, dq, gk, gk + nkv * 128, false, DA_MASK_FULL, det, st));
    } else if (p.action == 3) {
      ++c.attention_kernel_calls;
      c.q_scalars += rows * (2 * 128 + 2) * h_q;
      ++c.q_messages;
      const char* b = r->bundle[t % 2].as<char>();
      float* gq = r->q_send[t % 2].as<float>();
      DA_TRY(ck(cudaMemsetAsync(gq, 0, g_q, st), "gq zero"));
      DA_TRY(bwd_chunk(b, r->k, r->v, b + q_b, reinterpret_cast<const float*>(b + 2 * q_b),
                       reinterpret_cast<const float*>(b + 2 * q_b + nq * 4), h_q, h_kv, rows, rows,
                       gq, dk, dv, true, DA_MASK_FULL, det, st));
    }
    if (p.action) trace_push(r, 0, p.action, t, p.action == 1 ? w : p.peer, -1, te0,
                             trace_event(r, st));
    // results leave right after their kernels. They are completed one step
    // later (after step t+1's kernel is queued): the transfer of GradKV / dq
    // partials overlaps the next kernel instead of stalling the compute
    // stream, and the send buffers (double-buffered) are retired before
    // step t+2 rewrites them. Folds keep the ascending-sender order.
    if (P > 1) DA_TRY(exchange(r, pg.results[t], bwd_slot, st, &res_w[t % 2], 2 * t + 1));
    if (t >= 1) DA_TRY(complete(t - 1));
    pending = next;
  }
  if (T >= 1) DA_TRY(complete(T - 1));
  if (counters) *counters = c;
  return nccl_async_check(r);
}

// Re-installs a saved forward state (q, k, v, O, LSE of an earlier forward
// pass) for the next da_rank_backward: the rematerialisation hook of a
// checkpointed multi-layer model (ckptplan.cpp:198-206), whose attention
// backward runs with the saved O / LSE of ITS layer, never a recompute.
da_status da_rank_restore(da_rank* r, const void* q, const void* k, const void* v, void* out,
                          float* lse, int64_t h_q, int64_t h_kv, int64_t rows) {
  if (r == nullptr) return set_error(DA_ERR_CONFIG, "da_rank_restore: null runtime");
  if (!q || !k || !v || !out || !lse)
    return set_error(DA_ERR_STATE, "run_backward requires forward output and logsumexp");
  if (h_q < 1 || h_kv < 1 || h_q % h_kv != 0 || rows < 1)
    return set_error(DA_ERR_SHAPE, "da_rank_restore: bad shape");
  r->q = q;
  r->k = k;
  r->v = v;
  r->out = out;
  r->lse = lse;
  r->h_q = h_q;
  r->h_kv = h_kv;
  r->rows = rows;
  r->have_forward = true;
  return DA_OK;
}

static FlatSchedule rank_table(int workers, int32_t steps, const int32_t* tasks,
                               int64_t n_tasks, const int32_t* messages, int64_t n_messages) {
  FlatSchedule f;
  f.workers = workers;
  f.steps = steps;
  for (int64_t i = 0; tasks && i < n_tasks; ++i) {
    const int32_t* o = tasks + 6 * i;
    f.tasks.push_back({o[0], o[1], o[2], o[3], o[4], o[5]});
  }
  for (int64_t i = 0; messages && i < n_messages; ++i) {
    const int32_t* o = messages + 4 * i;
    f.messages.push_back({o[0], o[1], o[2], o[3]});
  }
  return f;
}

da_status da_rank_forward(da_rank* r, int schedule_kind, const void* q, const void* k,
                          const void* v, int64_t h_q, int64_t h_kv, int64_t rows, void* out,
                          float* lse, da_counters* counters, void* stream) {
  if (r == nullptr) return set_error(DA_ERR_CONFIG, "da_rank_forward: null runtime");
  bool ok = false;
  const FlatSchedule sch = forward_table(schedule_kind, r->world, &ok);
  if (!ok) return set_error(DA_ERR_CONFIG, "da_rank_forward: unknown schedule kind");
  return rank_forward_flat(r, sch, q, k, v, h_q, h_kv, rows, out, lse, counters, stream);
}

da_status da_rank_forward_table(da_rank* r, int32_t steps, const int32_t* tasks, int64_t n_tasks,
                                const int32_t* messages, int64_t n_messages, const void* q,
                                const void* k, const void* v, int64_t h_q, int64_t h_kv,
                                int64_t rows, void* out, float* lse, da_counters* counters,
                                void* stream) {
  if (r == nullptr) return set_error(DA_ERR_CONFIG, "da_rank_forward: null runtime");
  return rank_forward_flat(r, rank_table(r->world, steps, tasks, n_tasks, messages, n_messages),
                           q, k, v, h_q, h_kv, rows, out, lse, counters, stream);
}

da_status da_rank_backward(da_rank* r, int schedule_kind, const void* d_out, float* dq, float* dk,
                           float* dv, da_counters* counters, void* stream) {
  if (r == nullptr) return set_error(DA_ERR_CONFIG, "da_rank_backward: null runtime");
  bool ok = false;
  const FlatSchedule sch = backward_table(schedule_kind, r->world, &ok);
  if (!ok) return set_error(DA_ERR_CONFIG, "da_rank_backward: unknown schedule kind");
  return rank_backward_flat(r, sch, d_out, dq, dk, dv, counters, stream);
}

da_status da_rank_backward_table(da_rank* r, int32_t steps, const int32_t* tasks, int64_t n_tasks,
                                 const int32_t* messages, int64_t n_messages, const void* d_out,
                                 float* dq, float* dk, float* dv, da_counters* counters,
                                 void* stream) {
  if (r == nullptr) return set_error(DA_ERR_CONFIG, "da_rank_backward: null runtime");
  return rank_backward_flat(r, rank_table(r->world, steps, tasks, n_tasks, messages, n_messages),
                            d_out, dq, dk, dv, counters, stream);
}

void da_rank_set_trace(da_rank* r, int on) {
  if (r) r->trace_on = on != 0;
}

// Resolves the recorded events of the last pass of kind `pass` (synchronises
// on them once) into records with times in ms relative to the pass origin.
da_status da_rank_trace(da_rank* r, int pass, da_trace_rec* out, int64_t cap, int64_t* n) {
  if (r == nullptr || n == nullptr || pass < 0 || pass > 1)
    return set_error(DA_ERR_CONFIG, "da_rank_trace: bad arguments");
  if (!r->trace_ready[pass]) {
    if (r->trace_origin[pass] == nullptr)
      return set_error(DA_ERR_STATE, "da_rank_trace: the pass ran without tracing");
    for (cudaEvent_t e : r->trace_events[pass]) DA_TRY(ck(cudaEventSynchronize(e), "trace"));
    for (auto& x : r->pending[pass]) {
      da_trace_rec rec = x.rec;
      DA_TRY(ck(cudaEventElapsedTime(&rec.t0_ms, r->trace_origin[pass], x.e0), "trace"));
      DA_TRY(ck(cudaEventElapsedTime(&rec.t1_ms, r->trace_origin[pass], x.e1), "trace"));
      r->resolved[pass].push_back(rec);
    }
    trace_free(r, pass);
    r->trace_ready[pass] = true;
  }
  *n = static_cast<int64_t>(r->resolved[pass].size());
  for (int64_t i = 0; out != nullptr && i < *n && i < cap; ++i) out[i] = r->resolved[pass][i];
  return DA_OK;
}

// The pass's phase lists of one rank, without a device (protocol tests):
// per entry {pass (0 fwd, 1 bwd), phase (2t + 0 operands(t), 2t + 1
// results(t)), dir (0 send, 1 recv), peer (0-based), key}.
da_status da_rank_protocol(int world, int rank, int fwd_kind, int bwd_kind, int32_t* out,
                           int64_t cap, int64_t* n) {
  if (n == nullptr || world < 1 || rank < 0 || rank >= world)
    return set_error(DA_ERR_CONFIG, "da_rank_protocol: bad arguments");
  *n = 0;
  for (int pass = 0; pass < 2; ++pass) {
    bool ok = false;
    const FlatSchedule sch = pass == 0 ? forward_table(fwd_kind, world, &ok)
                                       : backward_table(bwd_kind, world, &ok);
    if (!ok) return set_error(DA_ERR_CONFIG, "da_rank_protocol: unknown schedule kind");
    Program pg;
    DA_TRY(pass == 0 ? forward_program(sch, rank + 1, &pg) : backward_program(sch, rank + 1, &pg));
    for (size_t t = 0; t < pg.plans.size(); ++t)
      for (int kind = 0; kind < 2; ++kind) {
        const Phase& ph = kind == 0 ? pg.operands[t] : pg.results[t];
        auto emit = [&](int dir, int peer, int key) {
          if (out != nullptr && *n < cap) {
            int32_t* e = out + 5 * (*n);
            e[0] = pass;
            e[1] = static_cast<int32_t>(2 * t + kind);
            e[2] = dir;
            e[3] = peer;
            e[4] = key;
          }
          ++*n;
        };
        for (const XSend& s : ph.sends) emit(0, s.dst, s.key);
        for (const XRecv& x : ph.recvs) emit(1, x.src, x.key);
      }
  }
  return DA_OK;
}

}  // extern "C"
