// Per-rank sequence-parallel runtime (one process per GPU) in C++.
//
// Each rank holds ONE contiguous chunk and runs the reference worker's
// operation order (runtime.cpp:390-487 forward, 653-716 backward; per step:
// the primary task, then the merges in helper order) from the same flat
// schedule tables as the rest of the library (schedule.cpp). Messages are
// pulls: the receiver's side stream copies straight from the sender's HBM
// (CUDA IPC mapping; the copy engines move the bytes over NVLink, no SM and
// no NCCL kernel involved) into its receive slot, prefetched one step ahead
// (double-buffered slots: the reference's residency bound of 2).
//
// Ordering between ranks uses 32-bit counters in device memory (csrc/peer.cu):
//   flags[dst]          "ready": bumped on the sender's compute stream after
//                       the producer of the n-th message to dst
//   flags[world + src]  "done": bumped on the receiver's side stream after
//                       the n-th pull from src
// The receiver's side stream waits for ready >= n before pulling; a sender
// that reuses a buffer (partials, gradient slots) or returns to its caller
// first waits (in its stream) for done >= n. Messages of a pair are matched
// by order, exactly as both sides walk the same schedule.
//
// Publication: before a pass every rank allgathers, per pulled buffer, the
// IPC handle of its allocation and the offset inside it (through the
// caller's allgather); peers open each allocation once and cache it.
#include <cuda.h>
#include <cuda_runtime.h>

#include <array>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "capi_internal.h"
#include "kernels.h"
#include "schedule_impl.h"

extern "C" da_status da_stream_write_u32(void* stream, void* addr, uint32_t value);
extern "C" da_status da_stream_wait_u32_geq(void* stream, const void* addr, uint32_t value);

namespace da {
namespace {

// buffers peers pull from (per pass)
enum Key : int {
  kK = 0, kV, kQ, kPart, kKHi, kVHi,                    // forward
  kDOut, kLse, kDVec, kGK0, kGV0, kGK1, kGV1, kGQ0, kGQ1,  // backward
  kNumKeys
};

struct PubRecord {
  cudaIpcMemHandle_t handle;
  uint64_t offset;
  uint64_t base;   // sender-side allocation base (cache key together with the rank)
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

struct Work {
  cudaEvent_t done = nullptr;                 // pulls landed (side stream)
  std::vector<std::pair<int, uint32_t>> expect;  // peers' done counters to await
};

}  // namespace
}  // namespace da

struct da_rank {
  int rank = 0, world = 1;
  da_allgather_fn ag = nullptr;
  void* ctx = nullptr;
  cudaStream_t side = nullptr;
  int* flags = nullptr;                 // [2 * world]
  std::vector<int*> rflags;             // peers' flags (mapped)
  std::vector<uint32_t> sent, pulled;   // per peer
  // (rank, allocation's IPC handle bytes) -> mapped base; the handle (not the
  // address) keys the cache, so a reused address of a new allocation remaps
  std::map<std::pair<int, std::string>, char*> opened;
  std::vector<std::array<char*, da::kNumKeys>> remote;  // [rank][key]
  // forward state (the rematerialisation hook: saved O / LSE, never recomputed)
  const void *q = nullptr, *k = nullptr, *v = nullptr;
  void* out = nullptr;
  float* lse = nullptr;
  int64_t h_q = 0, h_kv = 0, rows = 0;
  bool have_forward = false;
  // work buffers
  da::Buf acc, part, kv_slot[2], q_slot[2], k_lo, v_lo, k_hi, v_hi, kvh, flag;
  std::map<int, da::Buf> part_recv, gq_recv;
  da::Buf d_vec, bundle[2], g_send[2], q_send[2], g_recv;
};

namespace da {
namespace {

da_status ck(cudaError_t e, const char* where) {
  return e == cudaSuccess ? DA_OK : cuda_error(e, where);
}

#define DA_TRY(x)                    \
  do {                               \
    const da_status s_ = (x);        \
    if (s_ != DA_OK) return s_;      \
  } while (0)

// cuMemGetAddressRange through the runtime's driver entry point (the library
// must load without libcuda on machines that only build it)
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

// Publishes `ptrs` (nullptr = not published this pass) to every peer.
da_status publish(da_rank* r, const std::array<const void*, kNumKeys>& ptrs) {
  std::vector<PubRecord> mine(kNumKeys);
  for (int key = 0; key < kNumKeys; ++key) {
    PubRecord& rec = mine[key];
    std::memset(&rec, 0, sizeof(rec));
    if (ptrs[key] == nullptr) continue;
    CUdeviceptr base = 0;
    size_t size = 0;
    const AddrRangeFn range = addr_range_fn();
    if (range == nullptr ||
        range(&base, &size, reinterpret_cast<CUdeviceptr>(ptrs[key])) != CUDA_SUCCESS)
      return set_error(DA_ERR_CUDA, "da_rank: cuMemGetAddressRange failed");
    DA_TRY(ck(cudaIpcGetMemHandle(&rec.handle, reinterpret_cast<void*>(base)),
              "cudaIpcGetMemHandle"));
    rec.offset = reinterpret_cast<uint64_t>(ptrs[key]) - base;
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

da_status signal_ready(da_rank* r, int dst, cudaStream_t st) {
  ++r->sent[dst];
  return da_stream_write_u32(st, r->flags + dst, r->sent[dst]);
}

struct Recv {
  void* slot;
  size_t bytes;
  int src;
  Key key;
};

// Sends (dst per tensor, data produced in stream order on `cur`) and pulls.
da_status exchange(da_rank* r, const std::vector<int>& sends, const std::vector<Recv>& recvs,
                   cudaStream_t cur, Work* w) {
  w->expect.clear();
  w->done = nullptr;
  for (int dst : sends) {
    DA_TRY(signal_ready(r, dst, cur));
    w->expect.emplace_back(dst, r->sent[dst]);
  }
  if (recvs.empty()) return DA_OK;
  cudaEvent_t ready;
  DA_TRY(ck(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming), "event"));
  DA_TRY(ck(cudaEventRecord(ready, cur), "event record"));
  DA_TRY(ck(cudaStreamWaitEvent(r->side, ready, 0), "side wait"));
  cudaEventDestroy(ready);
  for (const Recv& x : recvs) {
    const char* src = r->remote[x.src][x.key];
    if (src == nullptr) return set_error(DA_ERR_STATE, "da_rank: pulled buffer was not published");
    ++r->pulled[x.src];
    DA_TRY(da_stream_wait_u32_geq(r->side, r->rflags[x.src] + r->rank, r->pulled[x.src]));
    DA_TRY(ck(cudaMemcpyAsync(x.slot, src, x.bytes, cudaMemcpyDeviceToDevice, r->side), "pull"));
    DA_TRY(da_stream_write_u32(r->side, r->flags + r->world + x.src, r->pulled[x.src]));
  }
  DA_TRY(ck(cudaEventCreateWithFlags(&w->done, cudaEventDisableTiming), "event"));
  return ck(cudaEventRecord(w->done, r->side), "event record");
}

da_status wait_work(da_rank* r, Work* w, cudaStream_t cur) {
  if (w->done) {
    DA_TRY(ck(cudaStreamWaitEvent(cur, w->done, 0), "wait pulls"));
    cudaEventDestroy(w->done);
    w->done = nullptr;
  }
  for (const auto& e : w->expect)
    DA_TRY(da_stream_wait_u32_geq(cur, r->rflags[e.first] + r->world + r->rank, e.second));
  w->expect.clear();
  return DA_OK;
}

struct Plan {
  int action = 0;  // 0 idle, 1 local, 2 direct, 3 help
  int peer = 0;    // 1-based
  int part = kPartWhole;
  std::vector<int> kv_sends, kvh_sends, q_sends, merges, gradkv_from;
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
    if (m.to == worker && m.kind == kMsgGradKV) p.gradkv_from.push_back(m.from);
  }
  return plans;
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
                    float* dq, float* dk, float* dv, bool accumulate_kv, int mask,
                    cudaStream_t st) {
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
  a.rows_kv = rows;
  a.d = 128;
  a.dq_acc = dq;
  a.dk_acc = dk;
  a.dv_acc = dv;
  a.accumulate_kv = accumulate_kv ? 1 : 0;
  a.mask = mask;
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

}  // namespace
}  // namespace da

using namespace da;

extern "C" {

da_status da_rank_create(int rank, int world, da_allgather_fn fn, void* ctx, da_rank** out) {
  if (out == nullptr || fn == nullptr) return set_error(DA_ERR_CONFIG, "da_rank_create: null");
  if (world < 1 || rank < 0 || rank >= world)
    return set_error(DA_ERR_CONFIG, "da_rank_create: bad rank / world");
  std::unique_ptr<da_rank> r(new da_rank());
  r->rank = rank;
  r->world = world;
  r->ag = fn;
  r->ctx = ctx;
  r->sent.assign(world, 0);
  r->pulled.assign(world, 0);
  r->remote.assign(world, {});
  for (auto& a : r->remote) a.fill(nullptr);
  DA_TRY(ck(cudaStreamCreateWithFlags(&r->side, cudaStreamNonBlocking), "side stream"));
  DA_TRY(ck(cudaMalloc(&r->flags, sizeof(int) * 2 * world), "flags"));
  DA_TRY(ck(cudaMemset(r->flags, 0, sizeof(int) * 2 * world), "flags"));
  r->rflags.assign(world, r->flags);
  // exchange the flag pages once
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
  *out = r.release();
  return DA_OK;
}

void da_rank_destroy(da_rank* r) {
  if (r == nullptr) return;
  cudaDeviceSynchronize();
  for (auto& kv : r->opened) cudaIpcCloseMemHandle(kv.second);
  for (int s = 0; s < r->world; ++s)
    if (r->rflags[s] != r->flags) cudaIpcCloseMemHandle(r->rflags[s]);
  if (r->flags) cudaFree(r->flags);
  if (r->side) cudaStreamDestroy(r->side);
  delete r;
}

da_status da_rank_forward(da_rank* r, int schedule_kind, const void* q, const void* k,
                          const void* v, int64_t h_q, int64_t h_kv, int64_t rows, void* out,
                          float* lse, da_counters* counters, void* stream) {
  if (r == nullptr) return set_error(DA_ERR_CONFIG, "da_rank_forward: null runtime");
  if (h_q < 1 || h_kv < 1 || h_q % h_kv != 0 || rows < 1)
    return set_error(DA_ERR_SHAPE, "da_rank_forward: bad shape");
  const int P = r->world, w = r->rank + 1;
  FlatSchedule sch;
  if (schedule_kind == DA_SCHEDULE_RING) sch = make_ring(P);
  else if (schedule_kind == DA_SCHEDULE_BALANCED) sch = make_balanced(P);
  else if (schedule_kind == DA_SCHEDULE_BALANCED_SPLIT) sch = make_balanced_split(P);
  else return set_error(DA_ERR_CONFIG, "da_rank_forward: unknown schedule kind");
  const auto errs = validate_flat(sch);
  if (!errs.empty()) return set_error(DA_ERR_SCHEDULE, "invalid schedule: " + errs.front());
  const auto plans = plans_for(sch, w);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
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
  std::array<const void*, kNumKeys> pub{};
  pub.fill(nullptr);
  pub[kK] = k;
  pub[kV] = v;
  pub[kQ] = q;
  pub[kPart] = r->part.p;
  if (split) {
    pub[kKHi] = r->k_hi.p;
    pub[kVHi] = r->v_hi.p;
  }
  if (P > 1) DA_TRY(publish(r, pub));

  da_counters c{};
  float* acc = r->acc.as<float>();
  bool have_acc = false;
  auto post = [&](int t, Work* work) -> da_status {
    const Plan& p = plans[t];
    std::vector<int> sends;
    std::vector<Recv> recvs;
    for (int dst : p.kv_sends) sends.insert(sends.end(), {dst - 1, dst - 1});
    for (int dst : p.kvh_sends) sends.insert(sends.end(), {dst - 1, dst - 1});
    for (int dst : p.q_sends) sends.push_back(dst - 1);
    if (p.action == 2 && p.part == kPartHigh) {
      recvs.push_back({r->kvh.p, static_cast<size_t>(h_kv) * hi * 256, p.peer - 1, kKHi});
      recvs.push_back({r->kvh.as<char>() + static_cast<size_t>(h_kv) * hi * 256,
                       static_cast<size_t>(h_kv) * hi * 256, p.peer - 1, kVHi});
    } else if (p.action == 2) {
      recvs.push_back({r->kv_slot[t % 2].p, kv_b, p.peer - 1, kK});
      recvs.push_back({r->kv_slot[t % 2].as<char>() + kv_b, kv_b, p.peer - 1, kV});
    } else if (p.action == 3) {
      recvs.push_back({r->q_slot[t % 2].p, q_b, p.peer - 1, kQ});
    }
    return exchange(r, sends, recvs, st, work);
  };

  Work pending, part_work;
  bool part_pending = false;
  int held = 0;
  if (P > 1) DA_TRY(post(0, &pending));
  for (int t = 0; t < static_cast<int>(plans.size()); ++t) {
    const Plan& p = plans[t];
    Work next;
    const bool has_next = t + 1 < static_cast<int>(plans.size());
    if (has_next) DA_TRY(post(t + 1, &next));  // prefetch: overlaps this step's compute
    DA_TRY(wait_work(r, &pending, st));
    const int cur_held = (p.action >= 2 ? 1 : 0) + (has_next && plans[t + 1].action >= 2 ? 1 : 0);
    held = cur_held > held ? cur_held : held;
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
      if (part_pending) DA_TRY(wait_work(r, &part_work, st));  // previous partial pulled
      const bool low = p.part == kPartLow;
      DA_TRY(fwd_chunk(r->q_slot[t % 2].p, low ? r->k_lo.p : k, low ? r->v_lo.p : v, h_q, h_kv,
                       rows, low ? lo : rows, nullptr, r->part.as<float>(), DA_MASK_FULL, st));
      DA_TRY(exchange(r, {p.peer - 1}, {}, st, &part_work));
      part_pending = true;
    }
    for (int hw : p.merges) {
      da::Buf& buf = r->part_recv[hw];
      DA_TRY(ck(buf.ensure(acc_f * 4), "da_rank workspace"));
      Work mw;
      DA_TRY(exchange(r, {}, {{buf.p, acc_f * 4, hw - 1, kPart}}, st, &mw));
      DA_TRY(wait_work(r, &mw, st));
      count(c, kMsgPartial, nq * 130);
      const float* b = buf.as<float>();
      DA_TRY(ck(launch_merge(acc, acc + nq * 128, acc + nq * 129, b, b + nq * 128, b + nq * 129,
                             acc, acc + nq * 128, acc + nq * 129, nq, st),
                "da_rank_forward merge"));
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
  r->h_q = h_q;
  r->h_kv = h_kv;
  r->rows = rows;
  r->have_forward = true;
  c.max_remote_chunks_held = held;
  if (counters) *counters = c;
  return da_check_degenerate(r->flag.as<int>(), stream);
}

da_status da_rank_backward(da_rank* r, int schedule_kind, const void* d_out, float* dq, float* dk,
                           float* dv, da_counters* counters, void* stream) {
  if (r == nullptr) return set_error(DA_ERR_CONFIG, "da_rank_backward: null runtime");
  if (!r->have_forward)
    return set_error(DA_ERR_STATE, "run_backward requires forward output and logsumexp");
  if (d_out == nullptr) return set_error(DA_ERR_STATE, "run_backward requires d_out");
  const int P = r->world, w = r->rank + 1;
  FlatSchedule sch;
  if (schedule_kind == DA_SCHEDULE_RING_BWD || schedule_kind == DA_SCHEDULE_RING)
    sch = make_ring_backward(P);
  else if (schedule_kind == DA_SCHEDULE_BALANCED_BWD || schedule_kind == DA_SCHEDULE_BALANCED)
    sch = make_balanced_backward(P);
  else
    return set_error(DA_ERR_CONFIG, "da_rank_backward: unknown schedule kind");
  const auto errs = validate_backward_flat(sch);
  if (!errs.empty()) return set_error(DA_ERR_SCHEDULE, "invalid schedule: " + errs.front());
  const auto plans = plans_for(sch, w);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
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
  DA_TRY(ck(r->g_recv.ensure(2 * g_kv), "da_rank workspace"));
  DA_TRY(ck(cudaMemsetAsync(dq, 0, g_q, st), "dq zero"));
  DA_TRY(ck(cudaMemsetAsync(dk, 0, g_kv, st), "dk zero"));
  DA_TRY(ck(cudaMemsetAsync(dv, 0, g_kv, st), "dv zero"));
  DA_TRY(ck(launch_bwd_preprocess(d_out, r->out, r->d_vec.as<float>(), nq, st), "preprocess"));
  std::array<const void*, kNumKeys> pub{};
  pub.fill(nullptr);
  pub[kK] = r->k;
  pub[kV] = r->v;
  pub[kQ] = r->q;
  pub[kDOut] = d_out;
  pub[kLse] = r->lse;
  pub[kDVec] = r->d_vec.p;
  pub[kGK0] = r->g_send[0].p;
  pub[kGV0] = r->g_send[0].as<char>() + g_kv;
  pub[kGK1] = r->g_send[1].p;
  pub[kGV1] = r->g_send[1].as<char>() + g_kv;
  pub[kGQ0] = r->q_send[0].p;
  pub[kGQ1] = r->q_send[1].p;
  if (P > 1) DA_TRY(publish(r, pub));

  da_counters c{};
  auto post = [&](int t, Work* work) -> da_status {
    const Plan& p = plans[t];
    std::vector<int> sends;
    std::vector<Recv> recvs;
    for (int dst : p.kv_sends) sends.insert(sends.end(), {dst - 1, dst - 1});
    for (int dst : p.q_sends) sends.insert(sends.end(), {dst - 1, dst - 1, dst - 1, dst - 1});
    if (p.action == 2) {
      recvs.push_back({r->kv_slot[t % 2].p, kv_b, p.peer - 1, kK});
      recvs.push_back({r->kv_slot[t % 2].as<char>() + kv_b, kv_b, p.peer - 1, kV});
    } else if (p.action == 3) {
      char* b = r->bundle[t % 2].as<char>();
      recvs.push_back({b, q_b, p.peer - 1, kQ});
      recvs.push_back({b + q_b, q_b, p.peer - 1, kDOut});
      recvs.push_back({b + 2 * q_b, static_cast<size_t>(nq) * 4, p.peer - 1, kLse});
      recvs.push_back({b + 2 * q_b + nq * 4, static_cast<size_t>(nq) * 4, p.peer - 1, kDVec});
    }
    return exchange(r, sends, recvs, st, work);
  };
  Work pending;
  if (P > 1) DA_TRY(post(0, &pending));
  for (int t = 0; t < static_cast<int>(plans.size()); ++t) {
    const Plan& p = plans[t];
    Work next;
    if (t + 1 < static_cast<int>(plans.size())) DA_TRY(post(t + 1, &next));
    DA_TRY(wait_work(r, &pending, st));
    std::vector<int> sends;
    if (p.action == 1) {
      ++c.attention_kernel_calls;
      DA_TRY(bwd_chunk(r->q, r->k, r->v, d_out, r->lse, r->d_vec.as<float>(), h_q, h_kv, rows, dq,
                       dk, dv, true, DA_MASK_DIAGONAL, st));
    } else if (p.action == 2) {
      ++c.attention_kernel_calls;
      count(c, kMsgKV, 2 * nkv * 128);
      const char* ks = r->kv_slot[t % 2].as<char>();
      float* gk = r->g_send[t % 2].as<float>();
      DA_TRY(bwd_chunk(r->q, ks, ks + kv_b, d_out, r->lse, r->d_vec.as<float>(), h_q, h_kv, rows,
                       dq, gk, gk + nkv * 128, false, DA_MASK_FULL, st));
      sends.insert(sends.end(), {p.peer - 1, p.peer - 1});
    } else if (p.action == 3) {
      ++c.attention_kernel_calls;
      c.q_scalars += rows * (2 * 128 + 2) * h_q;
      ++c.q_messages;
      const char* b = r->bundle[t % 2].as<char>();
      float* gq = r->q_send[t % 2].as<float>();
      DA_TRY(ck(cudaMemsetAsync(gq, 0, g_q, st), "gq zero"));
      DA_TRY(bwd_chunk(b, r->k, r->v, b + q_b, reinterpret_cast<const float*>(b + 2 * q_b),
                       reinterpret_cast<const float*>(b + 2 * q_b + nq * 4), h_q, h_kv, rows, gq,
                       dk, dv, true, DA_MASK_FULL, st));
      sends.push_back(p.peer - 1);
    }
    if (p.gradkv_from.size() > 1)
      return set_error(DA_ERR_SCHEDULE, "at most one GradKV per worker and step is supported");
    std::vector<Recv> recvs;
    const Key gk_key = (t % 2) ? kGK1 : kGK0, gv_key = (t % 2) ? kGV1 : kGV0;
    const Key gq_key = (t % 2) ? kGQ1 : kGQ0;
    for (int s : p.gradkv_from) {
      recvs.push_back({r->g_recv.p, g_kv, s - 1, gk_key});
      recvs.push_back({r->g_recv.as<char>() + g_kv, g_kv, s - 1, gv_key});
    }
    for (int hw : p.merges) {
      da::Buf& buf = r->gq_recv[hw];
      DA_TRY(ck(buf.ensure(g_q), "da_rank workspace"));
      recvs.push_back({buf.p, g_q, hw - 1, gq_key});
    }
    // results leave right after their kernels; waiting also retires the send
    // buffers before they are rewritten two steps later
    Work sw;
    DA_TRY(exchange(r, sends, recvs, st, &sw));
    DA_TRY(wait_work(r, &sw, st));
    if (!p.gradkv_from.empty()) {
      count(c, kMsgGradKV, 2 * nkv * 128);
      DA_TRY(ck(launch_add(dk, r->g_recv.as<float>(), nkv * 128, st), "GradKV fold"));
      DA_TRY(ck(launch_add(dv, r->g_recv.as<float>() + nkv * 128, nkv * 128, st), "GradKV fold"));
    }
    for (int hw : p.merges) {
      c.partial_scalars += nq * 128;
      ++c.partial_messages;
      DA_TRY(ck(launch_add(dq, r->gq_recv[hw].as<float>(), nq * 128, st), "dq fold"));
    }
    pending = next;
  }
  if (counters) *counters = c;
  return DA_OK;
}

}  // extern "C"
