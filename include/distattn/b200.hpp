// distattn::b200 — C++ host API over the C ABI (include/distattn_b200.h).
//
// The reference's public interface is header-level C++ in
// /root/reference/proj/include/distattn (flashcore.hpp, schedule.hpp,
// runtime.hpp, errors.hpp). This header restores those names and value
// semantics for device-resident data, so the reference's call sites
// (runtime.cpp, ckptplan.cpp) switch by namespace:
//   * exceptions: the reference taxonomy (errors.hpp:12-48), thrown from the
//     C ABI status codes with da_last_error() as the message;
//   * flashcore: block_attn_update takes the accumulator by value and returns
//     it (flashcore.hpp:136-141), rescale / finalize / backward_aux /
//     block_attn_backward as flashcore.hpp:202-337;
//   * schedule: Task / ScheduleMessage / Schedule (schedule.hpp:21-80),
//     build_ring_schedule / build_balanced_schedule / validate
//     (schedule.cpp:60-258) plus the extensions (balanced backward, split);
//   * runtime: SequenceShard / make_shards / run_forward / run_backward
//     (runtime.hpp:32-110) with P logical workers on one device.
// Data: bf16 chunks [heads, rows, 128] and fp32 statistics in device memory
// owned by RAII DeviceBuffer<T>; everything is enqueued on the given stream.
#ifndef DISTATTN_B200_HPP
#define DISTATTN_B200_HPP

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../distattn_b200.h"

namespace distattn {
namespace b200 {

// ---------------------------------------------------------------- errors.hpp
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ShapeError : Error {
  using Error::Error;
};
struct ConfigError : Error {
  using Error::Error;
};
struct ScheduleError : Error {
  using Error::Error;
};
struct StateError : Error {
  using Error::Error;
};
struct DegenerateRowError : Error {
  using Error::Error;
};

inline void check(da_status s) {
  switch (s) {
    case DA_OK: return;
    case DA_ERR_SHAPE: throw ShapeError(da_last_error());
    case DA_ERR_CONFIG: throw ConfigError(da_last_error());
    case DA_ERR_SCHEDULE: throw ScheduleError(da_last_error());
    case DA_ERR_STATE: throw StateError(da_last_error());
    case DA_ERR_DEGENERATE_ROW: throw DegenerateRowError(da_last_error());
    default: throw Error(da_last_error());
  }
}

inline void check_cuda(cudaError_t e, const char* where) {
  if (e != cudaSuccess) throw Error(std::string(where) + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------- memory
template <typename T>
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(size_t n) : n_(n) {
    if (n_ > 0) check_cuda(cudaMalloc(&p_, n_ * sizeof(T)), "cudaMalloc");
  }
  ~DeviceBuffer() {
    if (p_) cudaFree(p_);
  }
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(std::exchange(o.p_, nullptr)), n_(o.n_) {}
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    if (this != &o) {
      if (p_) cudaFree(p_);
      p_ = std::exchange(o.p_, nullptr);
      n_ = o.n_;
    }
    return *this;
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;

  T* data() { return p_; }
  const T* data() const { return p_; }
  size_t size() const { return n_; }

  void upload(const T* host, cudaStream_t st) {
    check_cuda(cudaMemcpyAsync(p_, host, n_ * sizeof(T), cudaMemcpyHostToDevice, st), "upload");
  }
  std::vector<T> download(cudaStream_t st) const {
    std::vector<T> h(n_);
    check_cuda(cudaMemcpyAsync(h.data(), p_, n_ * sizeof(T), cudaMemcpyDeviceToHost, st),
               "download");
    check_cuda(cudaStreamSynchronize(st), "download sync");
    return h;
  }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
};

using bf16_t = uint16_t;  // storage of one bfloat16 value
constexpr int64_t kHeadDim = 128;

// ---------------------------------------------------------------- flashcore.hpp
enum class MaskMode { Diagonal = DA_MASK_DIAGONAL, Full = DA_MASK_FULL, Empty = DA_MASK_EMPTY };

/// A bf16 chunk [heads, rows, 128] in device memory (non-owning view).
struct Chunk {
  const void* data = nullptr;
  int64_t heads = 0, rows = 0;
};

/// AttnAccumulatorT (flashcore.hpp:65-81): unnormalised o, running max m, sum l.
struct AttnAccumulator {
  DeviceBuffer<float> o, m, l;
  int64_t heads = 0, rows = 0;
  bool fresh = true;  // AttnAccumulator::fresh (m = -inf, l = 0, o = 0), not materialised

  static AttnAccumulator make_fresh(int64_t heads, int64_t rows) {
    AttnAccumulator a;
    a.heads = heads;
    a.rows = rows;
    a.fresh = true;
    return a;
  }
  void allocate() {
    o = DeviceBuffer<float>(heads * rows * kHeadDim);
    m = DeviceBuffer<float>(heads * rows);
    l = DeviceBuffer<float>(heads * rows);
  }
};

/// AttnOutputT (flashcore.hpp:83-87).
struct AttnOutput {
  DeviceBuffer<bf16_t> o;
  DeviceBuffer<float> lse;
  Chunk chunk() const { return Chunk{o.data(), heads, rows}; }
  int64_t heads = 0, rows = 0;
};

/// ChunkGradsT (flashcore.hpp:242-246), fp32.
struct ChunkGrads {
  DeviceBuffer<float> dq, dk, dv;
};

/// Caller-owned device scratch of the flashcore calls (the D vector of
/// backward_aux, the degenerate-row flag): grown on first use and reused, so
/// the per-task calls the reference's runtime makes in a loop
/// (runtime.cpp:286-328, 605-716) allocate nothing and never synchronise
/// except where the reference's semantics require it (finalize throwing
/// DegenerateRowError). One Workspace per stream.
class Workspace {
 public:
  float* d_vec(int64_t n) {
    if (static_cast<size_t>(n) > d_.size()) d_ = DeviceBuffer<float>(n);
    return d_.data();
  }
  int* flag() {
    if (flag_.size() == 0) flag_ = DeviceBuffer<int>(1);
    return flag_.data();
  }

 private:
  DeviceBuffer<float> d_;
  DeviceBuffer<int> flag_;
};

inline void check_kv(const Chunk& k, const Chunk& v, const char* op) {
  if (k.heads != v.heads || k.rows != v.rows)
    throw ShapeError(std::string(op) + ": k/v row mismatch");
}

inline void fill_fwd_args(da_fwd_args& a, const Chunk& q, const Chunk& k, const Chunk& v,
                          MaskMode mask, double scale) {
  a.q = q.data;
  a.k = k.data;
  a.v = v.data;
  a.h_q = q.heads;
  a.h_kv = k.heads;
  a.rows_q = q.rows;
  a.rows_kv = k.rows;
  a.d = kHeadDim;
  a.scale = static_cast<float>(scale);
  a.mask = static_cast<int>(mask);
}

/// block_attn_update (flashcore.hpp:135-197): absorbs one kv chunk; the
/// accumulator is taken by value and returned (the reference's semantics).
inline AttnAccumulator block_attn_update(const Chunk& q, const Chunk& k, const Chunk& v,
                                         AttnAccumulator acc, MaskMode mask, double scale,
                                         cudaStream_t st) {
  check_kv(k, v, "block_attn_update");
  if (acc.heads != q.heads || acc.rows != q.rows)
    throw ShapeError("block_attn_update: accumulator shape mismatch");
  da_fwd_args a{};
  fill_fwd_args(a, q, k, v, mask, scale);
  if (acc.fresh) {
    acc.allocate();
  } else {
    a.o_in = acc.o.data();
    a.m_in = acc.m.data();
    a.l_in = acc.l.data();
  }
  a.o_acc = acc.o.data();
  a.m_acc = acc.m.data();
  a.l_acc = acc.l.data();
  check(da_attn_fwd_chunk(&a, st));
  acc.fresh = false;
  return acc;
}

/// rescale (flashcore.hpp:202-224): merge of two partial accumulators.
inline AttnAccumulator rescale(const AttnAccumulator& x, const AttnAccumulator& y,
                               cudaStream_t st) {
  if (x.heads != y.heads || x.rows != y.rows)
    throw ShapeError("rescale: accumulator shapes disagree");
  if (x.fresh || y.fresh) throw StateError("rescale: materialise fresh accumulators first");
  AttnAccumulator out = AttnAccumulator::make_fresh(x.heads, x.rows);
  out.allocate();
  out.fresh = false;
  check(da_attn_merge(x.o.data(), x.m.data(), x.l.data(), y.o.data(), y.m.data(), y.l.data(),
                      out.o.data(), out.m.data(), out.l.data(), x.heads, x.rows, kHeadDim, st));
  return out;
}

/// rescale into a caller-owned accumulator (no allocation; `out` may be `x`).
inline void rescale_into(const AttnAccumulator& x, const AttnAccumulator& y, AttnAccumulator& out,
                         cudaStream_t st) {
  if (x.heads != y.heads || x.rows != y.rows || out.heads != x.heads || out.rows != x.rows)
    throw ShapeError("rescale: accumulator shapes disagree");
  if (x.fresh || y.fresh) throw StateError("rescale: materialise fresh accumulators first");
  if (out.fresh) out.allocate();
  out.fresh = false;
  check(da_attn_merge(x.o.data(), x.m.data(), x.l.data(), y.o.data(), y.m.data(), y.l.data(),
                      out.o.data(), out.m.data(), out.l.data(), x.heads, x.rows, kHeadDim, st));
}

/// finalize (flashcore.hpp:227-240): O = o / l (bf16), LSE = m + ln l;
/// throws DegenerateRowError when a row attended to no key.
inline void finalize_into(const AttnAccumulator& acc, AttnOutput& out, Workspace& ws,
                          cudaStream_t st) {
  if (acc.fresh) throw DegenerateRowError("finalize: a row attended to no key");
  if (out.o.size() != static_cast<size_t>(acc.heads * acc.rows * kHeadDim) ||
      out.lse.size() != static_cast<size_t>(acc.heads * acc.rows))
    throw ShapeError("finalize: output shape mismatch");
  out.heads = acc.heads;
  out.rows = acc.rows;
  int* flag = ws.flag();
  check_cuda(cudaMemsetAsync(flag, 0, sizeof(int), st), "finalize flag");
  check(da_attn_finalize(acc.o.data(), acc.m.data(), acc.l.data(), out.o.data(), out.lse.data(),
                         flag, acc.heads, acc.rows, kHeadDim, st));
  check(da_check_degenerate(flag, st));  // DegenerateRowError needs the flag on the host
}

inline AttnOutput finalize(const AttnAccumulator& acc, Workspace& ws, cudaStream_t st) {
  AttnOutput out;
  out.o = DeviceBuffer<bf16_t>(acc.heads * acc.rows * kHeadDim);
  out.lse = DeviceBuffer<float>(acc.heads * acc.rows);
  finalize_into(acc, out, ws, st);
  return out;
}

inline AttnOutput finalize(const AttnAccumulator& acc, cudaStream_t st) {
  thread_local Workspace ws;  // one flag per thread, reused
  return finalize(acc, ws, st);
}

/// backward_aux (flashcore.hpp:250-261): D = rowsum(dO o O).
inline DeviceBuffer<float> backward_aux(const Chunk& d_out, const Chunk& out, cudaStream_t st) {
  DeviceBuffer<float> d(out.heads * out.rows);
  check(da_attn_bwd_preprocess(d_out.data, out.data, d.data(), out.heads, out.rows, kHeadDim, st));
  return d;
}

/// block_attn_backward (flashcore.hpp:269-337) into caller-owned fp32
/// gradients: dq is accumulated into g.dq, dk / dv are added
/// (accumulate_kv) or overwritten. D goes to the workspace; nothing is
/// allocated and the stream is not synchronised.
inline void block_attn_backward_into(const Chunk& q, const Chunk& k, const Chunk& v,
                                     const Chunk& out, const float* lse, const Chunk& d_out,
                                     MaskMode mask, double scale, ChunkGrads& g, Workspace& ws,
                                     cudaStream_t st, bool accumulate_kv = false,
                                     bool deterministic = false) {
  check_kv(k, v, "block_attn_backward");
  if (out.heads != q.heads || out.rows != q.rows)
    throw ShapeError("block_attn_backward: output shape mismatch");
  if (d_out.heads != q.heads || d_out.rows != q.rows)
    throw ShapeError("block_attn_backward: upstream grad shape mismatch");
  if (g.dq.size() != static_cast<size_t>(q.heads * q.rows * kHeadDim) ||
      g.dk.size() != static_cast<size_t>(k.heads * k.rows * kHeadDim) ||
      g.dv.size() != static_cast<size_t>(k.heads * k.rows * kHeadDim))
    throw ShapeError("block_attn_backward: gradient shape mismatch");
  float* d = ws.d_vec(q.heads * q.rows);
  check(da_attn_bwd_preprocess(d_out.data, out.data, d, out.heads, out.rows, kHeadDim, st));
  da_bwd_args a{};
  a.q = q.data;
  a.k = k.data;
  a.v = v.data;
  a.d_out = d_out.data;
  a.lse = lse;
  a.d_vec = d;
  a.h_q = q.heads;
  a.h_kv = k.heads;
  a.rows_q = q.rows;
  a.rows_kv = k.rows;
  a.d = kHeadDim;
  a.dq_acc = g.dq.data();
  a.dk_acc = g.dk.data();
  a.dv_acc = g.dv.data();
  a.accumulate_kv = accumulate_kv ? 1 : 0;
  a.scale = static_cast<float>(scale);
  a.mask = static_cast<int>(mask);
  a.deterministic = deterministic ? 1 : 0;
  check(da_attn_bwd_chunk(&a, st));
}

/// Value form (the reference returns the contribution, flashcore.hpp:290):
/// allocates the returned gradients; D lives in the thread's workspace.
inline ChunkGrads block_attn_backward(const Chunk& q, const Chunk& k, const Chunk& v,
                                      const Chunk& out, const float* lse, const Chunk& d_out,
                                      MaskMode mask, double scale, cudaStream_t st,
                                      bool deterministic = false) {
  thread_local Workspace ws;
  ChunkGrads g{DeviceBuffer<float>(q.heads * q.rows * kHeadDim),
               DeviceBuffer<float>(k.heads * k.rows * kHeadDim),
               DeviceBuffer<float>(k.heads * k.rows * kHeadDim)};
  check_cuda(cudaMemsetAsync(g.dq.data(), 0, g.dq.size() * sizeof(float), st), "dq zero");
  block_attn_backward_into(q, k, v, out, lse, d_out, mask, scale, g, ws, st, false,
                           deterministic);
  return g;
}

// ---------------------------------------------------------------- schedule.hpp
enum class TaskKind { LocalAttn = 0, RemoteAttn = 1, RescaleMerge = 2, Idle = 3 };
enum class PayloadKind { KV = 0, Q = 1, PartialResult = 2, GradKV = 3, KVHalf = 4 };

struct Task {
  TaskKind kind = TaskKind::Idle;
  int worker = 0, query_owner = 0, kv_owner = 0, helper = 0;
  bool is_attention() const { return kind == TaskKind::LocalAttn || kind == TaskKind::RemoteAttn; }
};

struct ScheduleMessage {
  int step = 0, from = 0, to = 0;
  PayloadKind kind = PayloadKind::KV;
};

struct Schedule {
  int workers = 0;
  std::vector<std::vector<Task>> steps;
  std::vector<ScheduleMessage> messages;
  int step_count() const { return static_cast<int>(steps.size()); }
  int attention_task_count() const {
    int n = 0;
    for (const auto& s : steps)
      for (const auto& t : s) n += t.is_attention() ? 1 : 0;
    return n;
  }
  int idle_slot_count() const {
    int n = 0;
    for (const auto& s : steps)
      for (const auto& t : s) n += t.kind == TaskKind::Idle ? 1 : 0;
    return n;
  }
};

inline Schedule build_schedule(int workers, da_schedule_kind kind) {
  int32_t steps = 0;
  int64_t nt = 0, nm = 0;
  check(da_schedule_build(workers, kind, &steps, nullptr, &nt, nullptr, &nm));
  std::vector<int32_t> t(6 * nt), m(4 * (nm > 0 ? nm : 1));
  check(da_schedule_build(workers, kind, &steps, t.data(), &nt, m.data(), &nm));
  Schedule s;
  s.workers = workers;
  s.steps.resize(steps);
  for (int64_t i = 0; i < nt; ++i) {
    const int32_t* o = t.data() + 6 * i;
    s.steps[o[0]].push_back(Task{static_cast<TaskKind>(o[1]), o[2], o[3], o[4], o[5]});
  }
  for (int64_t i = 0; i < nm; ++i) {
    const int32_t* o = m.data() + 4 * i;
    s.messages.push_back(ScheduleMessage{o[0], o[1], o[2], static_cast<PayloadKind>(o[3])});
  }
  return s;
}

inline Schedule build_ring_schedule(int workers) { return build_schedule(workers, DA_SCHEDULE_RING); }
inline Schedule build_balanced_schedule(int workers) {
  return build_schedule(workers, DA_SCHEDULE_BALANCED);
}
inline Schedule build_balanced_split_schedule(int workers) {
  return build_schedule(workers, DA_SCHEDULE_BALANCED_SPLIT);
}
/// Backward schedules (extensions; the reference's backward is the ring order).
inline Schedule build_ring_backward_schedule(int workers) {
  return build_schedule(workers, DA_SCHEDULE_RING_BWD);
}
inline Schedule build_balanced_backward_schedule(int workers) {
  return build_schedule(workers, DA_SCHEDULE_BALANCED_BWD);
}
inline Schedule build_balanced_split_backward_schedule(int workers) {
  return build_schedule(workers, DA_SCHEDULE_BALANCED_SPLIT_BWD);
}

inline void flatten(const Schedule& s, std::vector<int32_t>& t, std::vector<int32_t>& m) {
  t.clear();
  m.clear();
  for (size_t st = 0; st < s.steps.size(); ++st)
    for (const Task& k : s.steps[st])
      t.insert(t.end(), {static_cast<int32_t>(st), static_cast<int32_t>(k.kind), k.worker,
                         k.query_owner, k.kv_owner, k.helper});
  for (const ScheduleMessage& x : s.messages)
    m.insert(m.end(), {x.step, x.from, x.to, static_cast<int32_t>(x.kind)});
}

/// validate (schedule.cpp:121-258): the violation messages (empty = valid).
inline std::vector<std::string> validate(const Schedule& s) {
  std::vector<int32_t> t, m;
  flatten(s, t, m);
  const int64_t n = da_schedule_validate(s.workers, s.step_count(), t.data(),
                                         static_cast<int64_t>(t.size() / 6), m.data(),
                                         static_cast<int64_t>(m.size() / 4));
  if (n < 0) throw ConfigError(da_last_error());
  std::vector<std::string> out;
  if (n == 0) return out;
  std::string all = da_last_error();
  size_t pos = 0;
  while (pos <= all.size()) {
    const size_t nl = all.find('\n', pos);
    out.push_back(all.substr(pos, nl == std::string::npos ? std::string::npos : nl - pos));
    if (nl == std::string::npos) break;
    pos = nl + 1;
  }
  return out;
}

// ---------------------------------------------------------------- runtime.hpp
/// SequenceShard (runtime.hpp:32-41): one worker's chunk, device resident.
struct SequenceShard {
  int worker = 0;
  DeviceBuffer<bf16_t> q, k, v, out, d_out;
  DeviceBuffer<float> lse, dq, dk, dv;
};

struct CommCounters {
  int64_t kv_scalars = 0, q_scalars = 0, partial_scalars = 0, grad_scalars = 0;
  int64_t kv_messages = 0, q_messages = 0, partial_messages = 0, grad_messages = 0;
  int64_t attention_kernel_calls = 0;
  int max_remote_chunks_held = 0;
};

/// P shards of `heads` heads x (n / P) rows; q/k/v/d_out uploaded from host
/// bf16 arrays laid out [heads][n][128] (the whole sequence).
inline std::vector<SequenceShard> make_shards(int workers, int64_t n, int64_t heads,
                                              const std::vector<bf16_t>& q,
                                              const std::vector<bf16_t>& k,
                                              const std::vector<bf16_t>& v,
                                              const std::vector<bf16_t>& d_out, cudaStream_t st) {
  if (workers < 1) throw ConfigError("need at least 1 worker");
  if (n < 1 || n % workers != 0) throw ConfigError("token count not divisible by workers");
  const int64_t rows = n / workers;
  std::vector<SequenceShard> s(workers);
  std::vector<bf16_t> tmp(heads * rows * kHeadDim);
  auto slice = [&](const std::vector<bf16_t>& full, int p, DeviceBuffer<bf16_t>& dst) {
    for (int64_t h = 0; h < heads; ++h)
      for (int64_t r = 0; r < rows; ++r)
        for (int64_t c = 0; c < kHeadDim; ++c)
          tmp[(h * rows + r) * kHeadDim + c] = full[(h * n + p * rows + r) * kHeadDim + c];
    dst = DeviceBuffer<bf16_t>(tmp.size());
    dst.upload(tmp.data(), st);
    check_cuda(cudaStreamSynchronize(st), "make_shards");
  };
  for (int p = 0; p < workers; ++p) {
    s[p].worker = p + 1;
    slice(q, p, s[p].q);
    slice(k, p, s[p].k);
    slice(v, p, s[p].v);
    slice(d_out, p, s[p].d_out);
    s[p].out = DeviceBuffer<bf16_t>(heads * rows * kHeadDim);
    s[p].lse = DeviceBuffer<float>(heads * rows);
  }
  return s;
}

struct ShardArrays {
  std::vector<const void*> q, k, v, d_out;
  std::vector<void*> out;
  std::vector<float*> lse, dq, dk, dv;
  da_shards c{};
};

inline ShardArrays shard_arrays(std::vector<SequenceShard>& s, int64_t heads, int64_t rows) {
  ShardArrays a;
  for (auto& x : s) {
    a.q.push_back(x.q.data());
    a.k.push_back(x.k.data());
    a.v.push_back(x.v.data());
    a.d_out.push_back(x.d_out.data());
    a.out.push_back(x.out.data());
    a.lse.push_back(x.lse.data());
    a.dq.push_back(x.dq.data());
    a.dk.push_back(x.dk.data());
    a.dv.push_back(x.dv.data());
  }
  a.c.workers = static_cast<int32_t>(s.size());
  a.c.h_q = heads;
  a.c.h_kv = heads;
  a.c.rows = rows;
  a.c.d = kHeadDim;
  a.c.q = a.q.data();
  a.c.k = a.k.data();
  a.c.v = a.v.data();
  a.c.out = a.out.data();
  a.c.lse = a.lse.data();
  a.c.d_out = a.d_out.data();
  a.c.dq = a.dq.data();
  a.c.dk = a.dk.data();
  a.c.dv = a.dv.data();
  return a;
}

inline CommCounters to_counters(const da_counters& c) {
  CommCounters o;
  o.kv_scalars = c.kv_scalars;
  o.q_scalars = c.q_scalars;
  o.partial_scalars = c.partial_scalars;
  o.grad_scalars = c.grad_scalars;
  o.kv_messages = c.kv_messages;
  o.q_messages = c.q_messages;
  o.partial_messages = c.partial_messages;
  o.grad_messages = c.grad_messages;
  o.attention_kernel_calls = c.attention_kernel_calls;
  o.max_remote_chunks_held = c.max_remote_chunks_held;
  return o;
}

/// run_forward (runtime.cpp:491-529): writes out / lse of every shard.
inline CommCounters run_forward(std::vector<SequenceShard>& s, int64_t heads,
                                da_schedule_kind kind, cudaStream_t st) {
  if (s.empty()) throw ConfigError("need at least 1 worker");
  const int64_t rows = static_cast<int64_t>(s[0].lse.size()) / heads;
  ShardArrays a = shard_arrays(s, heads, rows);
  da_counters c{};
  check(da_run_forward(&a.c, kind, &c, st));
  return to_counters(c);
}

/// run_backward (runtime.cpp:720-750): needs the saved O / LSE (no forward
/// recompute); writes fp32 dq / dk / dv of every shard.
inline CommCounters run_backward(std::vector<SequenceShard>& s, int64_t heads,
                                 da_schedule_kind kind, cudaStream_t st) {
  if (s.empty()) throw ConfigError("need at least 1 worker");
  const int64_t rows = static_cast<int64_t>(s[0].lse.size()) / heads;
  for (auto& x : s) {
    if (x.out.size() == 0 || x.lse.size() == 0)
      throw StateError("run_backward requires forward output and logsumexp");
    if (x.dq.size() != static_cast<size_t>(heads * rows * kHeadDim)) {  // reused across calls
      x.dq = DeviceBuffer<float>(heads * rows * kHeadDim);
      x.dk = DeviceBuffer<float>(heads * rows * kHeadDim);
      x.dv = DeviceBuffer<float>(heads * rows * kHeadDim);
    }
  }
  ShardArrays a = shard_arrays(s, heads, rows);
  da_counters c{};
  check(da_run_backward_sched(&a.c, kind, &c, st));
  return to_counters(c);
}

/// RunOptions (runtime.hpp:98-103). On the device both reference executor
/// modes are the same stream-ordered stepper (identical bits), and overlap is
/// the copy / compute concurrency of the stream; both fields are accepted for
/// source compatibility, blocks are validated (the GPU tiles are 128 x 128).
enum class ExecutorMode { Stepper, Concurrent };
struct RunOptions {
  ExecutorMode mode = ExecutorMode::Stepper;
  bool overlap = false;
  int64_t block_rows = 16, block_cols = 16;
  void check() const {
    if (block_rows <= 0 || block_cols <= 0) throw ConfigError("block sizes must be positive");
  }
};

/// run_forward over an arbitrary validated Schedule (runtime.hpp:106-109).
inline CommCounters run_forward(std::vector<SequenceShard>& s, int64_t heads,
                                const Schedule& schedule, const RunOptions& opts,
                                cudaStream_t st) {
  opts.check();
  if (s.empty()) throw ConfigError("need at least 1 worker");
  const int64_t rows = static_cast<int64_t>(s[0].lse.size()) / heads;
  ShardArrays a = shard_arrays(s, heads, rows);
  std::vector<int32_t> t, m;
  flatten(schedule, t, m);
  da_counters c{};
  check(da_run_forward_table(&a.c, schedule.step_count(), t.data(),
                             static_cast<int64_t>(t.size() / 6), m.data(),
                             static_cast<int64_t>(m.size() / 4), &c, st));
  return to_counters(c);
}

/// run_backward over an arbitrary validated backward Schedule.
inline CommCounters run_backward(std::vector<SequenceShard>& s, int64_t heads,
                                 const Schedule& schedule, const RunOptions& opts,
                                 cudaStream_t st) {
  opts.check();
  if (s.empty()) throw ConfigError("need at least 1 worker");
  const int64_t rows = static_cast<int64_t>(s[0].lse.size()) / heads;
  for (auto& x : s) {
    if (x.out.size() == 0 || x.lse.size() == 0)
      throw StateError("run_backward requires forward output and logsumexp");
    if (x.dq.size() != static_cast<size_t>(heads * rows * kHeadDim)) {
      x.dq = DeviceBuffer<float>(heads * rows * kHeadDim);
      x.dk = DeviceBuffer<float>(heads * rows * kHeadDim);
      x.dv = DeviceBuffer<float>(heads * rows * kHeadDim);
    }
  }
  ShardArrays a = shard_arrays(s, heads, rows);
  std::vector<int32_t> t, m;
  flatten(schedule, t, m);
  da_counters c{};
  check(da_run_backward_table(&a.c, schedule.step_count(), t.data(),
                              static_cast<int64_t>(t.size() / 6), m.data(),
                              static_cast<int64_t>(m.size() / 4), &c, st));
  return to_counters(c);
}

/// One rank of the sequence-parallel runtime, one process per GPU
/// (runtime.cpp:390-487, 653-716 for a single worker): messages go over
/// NCCL send/recv or copy-engine pulls from the peers' HBM. `allgather`
/// bootstraps the IPC mappings / the NCCL id (e.g. MPI_Allgather or
/// torch.distributed); calls are collective.
class RankRuntime {
 public:
  RankRuntime(int rank, int world, da_allgather_fn allgather, void* ctx) {
    check(da_rank_create(rank, world, allgather, ctx, &h_));
  }
  /// opts.transport: DA_TRANSPORT_NCCL (send/recv per phase on a side stream),
  /// DA_TRANSPORT_IPC (copy-engine pulls) or DA_TRANSPORT_NONE (no-comm arm);
  /// opts.deterministic: bitwise-reproducible backward.
  RankRuntime(int rank, int world, da_allgather_fn allgather, void* ctx,
              const da_rank_options& opts) {
    check(da_rank_create_ex(rank, world, allgather, ctx, &opts, &h_));
  }
  ~RankRuntime() { da_rank_destroy(h_); }
  RankRuntime(const RankRuntime&) = delete;
  RankRuntime& operator=(const RankRuntime&) = delete;

  /// run_forward for this rank's chunk; out / lse are kept as the backward's
  /// saved state (the attention forward is never recomputed).
  CommCounters forward(const Chunk& q, const Chunk& k, const Chunk& v, void* out, float* lse,
                       da_schedule_kind kind, cudaStream_t st) {
    da_counters c{};
    check(da_rank_forward(h_, kind, q.data, k.data, v.data, q.heads, k.heads, q.rows, out, lse,
                          &c, st));
    return to_counters(c);
  }
  CommCounters backward(const void* d_out, float* dq, float* dk, float* dv, da_schedule_kind kind,
                        cudaStream_t st) {
    da_counters c{};
    check(da_rank_backward(h_, kind, d_out, dq, dk, dv, &c, st));
    return to_counters(c);
  }

 private:
  da_rank* h_ = nullptr;
};

}  // namespace b200
}  // namespace distattn

#endif  // DISTATTN_B200_HPP
