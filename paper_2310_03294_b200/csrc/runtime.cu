// Device executor for P logical sequence-parallel workers on ONE GPU.
//
// This is the reference's stepper executor (runtime.cpp:266-330 forward,
// :605-651 backward) with every per-chunk "kernel" a real sm_100a launch.
// All shards live in one address space, so a message is the consumer
// kernel reading the producer's buffer directly (zero-copy, the single-box
// analogue of an NVSwitch peer read); counters still account each payload
// exactly like count_message (runtime.cpp:50-83), scaled by the head count.
//
// Per-worker operation order is the reference's: at step t every worker's
// primary task runs in ascending worker order, then the step's merges in
// schedule order (helper-ascending) — runtime.cpp:286-328.
#include <cuda_runtime.h>

#include <cmath>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "capi_internal.h"
#include "kernels.h"
#include "schedule_impl.h"

namespace da {
namespace {

struct Workspace {
  int P = 0;
  int64_t h_q = 0, rows = 0;
  std::vector<float*> o, m, l;  // per worker running accumulator
  std::vector<float*> po, pm, pl;  // per worker helper-partial slot
  std::vector<float*> dvec;       // per worker D (backward)
  void* kv_half = nullptr;        // packed k, v row half (split schedule), bf16
  size_t kv_half_bytes = 0;
  void* dkv_half = nullptr;       // dk, dv of a kv row half (split backward), fp32
  size_t dkv_half_bytes = 0;
  int* flag = nullptr;
  std::vector<void*> allocs;
  cudaStream_t stream = nullptr;

  void release() {
    for (void* p : allocs) cudaFree(p);
    allocs.clear();
    o.clear(); m.clear(); l.clear(); po.clear(); pm.clear(); pl.clear(); dvec.clear();
    flag = nullptr;
    kv_half = nullptr;
    kv_half_bytes = 0;
    dkv_half = nullptr;
    dkv_half_bytes = 0;
    P = 0;
  }

  // grows one of the split-schedule buffers (kv_half / dkv_half) to `bytes`
  cudaError_t grow(void** buf, size_t* cap, size_t bytes) {
    if (*cap >= bytes) return cudaSuccess;
    if (*buf) {
      cudaFree(*buf);
      for (auto& a : allocs)
        if (a == *buf) a = nullptr;
      *buf = nullptr;
      *cap = 0;
    }
    cudaError_t e = cudaMalloc(buf, bytes);
    if (e != cudaSuccess) return e;
    allocs.push_back(*buf);
    *cap = bytes;
    return cudaSuccess;
  }
  ~Workspace() { release(); }

  cudaError_t ensure(int P_, int64_t h_q_, int64_t rows_) {
    if (P_ == P && h_q_ == h_q && rows_ == rows) return cudaSuccess;
    if (!allocs.empty()) cudaStreamSynchronize(stream);  // in-flight users of the old buffers
    release();
    const size_t acc = static_cast<size_t>(h_q_) * rows_;
    auto get = [&](size_t bytes, void** out) {
      cudaError_t e = cudaMalloc(out, bytes);
      if (e == cudaSuccess) allocs.push_back(*out);
      return e;
    };
    for (int w = 0; w < P_; ++w) {
      void* buf = nullptr;
      // o, m, l, po, pm, pl, dvec
      cudaError_t e = get(acc * 4 * (2 * 128 + 5), &buf);
      if (e != cudaSuccess) { release(); return e; }
      float* f = static_cast<float*>(buf);
      o.push_back(f); f += acc * 128;
      po.push_back(f); f += acc * 128;
      m.push_back(f); f += acc;
      l.push_back(f); f += acc;
      pm.push_back(f); f += acc;
      pl.push_back(f); f += acc;
      dvec.push_back(f);
    }
    void* fl = nullptr;
    cudaError_t e = get(sizeof(int), &fl);
    if (e != cudaSuccess) { release(); return e; }
    flag = static_cast<int*>(fl);
    P = P_;
    h_q = h_q_;
    rows = rows_;
    return cudaSuccess;
  }
};

// One workspace per stream: executors on different streams (or threads) never
// share accumulators; calls on one stream are serialised by the stream.
// A workspace is resized only after its stream drained (ensure() below).
std::mutex g_ws_mu;
std::map<cudaStream_t, std::unique_ptr<Workspace>> g_ws_map;

Workspace& workspace_for(cudaStream_t st) {
  std::lock_guard<std::mutex> lock(g_ws_mu);
  auto& w = g_ws_map[st];
  if (!w) w.reset(new Workspace());
  w->stream = st;
  return *w;
}

// Packs rows [r0, r0 + n) of every head of a bf16 [h, rows, d] chunk into a
// contiguous [h, n, d] buffer (a strided 2-D copy: one row block per head).
cudaError_t pack_rows(const void* src, void* dst, int64_t h, int64_t rows, int64_t r0, int64_t n,
                      int64_t d, cudaStream_t st) {
  const size_t pitch_src = static_cast<size_t>(rows) * d * 2;
  const size_t width = static_cast<size_t>(n) * d * 2;
  return cudaMemcpy2DAsync(dst, width, static_cast<const char*>(src) + r0 * d * 2, pitch_src, width,
                           h, cudaMemcpyDeviceToDevice, st);
}

da_status check_shards(const da_shards* s, bool backward) {
  if (s == nullptr) return set_error(DA_ERR_CONFIG, "null shards");
  if (s->workers < 1) return set_error(DA_ERR_CONFIG, "need at least 1 worker");
  if (s->d != 128) return set_error(DA_ERR_UNSUPPORTED, "d must be 128");
  if (s->rows < 1) return set_error(DA_ERR_CONFIG, "tokens and d must be positive");
  if (s->h_q < 1 || s->h_kv < 1 || s->h_q % s->h_kv != 0)
    return set_error(DA_ERR_SHAPE, "h_q must be a positive multiple of h_kv");
  for (int w = 0; w < s->workers; ++w) {
    if (!s->q[w] || !s->k[w] || !s->v[w])
      return set_error(DA_ERR_SHAPE, "all shards must share the same q/k/v shape");
    if (backward) {
      if (!s->out[w] || !s->lse[w])
        return set_error(DA_ERR_STATE, "run_backward requires forward output and logsumexp");
      if (!s->d_out[w]) return set_error(DA_ERR_STATE, "run_backward requires d_out on every shard");
      if (!s->dq[w] || !s->dk[w] || !s->dv[w])
        return set_error(DA_ERR_CONFIG, "run_backward: missing gradient buffers");
    } else if (!s->out[w] || !s->lse[w]) {
      return set_error(DA_ERR_CONFIG, "run_forward: missing output buffers");
    }
  }
  return DA_OK;
}

struct Tally {
  da_counters c{};
  int held = 0, max_held = 0;
  void acquire() { ++held; max_held = held > max_held ? held : max_held; }
  void release() { --held; }
};

void count(da_counters& c, int kind, int64_t rows, int64_t d, int64_t heads) {
  switch (kind) {
    case kMsgKV: c.kv_scalars += 2 * rows * d * heads; ++c.kv_messages; break;
    case kMsgQ: c.q_scalars += rows * d * heads; ++c.q_messages; break;
    case kMsgPartial: c.partial_scalars += rows * (d + 2) * heads; ++c.partial_messages; break;
    case kMsgGradKV: c.grad_scalars += 2 * rows * d * heads; ++c.grad_messages; break;
    case kMsgKVHalf: c.kv_scalars += 2 * rows * d * heads; ++c.kv_messages; break;
  }
}

da_status fwd_update(const da_shards* s, int qw, int kvw, float* o_in, float* m_in, float* l_in,
                     float* o, float* m, float* l, int mask, cudaStream_t st) {
  da_fwd_args a{};
  a.q = s->q[qw - 1];
  a.k = s->k[kvw - 1];
  a.v = s->v[kvw - 1];
  a.h_q = s->h_q;
  a.h_kv = s->h_kv;
  a.rows_q = s->rows;
  a.rows_kv = s->rows;
  a.d = s->d;
  a.o_in = o_in;
  a.m_in = m_in;
  a.l_in = l_in;
  a.o_acc = o;
  a.m_acc = m;
  a.l_acc = l;
  a.scale = 0.f;
  a.mask = mask;
  a.finalize = 0;
  return da_attn_fwd_chunk(&a, st);
}

}  // namespace
}  // namespace da

using namespace da;

extern "C" {

void da_runtime_release(void) {
  std::lock_guard<std::mutex> lock(g_ws_mu);
  for (auto& kv : g_ws_map) {
    cudaStreamSynchronize(kv.first);
    kv.second->release();
  }
  g_ws_map.clear();
}

static FlatSchedule flat_from_table(int workers, int32_t steps, const int32_t* tasks,
                                    int64_t n_tasks, const int32_t* messages,
                                    int64_t n_messages) {
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

// The device executor over ANY schedule that passes the reference's
// validator (schedule.cpp:121-258) — the built-in kinds or a caller's table.
static da_status run_forward_flat(const da_shards* s, const FlatSchedule& sch,
                                  da_counters* counters, void* stream) {
  da_status rc = check_shards(s, false);
  if (rc != DA_OK) return rc;
  const int P = s->workers;
  if (sch.workers != P)
    return set_error(DA_ERR_SCHEDULE, "schedule worker count does not match the shards");
  const auto errs = validate_flat(sch);
  if (!errs.empty())
    return set_error(DA_ERR_SCHEDULE, "invalid schedule: " + errs.front() + " (" +
                                          std::to_string(errs.size()) + " violations)");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Workspace& g_ws = workspace_for(st);
  cudaError_t e = g_ws.ensure(P, s->h_q, s->rows);
  if (e != cudaSuccess) return cuda_error(e, "run_forward workspace");

  std::vector<Tally> tally(P);
  std::vector<bool> started(P, false);  // accumulator holds data (else fresh)
  for (int t = 0; t < sch.steps; ++t) {
    for (const Task& k : sch.tasks) {
      if (k.step != t || k.kind == kIdle || k.kind == kMerge) continue;
      const int w = k.worker;
      Tally& me = tally[w - 1];
      ++me.c.attention_kernel_calls;
      float* o = g_ws.o[w - 1];
      float* m = g_ws.m[w - 1];
      float* l = g_ws.l[w - 1];
      if (k.kind == kLocal) {
        rc = fwd_update(s, w, w, started[w - 1] ? o : nullptr, m, l, o, m, l, DA_MASK_DIAGONAL, st);
        started[w - 1] = true;
      } else if (k.helper != kPartWhole) {  // split step: one half of the kv rows
        const int64_t lo = s->rows / 2;
        const int64_t r0 = k.helper == kPartLow ? 0 : lo;
        const int64_t n = k.helper == kPartLow ? lo : s->rows - lo;
        const size_t bytes = static_cast<size_t>(s->h_kv) * (s->rows - lo) * s->d * 2 * 2;
        e = g_ws.grow(&g_ws.kv_half, &g_ws.kv_half_bytes, bytes);
        if (e != cudaSuccess) return cuda_error(e, "run_forward split workspace");
        void* kh = g_ws.kv_half;
        void* vh = static_cast<char*>(g_ws.kv_half) + bytes / 2;
        e = pack_rows(s->k[k.kv_owner - 1], kh, s->h_kv, s->rows, r0, n, s->d, st);
        if (e == cudaSuccess) e = pack_rows(s->v[k.kv_owner - 1], vh, s->h_kv, s->rows, r0, n, s->d, st);
        if (e != cudaSuccess) return cuda_error(e, "run_forward split pack");
        da_fwd_args a{};
        a.q = s->q[k.query_owner - 1];
        a.k = kh;
        a.v = vh;
        a.h_q = s->h_q;
        a.h_kv = s->h_kv;
        a.rows_q = s->rows;
        a.rows_kv = n;
        a.d = s->d;
        a.mask = DA_MASK_FULL;
        me.acquire();
        if (k.worker == k.query_owner) {  // owner: high half, accumulator in place
          count(me.c, kMsgKVHalf, n, s->d, s->h_kv);
          if (started[w - 1]) { a.o_in = o; a.m_in = m; a.l_in = l; }
          a.o_acc = o; a.m_acc = m; a.l_acc = l;
          started[w - 1] = true;
        } else {  // helper: low half of its own kv, fresh partial
          count(me.c, kMsgQ, s->rows, s->d, s->h_q);
          a.o_acc = g_ws.po[w - 1]; a.m_acc = g_ws.pm[w - 1]; a.l_acc = g_ws.pl[w - 1];
        }
        rc = da_attn_fwd_chunk(&a, st);
        me.release();
      } else if (k.worker == k.query_owner) {  // Direct: kv chunk of kv_owner
        me.acquire();
        count(me.c, kMsgKV, s->rows, s->d, s->h_kv);
        rc = fwd_update(s, w, k.kv_owner, started[w - 1] ? o : nullptr, m, l, o, m, l,
                        DA_MASK_FULL, st);
        started[w - 1] = true;
        me.release();
      } else {  // Help: owner's query against my kv, fresh partial
        me.acquire();
        count(me.c, kMsgQ, s->rows, s->d, s->h_q);
        rc = fwd_update(s, k.query_owner, w, nullptr, nullptr, nullptr, g_ws.po[w - 1],
                        g_ws.pm[w - 1], g_ws.pl[w - 1], DA_MASK_FULL, st);
        me.release();
      }
      if (rc != DA_OK) return rc;
    }
    for (const Task& k : sch.tasks) {
      if (k.step != t || k.kind != kMerge) continue;
      const int ow = k.worker, hw = k.helper;
      count(tally[ow - 1].c, kMsgPartial, s->rows, s->d, s->h_q);
      e = launch_merge(g_ws.o[ow - 1], g_ws.m[ow - 1], g_ws.l[ow - 1], g_ws.po[hw - 1],
                       g_ws.pm[hw - 1], g_ws.pl[hw - 1], g_ws.o[ow - 1], g_ws.m[ow - 1],
                       g_ws.l[ow - 1], s->h_q * s->rows, st);
      if (e != cudaSuccess) return cuda_error(e, "run_forward merge");
    }
  }
  e = cudaMemsetAsync(g_ws.flag, 0, sizeof(int), st);
  for (int w = 0; w < P && e == cudaSuccess; ++w)
    e = launch_finalize(g_ws.o[w], g_ws.m[w], g_ws.l[w], s->out[w], s->lse[w], g_ws.flag,
                        s->h_q * s->rows, st);
  if (e != cudaSuccess) return cuda_error(e, "run_forward finalize");
  if (counters) {
    da_counters c{};
    for (const Tally& ty : tally) {
      c.kv_scalars += ty.c.kv_scalars; c.q_scalars += ty.c.q_scalars;
      c.partial_scalars += ty.c.partial_scalars; c.grad_scalars += ty.c.grad_scalars;
      c.kv_messages += ty.c.kv_messages; c.q_messages += ty.c.q_messages;
      c.partial_messages += ty.c.partial_messages; c.grad_messages += ty.c.grad_messages;
      c.attention_kernel_calls += ty.c.attention_kernel_calls;
      c.max_remote_chunks_held = ty.max_held > c.max_remote_chunks_held ? ty.max_held
                                                                         : c.max_remote_chunks_held;
    }
    *counters = c;
  }
  return da_check_degenerate(g_ws.flag, stream);
}

da_status da_run_backward(const da_shards* s, da_counters* counters, void* stream) {
  return da_run_backward_sched(s, DA_SCHEDULE_RING_BWD, counters, stream);
}

// Backward over a ring or balanced backward schedule. Every pair (q chunk p,
// kv chunk r) is one block_attn_backward launch; dq goes to p's accumulator,
// dk/dv to r's (zero-copy GradKV / local for helpers). Ring order reproduces
// runtime.cpp:605-651; balanced order follows make_balanced_backward. A split
// step's halves (make_balanced_split_backward) pack the kv rows, compute into
// a half-size dk/dv and fold it into the kv owner's rows.
static da_status run_backward_flat(const da_shards* s, const FlatSchedule& sch,
                                   da_counters* counters, void* stream) {
  da_status rc = check_shards(s, true);
  if (rc != DA_OK) return rc;
  const int P = s->workers;
  if (sch.workers != P)
    return set_error(DA_ERR_SCHEDULE, "schedule worker count does not match the shards");
  const auto errs = validate_backward_flat(sch);
  if (!errs.empty())
    return set_error(DA_ERR_SCHEDULE, "invalid schedule: " + errs.front() + " (" +
                                          std::to_string(errs.size()) + " violations)");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Workspace& g_ws = workspace_for(st);
  cudaError_t e = g_ws.ensure(P, s->h_q, s->rows);
  if (e != cudaSuccess) return cuda_error(e, "run_backward workspace");
  const int64_t q_elems = s->h_q * s->rows * 128;
  const int64_t kv_elems = s->h_kv * s->rows * 128;
  for (int w = 0; w < P; ++w) {
    e = cudaMemsetAsync(s->dq[w], 0, q_elems * 4, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(s->dk[w], 0, kv_elems * 4, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(s->dv[w], 0, kv_elems * 4, st);
    if (e == cudaSuccess)
      e = launch_bwd_preprocess(s->d_out[w], s->out[w], g_ws.dvec[w], s->h_q * s->rows, st);
    if (e != cudaSuccess) return cuda_error(e, "run_backward setup");
  }
  std::vector<Tally> tally(P);
  // one pair (q chunk qw, kv chunk kvw) on kv rows [r0, r0 + n) (part of the
  // split step: packed k/v half in, that half's dk/dv folded into kvw's rows)
  const int64_t lo = s->rows / 2;
  auto chunk_part = [&](int qw, int kvw, int part) -> da_status {
    const int64_t r0 = part == kPartHigh ? lo : 0;
    const int64_t n = part == kPartLow ? lo : s->rows - lo;
    const size_t kv_b = static_cast<size_t>(s->h_kv) * (s->rows - lo) * s->d * 2;
    const size_t g_b = static_cast<size_t>(s->h_kv) * (s->rows - lo) * s->d * 4;
    cudaError_t e2 = g_ws.grow(&g_ws.kv_half, &g_ws.kv_half_bytes, 2 * kv_b);
    if (e2 == cudaSuccess) e2 = g_ws.grow(&g_ws.dkv_half, &g_ws.dkv_half_bytes, 2 * g_b);
    if (e2 != cudaSuccess) return cuda_error(e2, "run_backward split workspace");
    void* kh = g_ws.kv_half;
    void* vh = static_cast<char*>(g_ws.kv_half) + kv_b;
    float* gk = static_cast<float*>(g_ws.dkv_half);
    float* gv = reinterpret_cast<float*>(static_cast<char*>(g_ws.dkv_half) + g_b);
    e2 = pack_rows(s->k[kvw - 1], kh, s->h_kv, s->rows, r0, n, s->d, st);
    if (e2 == cudaSuccess) e2 = pack_rows(s->v[kvw - 1], vh, s->h_kv, s->rows, r0, n, s->d, st);
    if (e2 != cudaSuccess) return cuda_error(e2, "run_backward split pack");
    da_bwd_args a{};
    a.q = s->q[qw - 1];
    a.k = kh;
    a.v = vh;
    a.d_out = s->d_out[qw - 1];
    a.lse = s->lse[qw - 1];
    a.d_vec = g_ws.dvec[qw - 1];
    a.h_q = s->h_q;
    a.h_kv = s->h_kv;
    a.rows_q = s->rows;
    a.rows_kv = n;
    a.d = s->d;
    a.dq_acc = s->dq[qw - 1];
    a.dk_acc = gk;
    a.dv_acc = gv;
    a.accumulate_kv = 0;
    a.scale = 0.f;
    a.mask = DA_MASK_FULL;
    da_status r2 = da_attn_bwd_chunk(&a, st);
    if (r2 != DA_OK) return r2;
    e2 = launch_add_rows(s->dk[kvw - 1], gk, s->h_kv, s->rows, r0, n, st);
    if (e2 == cudaSuccess) e2 = launch_add_rows(s->dv[kvw - 1], gv, s->h_kv, s->rows, r0, n, st);
    return e2 == cudaSuccess ? DA_OK : cuda_error(e2, "run_backward split fold");
  };
  auto chunk = [&](int qw, int kvw, int mask) {
    da_bwd_args a{};
    a.q = s->q[qw - 1];
    a.k = s->k[kvw - 1];
    a.v = s->v[kvw - 1];
    a.d_out = s->d_out[qw - 1];
    a.lse = s->lse[qw - 1];
    a.d_vec = g_ws.dvec[qw - 1];
    a.h_q = s->h_q;
    a.h_kv = s->h_kv;
    a.rows_q = s->rows;
    a.rows_kv = s->rows;
    a.d = s->d;
    a.dq_acc = s->dq[qw - 1];
    a.dk_acc = s->dk[kvw - 1];
    a.dv_acc = s->dv[kvw - 1];
    a.accumulate_kv = 1;
    a.scale = 0.f;
    a.mask = mask;
    return da_attn_bwd_chunk(&a, st);
  };
  const int64_t R = s->rows, D = s->d;
  for (int t = 0; t < sch.steps; ++t) {
    for (const Task& k : sch.tasks) {
      if (k.step != t || k.kind == kIdle || k.kind == kMerge) continue;
      const int w = k.worker;
      Tally& me = tally[w - 1];
      ++me.c.attention_kernel_calls;
      const int part = k.kind == kRemote ? k.helper : kPartWhole;
      if (k.kind == kLocal) {
        rc = chunk(w, w, DA_MASK_DIAGONAL);
      } else if (k.worker == k.query_owner) {  // direct: KV (half) in, GradKV out
        count(me.c, part == kPartWhole ? kMsgKV : kMsgKVHalf,
              part == kPartWhole ? R : R - lo, D, s->h_kv);
        me.acquire();
        rc = part == kPartWhole ? chunk(w, k.kv_owner, DA_MASK_FULL)
                                : chunk_part(w, k.kv_owner, part);
        me.release();
      } else {  // helper: (q, dO, lse, D) bundle in, dq partial out
        me.acquire();
        me.c.q_scalars += R * (2 * D + 2) * s->h_q;
        ++me.c.q_messages;
        rc = part == kPartWhole ? chunk(k.query_owner, w, DA_MASK_FULL)
                                : chunk_part(k.query_owner, w, part);
        me.release();
      }
      if (rc != DA_OK) return rc;
    }
    // GradKV folds (ascending kv owner as runtime.cpp:636-649) and dq partial
    // folds (the schedule's merge order) — accounting only: the kernels above
    // already accumulated into the owners' buffers.
    for (const Message& m : sch.messages) {
      if (m.step != t) continue;
      if (m.kind == kMsgGradKV) {
        Tally& me = tally[m.to - 1];
        int part = kPartWhole;  // the sender's direct task of this step: a half's GradKV
        for (const Task& k : sch.tasks)
          if (k.step == t && k.kind == kRemote && k.worker == m.from && k.query_owner == m.from)
            part = k.helper;
        count(me.c, kMsgGradKV, part == kPartWhole ? R : (part == kPartLow ? lo : R - lo), D,
              s->h_kv);
        me.acquire();
        me.release();
      } else if (m.kind == kMsgPartial) {
        Tally& me = tally[m.to - 1];
        me.c.partial_scalars += R * D * s->h_q;
        ++me.c.partial_messages;
      }
    }
  }
  if (counters) {
    da_counters c{};
    for (const Tally& ty : tally) {
      c.kv_scalars += ty.c.kv_scalars; c.q_scalars += ty.c.q_scalars;
      c.partial_scalars += ty.c.partial_scalars; c.grad_scalars += ty.c.grad_scalars;
      c.kv_messages += ty.c.kv_messages; c.q_messages += ty.c.q_messages;
      c.partial_messages += ty.c.partial_messages; c.grad_messages += ty.c.grad_messages;
      c.attention_kernel_calls += ty.c.attention_kernel_calls;
      c.max_remote_chunks_held = ty.max_held > c.max_remote_chunks_held ? ty.max_held
                                                                         : c.max_remote_chunks_held;
    }
    *counters = c;
  }
  return DA_OK;
}

da_status da_run_forward(const da_shards* s, int schedule_kind, da_counters* counters,
                         void* stream) {
  if (s == nullptr) return set_error(DA_ERR_CONFIG, "null shards");
  const int P = s->workers;
  if (P < 1) return set_error(DA_ERR_CONFIG, "need at least 1 worker");
  if (schedule_kind == DA_SCHEDULE_RING) return run_forward_flat(s, make_ring(P), counters, stream);
  if (schedule_kind == DA_SCHEDULE_BALANCED)
    return run_forward_flat(s, make_balanced(P), counters, stream);
  if (schedule_kind == DA_SCHEDULE_BALANCED_SPLIT)
    return run_forward_flat(s, make_balanced_split(P), counters, stream);
  return set_error(DA_ERR_CONFIG, "unknown schedule kind");
}

da_status da_run_forward_table(const da_shards* s, int32_t steps, const int32_t* tasks,
                               int64_t n_tasks, const int32_t* messages, int64_t n_messages,
                               da_counters* counters, void* stream) {
  if (s == nullptr) return set_error(DA_ERR_CONFIG, "null shards");
  return run_forward_flat(s, flat_from_table(s->workers, steps, tasks, n_tasks, messages,
                                             n_messages),
                          counters, stream);
}

da_status da_run_backward_sched(const da_shards* s, int schedule_kind, da_counters* counters,
                                void* stream) {
  if (s == nullptr) return set_error(DA_ERR_CONFIG, "null shards");
  const int P = s->workers;
  if (P < 1) return set_error(DA_ERR_CONFIG, "need at least 1 worker");
  if (schedule_kind == DA_SCHEDULE_RING_BWD || schedule_kind == DA_SCHEDULE_RING)
    return run_backward_flat(s, make_ring_backward(P), counters, stream);
  if (schedule_kind == DA_SCHEDULE_BALANCED_BWD || schedule_kind == DA_SCHEDULE_BALANCED)
    return run_backward_flat(s, make_balanced_backward(P), counters, stream);
  if (schedule_kind == DA_SCHEDULE_BALANCED_SPLIT_BWD || schedule_kind == DA_SCHEDULE_BALANCED_SPLIT)
    return run_backward_flat(s, make_balanced_split_backward(P), counters, stream);
  return set_error(DA_ERR_CONFIG, "unknown schedule kind");
}

da_status da_run_backward_table(const da_shards* s, int32_t steps, const int32_t* tasks,
                                int64_t n_tasks, const int32_t* messages, int64_t n_messages,
                                da_counters* counters, void* stream) {
  if (s == nullptr) return set_error(DA_ERR_CONFIG, "null shards");
  return run_backward_flat(s, flat_from_table(s->workers, steps, tasks, n_tasks, messages,
                                              n_messages),
                           counters, stream);
}

}  // extern "C"
