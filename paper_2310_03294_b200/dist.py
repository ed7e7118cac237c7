"""Python model of the per-rank protocol (one process per rank), for the
host-logic tests and the wall-clock trace export.

The production multi-GPU path is the native per-rank runtime
(csrc/rank_runtime.cu, ``rank.RankRuntime``), which bench.py runs. This module
restates the same schedule-driven protocol in Python over a pluggable compute
backend so that the CPU suite can run it under gloo, bit-exactly against the
oracle stepper (tests/test_dist_gloo.py), and it records the reference's
trace schema (``Recorder``/``gather_trace``, runtime.cpp:752-797).

The per-rank plan comes from the native schedule (csrc/schedule.cpp, bit-exact
with schedule.cpp:60-108); the operation order per worker is the reference's
(runtime.cpp:266-330 forward, :605-651 backward):

forward (ring or load-balanced), worker w at step t:
    Local   — update(q_w, k_w, v_w, Diagonal)          (fresh accumulator)
    Direct  — recv KV(r); update(q_w, k_r, v_r, Full)  (accumulator in place)
    Help    — recv Q(o);  partial = update(q_o, k_w, v_w, Full, fresh); send Partial -> o
    then merges at the owner: recv Partial(h); acc = rescale(acc, partial)
    finally finalize -> out (bf16) and lse (fp32), the state the backward reuses
    (rematerialization-aware checkpointing: the forward is never recomputed).
backward (ring, BackwardMode::Vanilla), worker p at step t:
    t = 0: grads(q_p, k_p, v_p, Diagonal)
    t >= 1, p > t: recv KV(p - t); grads(q_p, k_r, v_r, Full); send GradKV -> r
    worker r folds GradKV from r + t.

Communication: every message is a point-to-point NCCL send/recv issued on a
dedicated comm stream. Immutable operands (KV, Q) of step t+1 are posted while
step t computes (prefetch depth 1, double-buffered receive slots — the
reference's residency bound of 2, acceptance_main.cpp:414-444); the compute
stream waits on the receive before the consuming kernel. Partials and GradKV
leave right after the kernel that produced them.

The compute backend is pluggable so the host logic runs on CPU under gloo in
the test-suite; the production backend (CudaBackend) is the sm_100a library.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass

import torch
import torch.distributed as tdist

from .schedule import (KVPart, TaskKind, build_balanced_backward_schedule,
                       build_balanced_schedule, build_balanced_split_schedule,
                       build_ring_backward_schedule, build_ring_schedule, validate,
                       validate_backward)
from .errors import ConfigError, ScheduleError, StateError


# ----------------------------------------------------------------------------- compute backend
class CudaBackend:
    """sm_100a kernels through the C ABI (flashcore)."""

    acc_dtype = torch.float32
    grad_dtype = torch.float32

    def __init__(self, device):
        from . import flashcore as F
        self.F = F
        self.device = device

    def new_acc(self, h, rows, d, packed: torch.Tensor | None = None):
        if packed is None:
            packed = torch.empty(h * rows * (d + 2), dtype=self.acc_dtype, device=self.device)
        o = packed[: h * rows * d].view(h, rows, d)
        m = packed[h * rows * d: h * rows * (d + 1)].view(h, rows)
        l = packed[h * rows * (d + 1):].view(h, rows)
        return self.F.AttnAccumulator(o, m, l), packed

    def update(self, q, k, v, acc_in, mask: str, out_acc):
        F = self.F
        mm = F.MaskMode.Diagonal if mask == "diagonal" else F.MaskMode.Full
        return F.block_attn_update(q, k, v, acc_in, mm, out=out_acc)

    def merge(self, acc, part):
        return self.F.rescale(acc, part, out=acc)

    def finalize(self, acc):
        o = self.F.finalize(acc)
        return o.o, o.lse

    def bwd_aux(self, d_out, out):
        return self.F.backward_aux(d_out, out)

    def grads(self, q, k, v, lse, d_out, d_vec, mask: str, dq, dk, dv, accumulate_kv: bool):
        """dq += contribution; dk/dv += (accumulate_kv) or = contribution."""
        F = self.F
        mm = F.MaskMode.Diagonal if mask == "diagonal" else F.MaskMode.Full
        F.block_attn_backward(q, k, v, None, lse, d_out, mm, d_vec=d_vec,
                              grads=F.ChunkGrads(dq, dk, dv), accumulate_kv=accumulate_kv)

    def add_(self, dst, src):
        dst.add_(src)


# ----------------------------------------------------------------------------- transport
class Transport:
    """Point-to-point messages over torch.distributed (NCCL on GPU, gloo on CPU).

    Ranks are 0-based; schedule workers are rank + 1. A receive is
    (slot, src_rank, key): the key names the sender's published tensor and is
    only used by the pull-based PeerTransport."""

    def __init__(self, group=None):
        self.group = group
        self.nccl = tdist.get_backend(group) == "nccl"
        self.cuda = self.nccl
        self.stream = torch.cuda.Stream() if self.nccl else None

    def publish(self, tensors: dict):
        """No-op: NCCL/gloo move data by send/recv pairs."""

    def exchange(self, sends, recvs):
        """Posts sends [(tensor, dst_rank)] and recvs [(tensor, src_rank, key)] as
        one group. On NCCL the group starts only after everything already
        enqueued on the current (compute) stream — so send data is produced and
        receive slots are no longer read — and the returned handle's wait()
        orders the current stream after the whole group. On gloo wait() blocks."""
        if not sends and not recvs:
            return _Done()
        sends = [(x[0], x[1]) for x in sends]
        recvs = [(x[0], x[1]) for x in recvs]
        if self.nccl:
            ready = torch.cuda.Event()
            ready.record()
            with torch.cuda.stream(self.stream):
                self.stream.wait_event(ready)
                ops = [tdist.P2POp(tdist.isend, t, r, self.group) for t, r in sends] + \
                      [tdist.P2POp(tdist.irecv, t, r, self.group) for t, r in recvs]
                works = tdist.batch_isend_irecv(ops)
            return _Works(works)
        works = [tdist.isend(t, r, self.group) for t, r in sends] + \
                [tdist.irecv(t, r, self.group) for t, r in recvs]
        return _Works(works)


class PeerTransport:
    """Peer-memory transport: copy-engine pulls from the other ranks' HBM.

    Every rank publishes the tensors it sends (CUDA IPC mappings, exchanged
    once per buffer with a host all_gather_object and cached); a receive is a
    cudaMemcpyAsync on a side stream straight from the sender's tensor into
    the local slot — over NVLink between GPUs, with no NCCL kernels, so the
    attention kernels keep every SM. Ordering is carried by 32-bit counters in
    device memory (csrc/peer.cu): per destination a "ready" counter bumped on
    the sender's compute stream when the data is produced, per source a
    "done" counter bumped after the pull. The receiver's side stream waits on
    the sender's ready counter, the sender's wait() on the receiver's done
    counter — all in-stream, no host synchronisation on the data path.
    Messages between a pair are matched by order, exactly as the schedule
    emits them on both sides.
    """

    def __init__(self, group=None, device=None):
        from torch.multiprocessing.reductions import reduce_tensor
        from . import _lib
        self._reduce = reduce_tensor
        self.lib = _lib.lib()
        self.group = group
        self.nccl = False
        self.cuda = True
        self.rank = tdist.get_rank(group)
        self.world = tdist.get_world_size(group)
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.stream = torch.cuda.Stream(self.device)
        w = self.world
        # [0, w): ready counters, one per destination; [w, 2w): done counters, one per source
        self.flags = torch.zeros(2 * w, dtype=torch.int32, device=self.device)
        self.sent = [0] * w
        self.pulled = [0] * w
        self._mine = {}     # key -> (data_ptr, numel, dtype) last published
        self.remote = {}    # (rank, key) -> tensor mapped from the peer
        self.remote_flags = [self.flags] * w
        if w > 1:
            allf = self._gather({"__flags__": self._reduce(self.flags)})
            for r, d in enumerate(allf):
                if r != self.rank:
                    self.remote_flags[r] = self._rebuild(d["__flags__"])

    @staticmethod
    def _rebuild(red):
        fn, args = red
        return fn(*args)

    def _gather(self, obj):
        out = [None] * self.world
        tdist.all_gather_object(out, obj, group=self.group)
        return out

    def publish(self, tensors: dict):
        """Collective: makes `tensors` pullable by every peer under their keys."""
        if self.world == 1:
            return
        mine = {}
        for key, t in tensors.items():
            sig = (t.data_ptr(), t.numel(), t.dtype)
            if self._mine.get(key) != sig:
                mine[key] = self._reduce(t)
                self._mine[key] = sig
        for r, d in enumerate(self._gather(mine)):
            if r == self.rank:
                continue
            for key, red in d.items():
                self.remote[(r, key)] = self._rebuild(red)

    def _write(self, stream, idx, value):
        from .errors import check
        check(self.lib.da_stream_write_u32(C.c_void_p(stream.cuda_stream),
                                           C.c_void_p(self.flags.data_ptr() + 4 * idx),
                                           value & 0xFFFFFFFF))

    def _wait(self, stream, rank, idx, value):
        from .errors import check
        check(self.lib.da_stream_wait_u32_geq(
            C.c_void_p(stream.cuda_stream),
            C.c_void_p(self.remote_flags[rank].data_ptr() + 4 * idx), value & 0xFFFFFFFF))

    def exchange(self, sends, recvs):
        if not sends and not recvs:
            return _Done()
        cur = torch.cuda.current_stream(self.device)
        w, me = self.world, self.rank
        expect = {}
        for x in sends:
            dst = x[1]
            self.sent[dst] += 1
            self._write(cur, dst, self.sent[dst])  # produced in stream order on `cur`
            expect[dst] = self.sent[dst]
        done = None
        if recvs:
            ready = torch.cuda.Event()
            ready.record(cur)  # receive slots are no longer read by earlier work
            self.stream.wait_event(ready)
            with torch.cuda.stream(self.stream):
                for slot, src, key in recvs:
                    self.pulled[src] += 1
                    self._wait(self.stream, src, me, self.pulled[src])
                    slot.copy_(self.remote[(src, key)], non_blocking=True)
                    self._write(self.stream, w + src, self.pulled[src])
            done = torch.cuda.Event()
            done.record(self.stream)
        return _PeerWork(self, cur, done, expect)


class _PeerWork:
    def __init__(self, tr, stream, done, expect):
        self.tr, self.stream, self.done, self.expect = tr, stream, done, expect

    def wait(self):
        cur = torch.cuda.current_stream(self.tr.device)
        if self.done is not None:
            cur.wait_event(self.done)
        for dst, n in self.expect.items():  # the peers pulled what I sent
            self.tr._wait(cur, dst, self.tr.world + self.tr.rank, n)


class _Done:
    def wait(self):
        pass


class _Works:
    def __init__(self, works):
        self.works = works

    def wait(self):
        for w in self.works:
            w.wait()


# ----------------------------------------------------------------------------- plans
@dataclass
class StepPlan:
    action: str = "idle"     # idle | local | direct | help
    peer: int = 0            # 1-based: kv owner (direct) or query owner (help)
    kv_sends: tuple = ()     # destinations (1-based) of my KV this step
    q_sends: tuple = ()      # destinations of my Q this step
    merges: tuple = ()       # helpers (1-based) whose partial I merge this step, in order
    part: int = 0            # kv rows of the pair: KVPart (split schedule extension)
    kvh_sends: tuple = ()    # destinations of the high half of my KV rows (KVHalf)


def forward_plan(schedule, worker: int) -> list[StepPlan]:
    """Per-worker view of a validated schedule (runtime.cpp:138-177)."""
    plans = []
    for t, step in enumerate(schedule.steps):
        p = StepPlan()
        for task in step:
            if task.worker != worker:
                continue
            if task.kind == TaskKind.LocalAttn:
                p.action = "local"
            elif task.kind == TaskKind.RemoteAttn:
                if task.query_owner == worker:
                    p.action, p.peer = "direct", task.kv_owner
                else:
                    p.action, p.peer = "help", task.query_owner
                p.part = int(task.kv_part)
            elif task.kind == TaskKind.RescaleMerge:
                p.merges += (task.helper,)
        p.kv_sends = tuple(m.to for m in schedule.messages
                           if m.step == t and m.from_ == worker and int(m.kind) == 0)
        p.kvh_sends = tuple(m.to for m in schedule.messages
                            if m.step == t and m.from_ == worker and int(m.kind) == 4)
        p.q_sends = tuple(m.to for m in schedule.messages
                          if m.step == t and m.from_ == worker and int(m.kind) == 1)
        plans.append(p)
    return plans


@dataclass
class BwdStepPlan:
    action: str = "idle"     # idle | local | direct | help
    peer: int = 0            # 1-based: kv owner (direct) or query owner (help)
    kv_sends: tuple = ()     # destinations of my KV this step
    q_sends: tuple = ()      # destinations of my (q, dO, lse, D) bundle
    gradkv_from: tuple = ()  # senders of GradKV folded into my dk/dv this step
    merges: tuple = ()       # helpers whose dq partial I fold this step, in order


def backward_plan(schedule, worker: int) -> list[BwdStepPlan]:
    plans = []
    for t, step in enumerate(schedule.steps):
        p = BwdStepPlan()
        for task in step:
            if task.worker != worker:
                continue
            if task.kind == TaskKind.LocalAttn:
                p.action = "local"
            elif task.kind == TaskKind.RemoteAttn:
                if task.query_owner == worker:
                    p.action, p.peer = "direct", task.kv_owner
                else:
                    p.action, p.peer = "help", task.query_owner
            elif task.kind == TaskKind.RescaleMerge:
                p.merges += (task.helper,)
        for m in schedule.messages:
            if m.step != t:
                continue
            if m.from_ == worker and int(m.kind) == 0:
                p.kv_sends += (m.to,)
            elif m.from_ == worker and int(m.kind) == 1:
                p.q_sends += (m.to,)
            elif m.to == worker and int(m.kind) == 3:
                p.gradkv_from += (m.from_,)
        plans.append(p)
    return plans


# ----------------------------------------------------------------------------- trace
_KIND = {0: "kv", 1: "q", 2: "partial", 3: "grad_kv", 4: "kv_half"}


class Recorder:
    """Per-rank wall-clock trace in the reference's ExecutionTrace terms
    (runtime.hpp:66-89): task events, messages (issue at the sender, arrival
    at the receiver) and byte-exact counters. CUDA events on GPU (resolved
    after the pass), perf_counter on CPU."""

    def __init__(self, cuda: bool, group=None, enabled: bool = True):
        import time
        self.cuda = cuda
        self.enabled = enabled
        if enabled and tdist.is_initialized() and tdist.get_world_size(group) > 1:
            tdist.barrier(group=group)  # common origin for every rank's clock
        self.origin_wall = time.time()
        self.t0 = self.mark()
        self.events = []      # (label, m0, m1)
        self.sends = []       # (key, mark)
        self.arrivals = []    # (key, mark)
        self.counters = {"kv_scalars": 0, "q_scalars": 0, "partial_scalars": 0, "grad_scalars": 0,
                         "kv_messages": 0, "q_messages": 0, "partial_messages": 0,
                         "grad_messages": 0, "kv_bytes": 0, "q_bytes": 0, "partial_bytes": 0,
                         "grad_bytes": 0}
        self.kernel_calls = 0

    def mark(self):
        if not self.enabled:
            return None
        if self.cuda:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            return e
        import time
        return time.time()

    def _ms(self, m):
        # CUDA: device time since this rank's barrier-aligned origin;
        # CPU: host wall clock (shared by the ranks of one host)
        if self.cuda:
            return self.t0.elapsed_time(m)
        return (m - self.t0) * 1e3

    def task(self, label, m0, m1, attention=True):
        self.kernel_calls += 1 if attention else 0
        if self.enabled:
            self.events.append((label, m0, m1))

    def send(self, step, kind, frm, to, mark):
        if self.enabled:
            self.sends.append(((step, kind, frm, to), mark))

    def arrive(self, step, kind, frm, to, mark, tensors, scalars_per_head_row=None):
        """Counted at the consumer like count_message (runtime.cpp:50-83):
        scalars are elements, bytes are the payload's storage."""
        if self.enabled:
            self.arrivals.append(((step, kind, frm, to), mark))
        name = {0: "kv", 1: "q", 2: "partial", 3: "grad", 4: "kv"}[kind]
        self.counters[f"{name}_scalars"] += sum(t.numel() for t in tensors)
        self.counters[f"{name}_bytes"] += sum(t.numel() * t.element_size() for t in tensors)
        self.counters[f"{name}_messages"] += 1

    def resolve(self):
        if self.cuda and self.enabled:
            torch.cuda.synchronize()
        return {"events": [(lbl, self._ms(a), self._ms(b)) for lbl, a, b in self.events],
                "sends": [(k, self._ms(m)) for k, m in self.sends],
                "arrivals": [(k, self._ms(m)) for k, m in self.arrivals],
                "counters": dict(self.counters), "kernel_calls": self.kernel_calls}


def gather_trace(rec: "Recorder", rank: int, world: int, held: int, group=None):
    """All ranks contribute; rank 0 returns the reference-schema trace dict
    (trace_to_json, runtime.cpp:752-782) and everyone else None."""
    mine = rec.resolve()
    if not rec.enabled:
        raise StateError("the pass ran without trace=True")
    if not rec.cuda:  # re-base host wall clocks on the earliest origin
        mine["origin"] = rec.origin_wall
    mine["rank"] = rank
    mine["held"] = held
    allr = [None] * world
    if world > 1:
        tdist.all_gather_object(allr, mine, group=group)
    else:
        allr = [mine]
    if rank != 0:
        return None
    if "origin" in allr[0]:
        base = min(r["origin"] for r in allr)
        for r in allr:
            sh = (r["origin"] - base) * 1e3
            r["events"] = [(lbl, a + sh, b + sh) for lbl, a, b in r["events"]]
            r["sends"] = [(k, t + sh) for k, t in r["sends"]]
            r["arrivals"] = [(k, t + sh) for k, t in r["arrivals"]]
    issue = {k: t for r in allr for k, t in r["sends"]}
    msgs = []
    for r in allr:
        for k, t in r["arrivals"]:
            msgs.append({"t_issue": issue.get(k, t), "t_arrive": t, "kind": _KIND[k[1]],
                         "from": k[2], "to": k[3]})
    msgs.sort(key=lambda m: (m["t_issue"], m["from"], m["to"]))
    counters = {}
    for r in allr:
        for c, v in r["counters"].items():
            counters[c] = counters.get(c, 0) + v
    workers = [{"worker": r["rank"] + 1,
                "events": [{"t0": a, "t1": b, "task": lbl} for lbl, a, b in r["events"]]}
               for r in sorted(allr, key=lambda r: r["rank"])]
    makespan = max((e["t1"] for w in workers for e in w["events"]), default=0.0)
    return {"workers": workers, "messages": msgs, "counters": counters,
            "attention_kernel_calls": sum(r["kernel_calls"] for r in allr),
            "max_remote_chunks_held": max(r["held"] for r in allr), "makespan": makespan,
            "time_unit": "ms"}


def trace_to_json(trace: dict) -> str:
    import json
    return json.dumps(trace, indent=2)


def trace_to_csv(trace: dict) -> str:
    """runtime.cpp:784-797 columns."""
    lines = ["worker,t0,t1,task"]
    for w in trace["workers"]:
        for e in w["events"]:
            lines.append(f"{w['worker']},{e['t0']!r},{e['t1']!r},{e['task']}")
    return "\n".join(lines) + "\n"


# ----------------------------------------------------------------------------- runtime
class DistRuntime:
    """Sequence-parallel attention for ONE rank holding chunk `rank` of the sequence.

    q/k/v: [heads, rows, d] (bf16 on GPU). Call forward() then backward(d_out).
    """

    def __init__(self, rank: int, world: int, backend=None, transport=None, device=None):
        self.rank, self.world = rank, world
        self.worker = rank + 1
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.backend = backend if backend is not None else CudaBackend(self.device)
        self.transport = transport if transport is not None else Transport()
        if self.transport.nccl and world > 1:
            # the first P2P batch must not be the group's first collective
            warm = torch.zeros(1, device=self.device)
            tdist.all_reduce(warm, group=self.transport.group)
        self.saved = None
        self.trace = {"messages_sent": 0, "bytes_sent": 0, "max_remote_chunks_held": 0}
        self._bufs = {}

    # -- buffers (allocated once per shape; not on the steady-state hot path)
    def _buf(self, key, shape, dtype):
        t = self._bufs.get(key)
        if t is None or t.shape != torch.Size(shape) or t.dtype != dtype:
            t = torch.empty(shape, dtype=dtype, device=self.device)
            self._bufs[key] = t
        return t

    def _sent(self, *tensors):
        self.trace["messages_sent"] += 1
        self.trace["bytes_sent"] += sum(t.numel() * t.element_size() for t in tensors)

    def forward(self, q, k, v, schedule: str = "balanced", overlap: bool = True,
                trace: bool = False):
        P, w = self.world, self.worker
        builders = {"balanced": build_balanced_schedule, "ring": build_ring_schedule,
                    "balanced_split": build_balanced_split_schedule}
        if schedule not in builders:
            raise ConfigError(f"unknown forward schedule {schedule!r}")
        sched = builders[schedule](P)
        viol = validate(sched)
        if viol:
            raise ScheduleError(f"invalid schedule: {viol[0]} ({len(viol)} violations)")
        plans = forward_plan(sched, w)
        h, rows, d = q.shape
        hk = k.shape[0]
        be, tr = self.backend, self.transport
        rec = self.rec = Recorder(tr.cuda, tr.group, trace)
        acc, _ = be.new_acc(h, rows, d, self._buf("acc", (h * rows * (d + 2),), be.acc_dtype))
        have_acc = False
        # receive slots: double-buffered (prefetch depth 1)
        kv_slot = [(self._buf(f"k{i}", (hk, rows, d), k.dtype), self._buf(f"v{i}", (hk, rows, d), v.dtype))
                   for i in range(2)]
        q_slot = [self._buf(f"q{i}", (h, rows, d), q.dtype) for i in range(2)]
        part_pk = self._buf("part_send", (h * rows * (d + 2),), be.acc_dtype)
        part, _ = be.new_acc(h, rows, d, part_pk)
        recv_part = {}
        # split step (balanced_split): kv rows [0, lo) stay with the helper,
        # [lo, rows) travel to the owner as one packed KVHalf message
        lo = rows // 2
        if any(p.part != 0 for p in plans) or any(p.kvh_sends for p in plans):
            k_lo = self._buf("k_lo", (hk, lo, d), k.dtype)
            v_lo = self._buf("v_lo", (hk, lo, d), v.dtype)
            k_hi = self._buf("k_hi", (hk, rows - lo, d), k.dtype)
            v_hi = self._buf("v_hi", (hk, rows - lo, d), v.dtype)
            k_lo.copy_(k[:, :lo])
            v_lo.copy_(v[:, :lo])
            k_hi.copy_(k[:, lo:])
            v_hi.copy_(v[:, lo:])
            kvh_slot = (self._buf("kh_recv", (hk, rows - lo, d), k.dtype),
                        self._buf("vh_recv", (hk, rows - lo, d), v.dtype))

        pub = {"k": k, "v": v, "q": q, "part": part_pk}
        if any(p.part != 0 for p in plans) or any(p.kvh_sends for p in plans):
            pub.update(k_hi=k_hi, v_hi=v_hi)
        tr.publish(pub)  # collective (pull transport); no-op for send/recv transports

        def post_operands(t):
            """sends of my immutable KV/Q for step t + the receive my step-t action needs."""
            p = plans[t]
            sends, recvs = [], []
            mk = rec.mark()
            for dst in p.kv_sends:
                sends += [(k, dst - 1), (v, dst - 1)]
                self._sent(k, v)
                rec.send(t, 0, w, dst, mk)
            for dst in p.kvh_sends:
                sends += [(k_hi, dst - 1), (v_hi, dst - 1)]
                self._sent(k_hi, v_hi)
                rec.send(t, 4, w, dst, mk)
            for dst in p.q_sends:
                sends.append((q, dst - 1))
                self._sent(q)
                rec.send(t, 1, w, dst, mk)
            if p.action == "direct" and p.part == KVPart.High:
                recvs += [(kvh_slot[0], p.peer - 1, "k_hi"), (kvh_slot[1], p.peer - 1, "v_hi")]
            elif p.action == "direct":
                ks, vs = kv_slot[t % 2]
                recvs += [(ks, p.peer - 1, "k"), (vs, p.peer - 1, "v")]
            elif p.action == "help":
                recvs.append((q_slot[t % 2], p.peer - 1, "q"))
            return tr.exchange(sends, recvs)

        held = 0
        part_handle = None
        pending = post_operands(0) if P > 1 else _Done()
        for t, p in enumerate(plans):
            handle = pending
            nxt = None
            if overlap and t + 1 < len(plans):
                nxt = post_operands(t + 1)  # prefetch: overlaps this step's compute
            handle.wait()
            cur_held = (1 if p.action in ("direct", "help") else 0) + (1 if nxt is not None and plans[t + 1].action in ("direct", "help") else 0)
            held = max(held, cur_held)
            m0 = rec.mark()
            if p.action == "direct" and p.part == KVPart.High:
                rec.arrive(t, 4, p.peer, w, m0, kvh_slot)
            elif p.action == "direct":
                rec.arrive(t, 0, p.peer, w, m0, kv_slot[t % 2])
            elif p.action == "help":
                rec.arrive(t, 1, p.peer, w, m0, [q_slot[t % 2]])
            if p.action == "local":
                be.update(q, k, v, acc if have_acc else None, "diagonal", acc)
                have_acc = True
                rec.task("local_attn", m0, rec.mark())
            elif p.action == "direct":
                ks, vs = kvh_slot if p.part == KVPart.High else kv_slot[t % 2]
                be.update(q, ks, vs, acc if have_acc else None, "full", acc)
                have_acc = True
                rec.task(f"remote_attn q={w} kv={p.peer}" +
                         (" rows=high" if p.part == KVPart.High else ""), m0, rec.mark())
            elif p.action == "help":
                if part_handle is not None:
                    part_handle.wait()  # the previous partial has left this buffer
                kk, vv = (k_lo, v_lo) if p.part == KVPart.Low else (k, v)
                be.update(q_slot[t % 2], kk, vv, None, "full", part)
                m1 = rec.mark()
                rec.task(f"helper_attn q={p.peer} kv={w}", m0, m1)
                part_handle = tr.exchange([(part_pk, p.peer - 1)], [])
                rec.send(t, 2, w, p.peer, m1)
                self._sent(part_pk)
            # merges of partials computed by helpers this step
            for hw in p.merges:
                buf = recv_part.get(hw)
                if buf is None:
                    buf = self._buf(f"part_recv{hw}", (h * rows * (d + 2),), be.acc_dtype)
                    recv_part[hw] = buf
                tr.exchange([], [(buf, hw - 1, "part")]).wait()
                m0 = rec.mark()
                rec.arrive(t, 2, hw, w, m0, [buf])
                pa, _ = be.new_acc(h, rows, d, buf)
                be.merge(acc, pa)
                rec.task(f"rescale_merge helper={hw}", m0, rec.mark(), attention=False)
            if not overlap and t + 1 < len(plans):
                nxt = post_operands(t + 1)
            pending = nxt if nxt is not None else _Done()
        if part_handle is not None:
            part_handle.wait()
        self.trace["max_remote_chunks_held"] = held
        out, lse = be.finalize(acc)
        self.saved = (q, k, v, out, lse)
        return out, lse

    def backward(self, d_out, schedule: str = "ring", overlap: bool = True, trace: bool = False):
        """Backward reusing the saved O and LSE (no forward recompute).

        schedule="ring": the reference order (runtime.cpp:605-651);
        schedule="balanced": the load-balanced extension (helpers compute the
        wrap-around owners' pairs on their own kv and return dq)."""
        if self.saved is None:
            raise StateError("run_backward requires forward output and logsumexp")
        q, k, v, out, lse = self.saved
        P, w = self.world, self.worker
        h, rows, d = q.shape
        hk = k.shape[0]
        be, tr = self.backend, self.transport
        builders = {"balanced": build_balanced_backward_schedule, "ring": build_ring_backward_schedule}
        if schedule not in builders:
            raise ConfigError(f"unknown backward schedule {schedule!r}")
        sched = builders[schedule](P)
        viol = validate_backward(sched)
        if viol:
            raise ScheduleError(f"invalid schedule: {viol[0]} ({len(viol)} violations)")
        plans = backward_plan(sched, w)
        rec = self.rec_bwd = Recorder(tr.cuda, tr.group, trace)
        gd = be.grad_dtype
        dq = self._buf("dq", (h, rows, d), gd)
        dk = self._buf("dk", (hk, rows, d), gd)
        dv = self._buf("dv", (hk, rows, d), gd)
        for t_ in (dq, dk, dv):
            t_.zero_()
        d_vec = be.bwd_aux(d_out, out)
        kv_slot = [(self._buf(f"bk{i}", (hk, rows, d), k.dtype), self._buf(f"bv{i}", (hk, rows, d), v.dtype))
                   for i in range(2)]
        bundle = [(self._buf(f"bq{i}", (h, rows, d), q.dtype), self._buf(f"bdo{i}", (h, rows, d), d_out.dtype),
                   self._buf(f"blse{i}", (h, rows), lse.dtype), self._buf(f"bD{i}", (h, rows), d_vec.dtype))
                  for i in range(2)]
        g_send = [(self._buf(f"gk{i}", (hk, rows, d), gd), self._buf(f"gv{i}", (hk, rows, d), gd))
                  for i in range(2)]
        q_send = [self._buf(f"gq{i}", (h, rows, d), gd) for i in range(2)]
        g_recv = (self._buf("grk", (hk, rows, d), gd), self._buf("grv", (hk, rows, d), gd))
        tr.publish({"k": k, "v": v, "q": q, "d_out": d_out, "lse": lse, "d_vec": d_vec,
                    "gk0": g_send[0][0], "gv0": g_send[0][1], "gk1": g_send[1][0],
                    "gv1": g_send[1][1], "gq0": q_send[0], "gq1": q_send[1]})

        def post_operands(t):
            p = plans[t]
            sends, recvs = [], []
            mk = rec.mark()
            for dst in p.kv_sends:
                sends += [(k, dst - 1), (v, dst - 1)]
                self._sent(k, v)
                rec.send(t, 0, w, dst, mk)
            for dst in p.q_sends:
                sends += [(q, dst - 1), (d_out, dst - 1), (lse, dst - 1), (d_vec, dst - 1)]
                self._sent(q, d_out, lse, d_vec)
                rec.send(t, 1, w, dst, mk)
            if p.action == "direct":
                ks, vs = kv_slot[t % 2]
                recvs += [(ks, p.peer - 1, "k"), (vs, p.peer - 1, "v")]
            elif p.action == "help":
                recvs += [(x, p.peer - 1, key) for x, key in
                          zip(bundle[t % 2], ("q", "d_out", "lse", "d_vec"))]
            return tr.exchange(sends, recvs)

        held = 0
        pending = post_operands(0) if P > 1 else _Done()
        for t, p in enumerate(plans):
            handle = pending
            nxt = post_operands(t + 1) if (overlap and t + 1 < len(plans)) else None
            handle.wait()
            held = max(held, (1 if p.action in ("direct", "help") else 0) +
                       (1 if nxt is not None and plans[t + 1].action in ("direct", "help") else 0))
            sends = []
            m0 = rec.mark()
            if p.action == "local":
                be.grads(q, k, v, lse, d_out, d_vec, "diagonal", dq, dk, dv, accumulate_kv=True)
                rec.task("bwd_local", m0, rec.mark())
            elif p.action == "direct":
                rec.arrive(t, 0, p.peer, w, m0, kv_slot[t % 2])
                ks, vs = kv_slot[t % 2]
                gk, gv = g_send[t % 2]
                be.grads(q, ks, vs, lse, d_out, d_vec, "full", dq, gk, gv, accumulate_kv=False)
                m1 = rec.mark()
                rec.task(f"bwd_remote kv={p.peer}", m0, m1)
                sends += [(gk, p.peer - 1), (gv, p.peer - 1)]
                self._sent(gk, gv)
                rec.send(t, 3, w, p.peer, m1)
            elif p.action == "help":
                rec.arrive(t, 1, p.peer, w, m0, bundle[t % 2])
                bq, bdo, blse, bD = bundle[t % 2]
                gq = q_send[t % 2]
                gq.zero_()
                be.grads(bq, k, v, blse, bdo, bD, "full", gq, dk, dv, accumulate_kv=True)
                m1 = rec.mark()
                rec.task(f"bwd_helper q={p.peer}", m0, m1)
                sends.append((gq, p.peer - 1))
                self._sent(gq)
                rec.send(t, 2, w, p.peer, m1)
            recvs = [(g_recv[0], s - 1, f"gk{t % 2}") for s in p.gradkv_from[:1]] + \
                    [(g_recv[1], s - 1, f"gv{t % 2}") for s in p.gradkv_from[:1]]
            part_bufs = []
            for hw in p.merges:
                buf = self._buf(f"gqr{hw}", (h, rows, d), gd)
                part_bufs.append(buf)
                recvs.append((buf, hw - 1, f"gq{t % 2}"))
            if len(p.gradkv_from) > 1:
                raise ScheduleError("at most one GradKV per worker and step is supported")
            # results leave right after their kernels; waiting also retires the
            # send buffers before they are rewritten two steps later
            tr.exchange(sends, recvs).wait()
            m2 = rec.mark()
            if p.gradkv_from:
                rec.arrive(t, 3, p.gradkv_from[0], w, m2, g_recv)
                be.add_(dk, g_recv[0])
                be.add_(dv, g_recv[1])
            for hw, buf in zip(p.merges, part_bufs):
                rec.arrive(t, 2, hw, w, m2, [buf])
                be.add_(dq, buf)
            if not overlap and t + 1 < len(plans):
                nxt = post_operands(t + 1)
            pending = nxt if nxt is not None else _Done()
        self.trace["max_remote_chunks_held_bwd"] = held
        return dq, dk, dv

    def forward_trace(self, group=None):
        """Collective: rank 0 gets the forward pass trace (reference schema)."""
        return gather_trace(self.rec, self.rank, self.world, self.trace["max_remote_chunks_held"],
                            group)

    def backward_trace(self, group=None):
        return gather_trace(self.rec_bwd, self.rank, self.world,
                            self.trace.get("max_remote_chunks_held_bwd", 0), group)
