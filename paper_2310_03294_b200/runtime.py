"""Sequence-parallel executors, mirroring /root/reference/proj/include/distattn/runtime.hpp.

Two executors share the reference's per-worker operation order:

* ``run_forward`` / ``run_backward`` — P logical workers on ONE device
  (the reference's stepper, runtime.cpp:266-330 / 605-651), implemented
  natively (csrc/runtime.cu) with every chunk a sm_100a kernel.
* ``rank.RankRuntime`` — one process per GPU, the production multi-GPU path:
  the native per-rank runtime (csrc/rank_runtime.cu) with NCCL send/recv
  (or CUDA-IPC pulls when ranks share a GPU) on a side stream.

``dist.DistRuntime`` is the same protocol written in Python over a pluggable
compute backend: it is the host-logic model the CPU suite runs under gloo
against the oracle (tests/test_dist_gloo.py) and the wall-clock trace
exporter; it is not what bench.py or a production caller runs.

Shards are device tensors [heads, rows, 128] (bf16 q/k/v/out/d_out, fp32
lse/dq/dk/dv).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import torch

from . import _lib
from .errors import ConfigError, StateError, check
from .schedule import Schedule

GOLDEN = 0x9E3779B97F4A7C15
MASK64 = (1 << 64) - 1


class Rng:
    """splitmix64, numerics.hpp:140-174. Host-side draws are exact Python
    integers; ``fill`` continues the same stream on the device."""

    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next_u64(self) -> int:
        self.state = (self.state + GOLDEN) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def next_unit(self) -> float:
        return (self.next_u64() >> 11) * 2.0 ** -53

    def uniform(self, lo: float, hi: float) -> float:
        return lo + (hi - lo) * self.next_unit()

    def fork(self) -> "Rng":
        return Rng(self.next_u64())

    def fill(self, out: torch.Tensor, lo: float = -1.0, hi: float = 1.0, stream=None) -> torch.Tensor:
        """Row-major device fill, one draw per entry (Rng::matrix, numerics.hpp:162-167)."""
        dtype = {torch.float32: 0, torch.bfloat16: 1, torch.float64: 2}[out.dtype]
        n = out.numel()
        s = stream if stream is not None else torch.cuda.current_stream()
        check(_lib.lib().da_rng_uniform(self.state, n, lo, hi, dtype, C.c_void_p(out.data_ptr()),
                                        C.c_void_p(s.cuda_stream)))
        self.state = (self.state + n * GOLDEN) & MASK64
        return out


@dataclass
class SequenceShard:
    """runtime.hpp:32-41 (device tensors, [heads, rows, d])."""
    worker: int
    q: torch.Tensor
    k: torch.Tensor
    v: torch.Tensor
    out: torch.Tensor | None = None
    lse: torch.Tensor | None = None
    d_out: torch.Tensor | None = None
    dq: torch.Tensor | None = None
    dk: torch.Tensor | None = None
    dv: torch.Tensor | None = None

    def has_forward_state(self) -> bool:
        return self.out is not None and self.lse is not None


def make_shards(workers: int, total_tokens: int, d: int, rng: Rng, *, device="cuda",
                dtype=torch.bfloat16) -> list[SequenceShard]:
    """runtime.cpp:24-46 for one head: draw the full q, then k, then v
    (U[-1,1), row-major) and give worker p rows [(p-1)N/P, pN/P)."""
    if workers < 1:
        raise ConfigError("need at least 1 worker")
    if total_tokens < 1 or d < 1:
        raise ConfigError("tokens and d must be positive")
    if total_tokens % workers != 0:
        raise ConfigError(f"token count {total_tokens} not divisible by {workers} workers")
    full = [rng.fill(torch.empty(total_tokens, d, dtype=dtype, device=device)) for _ in range(3)]
    rows = total_tokens // workers
    return [SequenceShard(p + 1, *(t[p * rows:(p + 1) * rows].unsqueeze(0).contiguous() for t in full))
            for p in range(workers)]


def make_parity_shards(seed: int, workers: int, total_tokens: int, heads: int, d: int = 128, *,
                       heads_kv: int | None = None, device="cuda") -> list[SequenceShard]:
    """Multi-head parity inputs: per head h, head_rng =
    Rng(seed).fork() (h+1-th fork), make_shards(head_rng), then d_out drawn
    from head_rng. GQA keeps the k/v of the first heads_kv heads."""
    heads_kv = heads_kv or heads
    root = Rng(seed)
    per_head = []
    for _ in range(heads):
        hr = root.fork()
        sh = make_shards(workers, total_tokens, d, hr, device=device)
        dout = hr.fill(torch.empty(total_tokens, d, dtype=torch.bfloat16, device=device))
        per_head.append((sh, dout))
    rows = total_tokens // workers
    shards = []
    for p in range(workers):
        cat = lambda xs: torch.cat(xs, 0).contiguous()  # noqa: E731
        shards.append(SequenceShard(
            p + 1,
            q=cat([ph[0][p].q for ph in per_head]),
            k=cat([ph[0][p].k for ph in per_head[:heads_kv]]),
            v=cat([ph[0][p].v for ph in per_head[:heads_kv]]),
            d_out=cat([ph[1][p * rows:(p + 1) * rows].unsqueeze(0) for ph in per_head])))
    return shards


@dataclass
class CommCounters:
    """runtime.hpp:49-63 (scalars per payload kind, summed over heads)."""
    kv_scalars: int = 0
    q_scalars: int = 0
    partial_scalars: int = 0
    grad_scalars: int = 0
    kv_messages: int = 0
    q_messages: int = 0
    partial_messages: int = 0
    grad_messages: int = 0

    def total_scalars(self) -> int:
        return self.kv_scalars + self.q_scalars + self.partial_scalars + self.grad_scalars


@dataclass
class ExecutionTrace:
    """runtime.hpp:80-89 (counters + kernel calls + residency)."""
    workers: int = 0
    counters: CommCounters = field(default_factory=CommCounters)
    attention_kernel_calls: int = 0
    max_remote_chunks_held: int = 0


def _ptr_array(ts):
    arr = (C.c_void_p * len(ts))(*[C.c_void_p(t.data_ptr()) if t is not None else None for t in ts])
    return arr


def _shards_struct(shards: list[SequenceShard], backward: bool):
    s0 = shards[0]
    h_q, rows, d = s0.q.shape
    h_kv = s0.k.shape[0]
    for i, s in enumerate(shards):
        if s.worker != i + 1:
            raise ConfigError("shards must be ordered by worker id")
        if s.q.shape != s0.q.shape or s.k.shape != s0.k.shape or s.v.shape != s0.v.shape:
            from .errors import ShapeError
            raise ShapeError("all shards must share the same q/k/v shape")
    keep = []
    st = _lib.Shards()
    st.workers, st.h_q, st.h_kv, st.rows, st.d = len(shards), h_q, h_kv, rows, d
    fields = ["q", "k", "v", "out", "lse", "d_out", "dq", "dk", "dv"]
    for f in fields:
        arr = _ptr_array([getattr(s, f) for s in shards])
        keep.append(arr)
        setattr(st, f, C.cast(arr, C.POINTER(C.c_void_p)))
    return st, keep


def _trace(P: int, c: _lib.Counters) -> ExecutionTrace:
    cc = CommCounters(c.kv_scalars, c.q_scalars, c.partial_scalars, c.grad_scalars,
                      c.kv_messages, c.q_messages, c.partial_messages, c.grad_messages)
    return ExecutionTrace(P, cc, c.attention_kernel_calls, c.max_remote_chunks_held)


def run_forward(shards: list[SequenceShard], schedule: Schedule | str = "balanced",
                stream=None) -> ExecutionTrace:
    """runtime.cpp:491-529: runs the schedule's forward over all P workers on
    this device; writes out (bf16) / lse (fp32) into the shards."""
    if isinstance(schedule, str) and schedule not in ("ring", "balanced", "balanced_split"):
        from .errors import ConfigError
        raise ConfigError(f"unknown forward schedule {schedule!r}")
    for s in shards:
        h, rows, d = s.q.shape
        if s.out is None:
            s.out = torch.empty(h, rows, d, dtype=torch.bfloat16, device=s.q.device)
        if s.lse is None:
            s.lse = torch.empty(h, rows, dtype=torch.float32, device=s.q.device)
    st, keep = _shards_struct(shards, False)
    c = _lib.Counters()
    strm = stream if stream is not None else torch.cuda.current_stream()
    sptr = C.c_void_p(strm.cuda_stream)
    if isinstance(schedule, str):
        kind_i = {"ring": 0, "balanced": 1, "balanced_split": 4}[schedule]
        check(_lib.lib().da_run_forward(C.byref(st), kind_i, C.byref(c), sptr))
    else:  # any schedule that passes the reference validator (runtime.hpp:106-118)
        steps, t, nt, m, nm = _table(schedule)
        check(_lib.lib().da_run_forward_table(C.byref(st), steps, t, nt, m, nm, C.byref(c), sptr))
    del keep
    return _trace(len(shards), c)


def run_backward(shards: list[SequenceShard], schedule="ring",
                 stream=None) -> ExecutionTrace:
    """runtime.cpp:720-750. schedule="ring" is the reference order
    (BackwardMode::Vanilla); "balanced" is the load-balanced backward
    extension (schedule.build_balanced_backward_schedule), "balanced_split"
    its even-P split (build_balanced_split_backward_schedule). Requires forward
    state and d_out; writes fp32 dq/dk/dv into the shards."""
    for s in shards:
        if not s.has_forward_state():
            raise StateError("run_backward requires forward output and logsumexp")
        if s.d_out is None:
            raise StateError("run_backward requires d_out on every shard")
        h, rows, d = s.q.shape
        hk = s.k.shape[0]
        if s.dq is None:
            s.dq = torch.empty(h, rows, d, dtype=torch.float32, device=s.q.device)
        if s.dk is None:
            s.dk = torch.empty(hk, rows, d, dtype=torch.float32, device=s.q.device)
        if s.dv is None:
            s.dv = torch.empty(hk, rows, d, dtype=torch.float32, device=s.q.device)
    st, keep = _shards_struct(shards, True)
    c = _lib.Counters()
    strm = stream if stream is not None else torch.cuda.current_stream()
    sptr = C.c_void_p(strm.cuda_stream)
    if isinstance(schedule, str):
        if schedule not in ("ring", "balanced", "balanced_split"):
            from .errors import ConfigError
            raise ConfigError(f"unknown backward schedule {schedule!r}")
        kind = {"ring": 2, "balanced": 3, "balanced_split": 5}[schedule]
        check(_lib.lib().da_run_backward_sched(C.byref(st), kind, C.byref(c), sptr))
    else:  # a backward schedule table (validate_backward invariants)
        steps, t, nt, m, nm = _table(schedule)
        check(_lib.lib().da_run_backward_table(C.byref(st), steps, t, nt, m, nm, C.byref(c), sptr))
    del keep
    return _trace(len(shards), c)


def _table(s: Schedule):
    """Flat int32 encoding of a Schedule for the *_table C entry points."""
    tasks, msgs = s.flat()
    t = (C.c_int32 * max(1, len(tasks)))(*tasks)
    m = (C.c_int32 * max(1, len(msgs)))(*msgs)
    return len(s.steps), t, len(tasks) // 6, m, len(msgs) // 4
