"""Schedules, mirroring /root/reference/proj/include/distattn/schedule.hpp.

The tables are built by the native library (csrc/schedule.cpp) and decoded
here into the reference's Task / ScheduleMessage / Schedule shapes. Exact
rational idle fractions and speedups use fractions.Fraction (rational.hpp).
"""
from __future__ import annotations

import ctypes as C
import enum
import json
from dataclasses import dataclass, field
from fractions import Fraction

from . import _lib
from .errors import ConfigError, check


class TaskKind(enum.IntEnum):
    LocalAttn = 0
    RemoteAttn = 1
    RescaleMerge = 2
    Idle = 3


class PayloadKind(enum.IntEnum):
    KV = 0
    Q = 1
    PartialResult = 2
    GradKV = 3
    KVHalf = 4  # split-schedule extension: half of a kv chunk's rows


class KVPart(enum.IntEnum):
    """Rows of the kv chunk a RemoteAttn task covers (split extension; carried
    in Task.helper, which the reference only uses for RescaleMerge)."""
    Whole = 0
    Low = 1    # rows [0, c/2)
    High = 2   # rows [c/2, c)


_TASK_NAMES = {0: "local_attn", 1: "remote_attn", 2: "rescale_merge", 3: "idle"}
_PAYLOAD_NAMES = {0: "kv", 1: "q", 2: "partial", 3: "grad_kv", 4: "kv_half"}


@dataclass(frozen=True)
class Task:
    kind: TaskKind = TaskKind.Idle
    worker: int = 0
    query_owner: int = 0
    kv_owner: int = 0
    helper: int = 0

    def is_attention(self) -> bool:
        return self.kind in (TaskKind.LocalAttn, TaskKind.RemoteAttn)

    @property
    def kv_part(self) -> KVPart:
        return KVPart(self.helper) if self.kind == TaskKind.RemoteAttn else KVPart.Whole

    def weight(self) -> Fraction:
        """Chunk pairs of work: 1, or 1/2 for a split-step half task."""
        if not self.is_attention():
            return Fraction(0)
        return Fraction(1) if self.kv_part == KVPart.Whole else Fraction(1, 2)


@dataclass(frozen=True)
class ScheduleMessage:
    step: int
    from_: int
    to: int
    kind: PayloadKind


@dataclass
class Schedule:
    workers: int = 0
    steps: list = field(default_factory=list)      # list[list[Task]]
    messages: list = field(default_factory=list)   # list[ScheduleMessage]

    def step_count(self) -> int:
        return len(self.steps)

    def primaries(self, t: int):
        return self.steps[t][: self.workers]

    def merges(self, t: int):
        return self.steps[t][self.workers:]

    def attention_task_count(self) -> int:
        return sum(1 for s in self.steps for t in s if t.is_attention())

    def idle_slot_count(self) -> int:
        return sum(1 for s in self.steps for t in s if t.kind == TaskKind.Idle)

    def merge_count(self) -> int:
        return sum(1 for s in self.steps for t in s if t.kind == TaskKind.RescaleMerge)

    # flat encoding used by the C ABI
    def flat(self):
        tasks, msgs = [], []
        for t, step in enumerate(self.steps):
            for k in step:
                tasks += [t, int(k.kind), k.worker, k.query_owner, k.kv_owner, k.helper]
        for m in self.messages:
            msgs += [m.step, m.from_, m.to, int(m.kind)]
        return tasks, msgs


def _build(workers: int, kind: int) -> Schedule:
    lib = _lib.lib()
    steps = C.c_int32(0)
    nt, nm = C.c_int64(0), C.c_int64(0)
    check(lib.da_schedule_build(workers, kind, C.byref(steps), None, C.byref(nt), None, C.byref(nm)))
    tasks = (C.c_int32 * (6 * nt.value))()
    msgs = (C.c_int32 * (4 * max(nm.value, 1)))()
    check(lib.da_schedule_build(workers, kind, C.byref(steps), tasks, C.byref(nt), msgs, C.byref(nm)))
    s = Schedule(workers=workers, steps=[[] for _ in range(steps.value)])
    for i in range(nt.value):
        st, k, w, qo, kvo, h = tasks[6 * i: 6 * i + 6]
        s.steps[st].append(Task(TaskKind(k), w, qo, kvo, h))
    for i in range(nm.value):
        st, f, to, k = msgs[4 * i: 4 * i + 4]
        s.messages.append(ScheduleMessage(st, f, to, PayloadKind(k)))
    return s


def build_ring_schedule(workers: int) -> Schedule:
    """schedule.cpp:60-77"""
    return _build(workers, 0)


def build_balanced_schedule(workers: int) -> Schedule:
    """schedule.cpp:79-108"""
    return _build(workers, 1)


def build_balanced_split_schedule(workers: int) -> Schedule:
    """Balanced forward with the even-P last step split (extension, SURVEY
    §8(f)2; DA_SCHEDULE_BALANCED_SPLIT). At t = P/2 helper p computes pair
    (p + P/2, p) on the low half of its kv rows (Q in, Partial out) and the
    owner on the high half (KVHalf in). Odd P: the balanced schedule."""
    return _build(workers, 4)


def build_ring_backward_schedule(workers: int) -> Schedule:
    """The reference run_backward order (runtime.cpp:605-651) as an explicit
    schedule: the ring task table plus a GradKV message per direct pair."""
    return _build(workers, 2)


def build_balanced_backward_schedule(workers: int) -> Schedule:
    """Load-balanced backward (extension): the balanced task
    table; direct pairs exchange KV/GradKV, helpers receive the owner's
    (q, dO, lse, D) bundle as the Q message and return dq as the Partial."""
    return _build(workers, 3)


def build_balanced_split_backward_schedule(workers: int) -> Schedule:
    """Backward of the split schedule (extension; DA_SCHEDULE_BALANCED_SPLIT_BWD):
    the balanced_split task table with the backward messages. At t = P/2 the
    owner computes its pair on the high half of the kv rows (KVHalf in, that
    half's GradKV back) and the helper on the low half (Q bundle in, dq
    Partial back). Odd P: the balanced backward."""
    return _build(workers, 5)


def validate_backward(s: Schedule) -> list:
    """validate() plus GradKV coverage of every direct pair."""
    return validate(s, backward=True)


def validate(s: Schedule, backward: bool = False) -> list:
    """schedule.cpp:121-258: the list of violation messages (empty = valid)."""
    tasks, msgs = s.flat()
    ta = (C.c_int32 * max(len(tasks), 1))(*tasks)
    ma = (C.c_int32 * max(len(msgs), 1))(*msgs)
    lib = _lib.lib()
    fn = lib.da_schedule_validate_backward if backward else lib.da_schedule_validate
    n = fn(s.workers, len(s.steps), ta, len(tasks) // 6, ma, len(msgs) // 4)
    if n < 0:
        raise ConfigError(lib.da_last_error().decode())
    if n == 0:
        return []
    msgs = lib.da_last_error().decode().split("\n")
    assert len(msgs) == n, (n, msgs)
    return msgs


def idle_fraction(s: Schedule) -> Fraction:
    slots = s.workers * s.step_count()
    return Fraction(0) if slots == 0 else Fraction(s.idle_slot_count(), slots)


def expected_speedup(s: Schedule) -> Fraction:
    return Fraction(0) if s.step_count() == 0 else Fraction(s.attention_task_count(), s.step_count())


def weighted_makespan(s: Schedule, diag_weight: Fraction = Fraction(1)) -> Fraction:
    """Sum over steps of the heaviest primary task (chunk-pair units; half
    tasks weigh 1/2, the causal diagonal `diag_weight`)."""
    total = Fraction(0)
    for step in s.steps:
        w = [diag_weight if t.kind == TaskKind.LocalAttn else t.weight() for t in step]
        total += max(w, default=Fraction(0))
    return total


def weighted_speedup(s: Schedule, diag_weight: Fraction = Fraction(1)) -> Fraction:
    """Ideal speedup over one worker doing all pairs, counting work instead of
    tasks: with diag_weight = 1/2 (causal diagonal costs half a pair) this is
    the FLOP-level ceiling (P=8: ring 64/15, balanced 64/9, balanced_split 8;
    split over ring 1.875x vs balanced over ring 5/3)."""
    work = sum((diag_weight if t.kind == TaskKind.LocalAttn else t.weight())
               for st in s.steps for t in st)
    ms = weighted_makespan(s, diag_weight)
    return Fraction(0) if ms == 0 else work / ms


def ring_idle_fraction_formula(workers: int) -> Fraction:
    if workers < 1:
        raise ConfigError("need at least 1 worker")
    return Fraction(workers * workers - workers, 2 * workers * workers)


def balanced_idle_fraction_reference(workers: int) -> Fraction:
    if workers < 1:
        raise ConfigError("need at least 1 worker")
    return Fraction(0) if workers % 2 == 1 else Fraction(1, 2 * workers)


def schedule_to_json(s: Schedule) -> str:
    """schedule.cpp:301-327 (same keys)."""
    def task_json(t: Task):
        j = {"kind": _TASK_NAMES[int(t.kind)]}
        if t.kind == TaskKind.RemoteAttn:
            j["query_owner"] = t.query_owner
            j["kv_owner"] = t.kv_owner
            if t.kv_part != KVPart.Whole:
                j["kv_part"] = t.kv_part.name.lower()
        elif t.kind == TaskKind.RescaleMerge:
            j["helper"] = t.helper
        return j
    j = {"P": s.workers,
         "steps": [[{"task": task_json(t), "worker": t.worker} for t in step] for step in s.steps],
         "messages": [{"from": m.from_, "kind": _PAYLOAD_NAMES[int(m.kind)], "step": m.step,
                       "to": m.to} for m in s.messages]}
    return json.dumps(j, indent=2, sort_keys=True)


def schedule_to_csv(s: Schedule) -> str:
    """schedule.cpp:329-342 (same columns)."""
    lines = ["step,worker,task,query_owner,kv_owner,helper"]
    for t, step in enumerate(s.steps):
        for k in step:
            row = f"{t},{k.worker},{_TASK_NAMES[int(k.kind)]},"
            if k.kind == TaskKind.RemoteAttn:
                row += f"{k.query_owner},{k.kv_owner},"
            elif k.kind == TaskKind.LocalAttn:
                row += f"{k.worker},{k.worker},"
            else:
                row += ",,"
            if k.kind == TaskKind.RescaleMerge:
                row += f"{k.helper}"
            lines.append(row)
    return "\n".join(lines) + "\n"
