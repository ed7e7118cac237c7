"""Python handle on the native per-rank runtime (csrc/rank_runtime.cu).

The C++ runtime executes this rank's schedule (forward and backward) with
copy-engine pulls from the peers' HBM; Python only supplies the bootstrap
allgather (torch.distributed, any backend) and device tensors. Mirrors
runtime.hpp's worker for one process per GPU (runtime.cpp:390-487, 653-716).
"""
from __future__ import annotations

import ctypes as C

import torch
import torch.distributed as tdist

from . import _lib
from .errors import check
from .runtime import CommCounters

_AG = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p)
_FWD = {"ring": 0, "balanced": 1, "balanced_split": 4}
_BWD = {"ring": 2, "balanced": 3, "balanced_split": 5}


class RankRuntime:
    """One rank of the sequence-parallel runtime; all calls are collective.

    transport: "nccl" (grouped send/recv per phase on a side stream; ranks on
    distinct GPUs), "ipc" (copy-engine pulls from peer HBM; ranks may share a
    GPU) or "none" (no transfer: the no-communication timing arm).
    deterministic: ordered dq reductions, bitwise-reproducible backward."""

    def __init__(self, rank: int, world: int, group=None, transport: str = "ipc",
                 deterministic: bool = False, nccl_max_ctas: int = 0):
        from .errors import ConfigError
        if transport not in _lib.TRANSPORT:
            raise ConfigError(f"unknown transport {transport!r}")
        self.rank, self.world, self.group = rank, world, group
        self.transport, self.deterministic = transport, deterministic
        self._cb = _AG(self._allgather)  # keep the trampoline alive
        opts = _lib.RankOptions(_lib.TRANSPORT[transport], 1 if deterministic else 0,
                                int(nccl_max_ctas))
        h = C.c_void_p()
        check(_lib.lib().da_rank_create_ex(rank, world, C.cast(self._cb, C.c_void_p), None,
                                           C.byref(opts), C.byref(h)))
        self._h = h
        self._saved = None

    def _allgather(self, ctx, send, nbytes, recv):
        try:
            mine = C.string_at(send, nbytes)
            outs = [None] * self.world
            tdist.all_gather_object(outs, mine, group=self.group)
            C.memmove(recv, b"".join(outs), nbytes * self.world)
            return 0
        except Exception:  # pragma: no cover - surfaced as a ConfigError by the C side
            return 1

    def forward(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                schedule: str = "balanced", stream=None, trace: bool = False):
        from .errors import ConfigError, ShapeError
        from .flashcore import _check_qkv
        _check_qkv(q, k, v, "run_forward")
        if q.shape[2] != 128:
            from .errors import UnsupportedError
            raise UnsupportedError("run_forward: d must be 128")
        if k.shape[1] != q.shape[1]:
            raise ShapeError("all shards must share the same q/k/v shape")
        if q.shape[0] % k.shape[0] != 0:
            raise ShapeError("h_q must be a positive multiple of h_kv")
        if isinstance(schedule, str) and schedule not in _FWD:
            raise ConfigError(f"unknown forward schedule {schedule!r}")
        h, rows, _ = q.shape
        hk = k.shape[0]
        self._set_trace(trace)
        out = torch.empty_like(q)
        lse = torch.empty(h, rows, dtype=torch.float32, device=q.device)
        c = _lib.Counters()
        st = stream if stream is not None else torch.cuda.current_stream()
        if isinstance(schedule, str):
            check(_lib.lib().da_rank_forward(self._h, _FWD[schedule], q.data_ptr(), k.data_ptr(),
                                             v.data_ptr(), h, hk, rows, out.data_ptr(),
                                             lse.data_ptr(), C.byref(c), st.cuda_stream))
        else:  # a validated Schedule object (runtime.hpp:106-109), the same on every rank
            from .runtime import _table
            steps, t, nt, m, nm = _table(schedule)
            check(_lib.lib().da_rank_forward_table(self._h, steps, t, nt, m, nm, q.data_ptr(),
                                                   k.data_ptr(), v.data_ptr(), h, hk, rows,
                                                   out.data_ptr(), lse.data_ptr(), C.byref(c),
                                                   st.cuda_stream))
        self._saved = (q, k, v, out, lse)  # the runtime holds pointers to these
        return out, lse, _counters(c)

    def backward(self, d_out: torch.Tensor, schedule: str = "ring", stream=None, saved=None,
                 trace: bool = False):
        """run_backward of this rank. `saved` = (q, k, v, out, lse) of an earlier
        forward re-installs that pass's state (a checkpointed multi-layer
        model: each layer's backward uses its own saved O / LSE); default: the
        last forward."""
        from .errors import ConfigError, ShapeError, StateError
        from .flashcore import _req
        if saved is not None:
            q, k, v, out, lse = saved
            if out is None or lse is None:
                raise StateError("run_backward requires forward output and logsumexp")
            for t, n in ((q, "q"), (k, "k"), (v, "v"), (out, "out")):
                _req(t, torch.bfloat16, n)
            _req(lse, torch.float32, "lse")
            if out.shape != q.shape or tuple(lse.shape) != tuple(q.shape[:2]) or \
                    k.shape != v.shape or k.shape[1] != q.shape[1]:
                raise ShapeError("run_backward: saved state shapes disagree")
            check(_lib.lib().da_rank_restore(self._h, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                             out.data_ptr(), lse.data_ptr(), q.shape[0],
                                             k.shape[0], q.shape[1]))
            self._saved = (q, k, v, out, lse)
        q, k, v, out, lse = self._saved if self._saved else (None,) * 5
        if q is None:
            raise StateError("run_backward requires forward output and logsumexp")
        _req(d_out, torch.bfloat16, "d_out")
        if d_out.shape != q.shape:
            raise ShapeError("block_attn_backward: upstream grad shape mismatch")
        if isinstance(schedule, str) and schedule not in _BWD:
            raise ConfigError(f"unknown backward schedule {schedule!r}")
        self._set_trace(trace)
        dq = torch.empty(q.shape, dtype=torch.float32, device=q.device)
        dk = torch.empty(k.shape, dtype=torch.float32, device=q.device)
        dv = torch.empty(k.shape, dtype=torch.float32, device=q.device)
        c = _lib.Counters()
        st = stream if stream is not None else torch.cuda.current_stream()
        if isinstance(schedule, str):
            check(_lib.lib().da_rank_backward(self._h, _BWD[schedule], d_out.data_ptr(),
                                              dq.data_ptr(), dk.data_ptr(), dv.data_ptr(),
                                              C.byref(c), st.cuda_stream))
        else:
            from .runtime import _table
            steps, t, nt, m, nm = _table(schedule)
            check(_lib.lib().da_rank_backward_table(self._h, steps, t, nt, m, nm,
                                                    d_out.data_ptr(), dq.data_ptr(),
                                                    dk.data_ptr(), dv.data_ptr(), C.byref(c),
                                                    st.cuda_stream))
        self._keep_dout = d_out
        return dq, dk, dv, _counters(c)

    def _set_trace(self, on: bool):
        if on:  # a common origin: every rank records its pass origin after the barrier
            torch.cuda.synchronize()
            if self.world > 1:
                tdist.barrier(group=self.group)
        _lib.lib().da_rank_set_trace(self._h, 1 if on else 0)

    def trace_records(self, pass_: str = "forward") -> list[dict]:
        """This rank's resolved trace records of the last traced pass."""
        pi = {"forward": 0, "backward": 1}[pass_]
        n = C.c_int64(0)
        check(_lib.lib().da_rank_trace(self._h, pi, None, 0, C.byref(n)))
        buf = (_lib.TraceRec * max(1, n.value))()
        check(_lib.lib().da_rank_trace(self._h, pi, C.cast(buf, C.c_void_p), n.value, C.byref(n)))
        return [{f: getattr(buf[i], f) for f, _ in _lib.TraceRec._fields_ if f != "pad"}
                for i in range(n.value)]

    def gather_trace(self, pass_: str = "forward", counters=None, held: int = 0):
        """Collective: rank 0 gets the pass's trace in the reference schema
        (trace_to_json, runtime.cpp:752-782 / runtime.hpp:66-89) and the other
        ranks None. Times are ms from the pass origin (each rank's origin is
        recorded right after a barrier). `counters`: this rank's CommCounters
        of the pass (summed over ranks into the trace)."""
        mine = {"rank": self.rank, "records": self.trace_records(pass_),
                "counters": dict(counters.__dict__) if counters is not None else {},
                "held": held}
        allr = [None] * self.world
        if self.world > 1:
            tdist.all_gather_object(allr, mine, group=self.group)
        else:
            allr = [mine]
        if self.rank != 0:
            return None
        return assemble_trace(allr, pass_)

    def close(self):
        if self._h:
            _lib.lib().da_rank_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def _counters(c) -> CommCounters:
    """The reference's CommCounters (runtime.hpp:49-63) plus the trace's kernel
    call count and residency high-water mark (ExecutionTrace, runtime.hpp:83-91)."""
    cc = CommCounters(c.kv_scalars, c.q_scalars, c.partial_scalars, c.grad_scalars,
                      c.kv_messages, c.q_messages, c.partial_messages, c.grad_messages)
    cc.attention_kernel_calls = c.attention_kernel_calls
    cc.max_remote_chunks_held = c.max_remote_chunks_held
    return cc


# buffer keys of csrc/rank_runtime.cu -> the reference's PayloadKind names
_FWD_KIND = {0: "kv", 1: "kv", 2: "q", 3: "partial", 4: "kv_half", 5: "kv_half"}
_BWD_KIND = {0: "kv", 1: "kv", 2: "q", 4: "kv_half", 5: "kv_half", 6: "q", 7: "q", 8: "q",
             9: "grad_kv", 10: "grad_kv", 11: "grad_kv", 12: "grad_kv", 13: "partial",
             14: "partial", 15: "grad_kv", 16: "grad_kv"}
_TASK = {1: "local_attn", 2: "remote_attn", 3: "helper_attn", 4: "rescale_merge", 5: "fold"}


def _task_label(code: int, worker: int, peer: int) -> str:
    """runtime.cpp:179-191 action_label (+ merge / fold events)."""
    if code == 1:
        return "local_attn"
    if code == 2:
        return f"remote_attn q={worker} kv={peer}"
    if code == 3:
        return f"helper_attn q={peer} kv={worker}"
    if code == 4:
        return f"rescale_merge helper={peer}"
    return f"fold from={peer}"


def assemble_trace(allr: list[dict], pass_: str) -> dict:
    """Per-rank native records -> the reference's ExecutionTrace JSON shape:
    workers[].events {t0, t1, task}, messages {t_issue (sender), t_arrive
    (receiver), kind, from, to} (one per payload: a KV message is its k and v
    tensors, the backward's Q message the q/dO/lse/D bundle), summed counters,
    kernel calls, residency and makespan."""
    kinds = _FWD_KIND if pass_ == "forward" else _BWD_KIND
    workers, issue, arrive = [], {}, {}
    calls = 0
    for r in sorted(allr, key=lambda x: x["rank"]):
        w = r["rank"] + 1
        ev = []
        for rec in r["records"]:
            if rec["kind"] == 0:
                ev.append({"t0": rec["t0_ms"], "t1": rec["t1_ms"],
                           "task": _task_label(rec["code"], w, rec["peer"])})
                calls += rec["code"] in (1, 2, 3)
            elif rec["kind"] == 1:
                key = (rec["phase"], w, rec["peer"] + 1, kinds.get(rec["code"], "?"))
                issue[key] = min(issue.get(key, rec["t0_ms"]), rec["t0_ms"])
            else:
                key = (rec["phase"], rec["peer"] + 1, w, kinds.get(rec["code"], "?"))
                arrive[key] = max(arrive.get(key, rec["t1_ms"]), rec["t1_ms"])
        workers.append({"worker": w, "events": sorted(ev, key=lambda e: e["t0"])})
    msgs = [{"t_issue": issue.get(k, t), "t_arrive": t, "kind": k[3], "from": k[1], "to": k[2]}
            for k, t in arrive.items()]
    msgs.sort(key=lambda m: (m["t_issue"], m["from"], m["to"]))
    counters = {}
    for r in allr:
        for c, v in r["counters"].items():
            if c not in ("attention_kernel_calls", "max_remote_chunks_held"):
                counters[c] = counters.get(c, 0) + v
    makespan = max((e["t1"] for w in workers for e in w["events"]), default=0.0)
    return {"workers": workers, "messages": msgs, "counters": counters,
            "attention_kernel_calls": calls,
            "max_remote_chunks_held": max((r["held"] for r in allr), default=0),
            "makespan": makespan, "time_unit": "ms", "clock": "CUDA events per rank"}
