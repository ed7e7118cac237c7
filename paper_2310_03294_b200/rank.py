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
_BWD = {"ring": 2, "balanced": 3}


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
                schedule: str = "balanced", stream=None):
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
        if schedule not in _FWD:
            raise ConfigError(f"unknown forward schedule {schedule!r}")
        h, rows, _ = q.shape
        hk = k.shape[0]
        out = torch.empty_like(q)
        lse = torch.empty(h, rows, dtype=torch.float32, device=q.device)
        c = _lib.Counters()
        st = stream if stream is not None else torch.cuda.current_stream()
        check(_lib.lib().da_rank_forward(self._h, _FWD[schedule], q.data_ptr(), k.data_ptr(),
                                         v.data_ptr(), h, hk, rows, out.data_ptr(),
                                         lse.data_ptr(), C.byref(c), st.cuda_stream))
        self._saved = (q, k, v, out, lse)  # the runtime holds pointers to these
        return out, lse, _counters(c)

    def backward(self, d_out: torch.Tensor, schedule: str = "ring", stream=None, saved=None):
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
        if schedule not in _BWD:
            raise ConfigError(f"unknown backward schedule {schedule!r}")
        dq = torch.empty(q.shape, dtype=torch.float32, device=q.device)
        dk = torch.empty(k.shape, dtype=torch.float32, device=q.device)
        dv = torch.empty(k.shape, dtype=torch.float32, device=q.device)
        c = _lib.Counters()
        st = stream if stream is not None else torch.cuda.current_stream()
        check(_lib.lib().da_rank_backward(self._h, _BWD[schedule], d_out.data_ptr(), dq.data_ptr(),
                                          dk.data_ptr(), dv.data_ptr(), C.byref(c),
                                          st.cuda_stream))
        self._keep_dout = d_out
        return dq, dk, dv, _counters(c)

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
