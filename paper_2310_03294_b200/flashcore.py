"""Per-chunk attention API, mirroring /root/reference/proj/include/distattn/flashcore.hpp.

Device tensors in, device tensors out; every call goes through the C ABI of
libdistattn_b200.so (sm_100a kernels). Layout per chunk: q/k/v bf16
[heads, rows, 128]; accumulator o fp32 [heads, rows, 128], m/l fp32
[heads, rows]. There is no CPU path: the functions raise when the library or a
B200 is absent.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass

import torch

from . import _lib
from .errors import check


class MaskMode(enum.IntEnum):
    """flashcore.hpp:30"""
    Diagonal = 0
    Full = 1
    Empty = 2


@dataclass
class AttnAccumulator:
    """AttnAccumulatorT (flashcore.hpp:65-81): unnormalised o, running max m, sum l."""
    o: torch.Tensor
    m: torch.Tensor
    l: torch.Tensor

    @staticmethod
    def fresh(heads: int, rows: int, d: int = 128, device="cuda") -> "AttnAccumulator":
        return AttnAccumulator(torch.zeros(heads, rows, d, dtype=torch.float32, device=device),
                               torch.full((heads, rows), -math.inf, dtype=torch.float32, device=device),
                               torch.zeros(heads, rows, dtype=torch.float32, device=device))

    def rows(self) -> int:
        return self.o.shape[1]

    def dim(self) -> int:
        return self.o.shape[2]


@dataclass
class AttnOutput:
    """AttnOutputT (flashcore.hpp:83-87)."""
    o: torch.Tensor    # bf16 [heads, rows, d]
    lse: torch.Tensor  # fp32 [heads, rows]


@dataclass
class ChunkGrads:
    """ChunkGradsT (flashcore.hpp:242-246); fp32 accumulators."""
    dq: torch.Tensor
    dk: torch.Tensor
    dv: torch.Tensor


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _req(t: torch.Tensor, dtype, name: str):
    if t.dtype != dtype or not t.is_cuda or not t.is_contiguous():
        raise TypeError(f"{name}: expected a contiguous CUDA {dtype} tensor, got {t.dtype} "
                        f"on {t.device} (contiguous={t.is_contiguous()})")


def _shape_error(msg: str):
    from .errors import ShapeError
    raise ShapeError(msg)


def _check_qkv(q, k, v, op: str):
    """flashcore.hpp:143-147 / 284-287: the reference's operand checks, done
    before any pointer reaches the C ABI (which cannot see tensor shapes: a
    mismatch there would be an out-of-bounds device access, not an error)."""
    for t, n in ((q, "q"), (k, "k"), (v, "v")):
        _req(t, torch.bfloat16, n)
        if t.dim() != 3:
            _shape_error(f"{op}: {n} must be [heads, rows, d]")
    if not (q.shape[2] == k.shape[2] == v.shape[2]):
        _shape_error(f"{op}: hidden dims disagree")
    if k.shape[1] != v.shape[1] or k.shape[0] != v.shape[0]:
        _shape_error(f"{op}: k/v row mismatch")


def _check_acc(acc: "AttnAccumulator", h_q: int, rows_q: int, d: int, op: str):
    for t, shape in ((acc.o, (h_q, rows_q, d)), (acc.m, (h_q, rows_q)), (acc.l, (h_q, rows_q))):
        _req(t, torch.float32, "accumulator")
        if tuple(t.shape) != shape:
            _shape_error(f"{op}: accumulator shape mismatch")


def _fwd(q, k, v, acc_in, mask, scale, finalize, acc_out=None, stream=None, degenerate_flag=None):
    _check_qkv(q, k, v, "block_attn_update")
    h_q, rows_q, d = q.shape
    h_kv, rows_kv, _ = k.shape
    if acc_in is not None:
        _check_acc(acc_in, h_q, rows_q, d, "block_attn_update")
    if acc_out is not None:
        _check_acc(acc_out, h_q, rows_q, d, "block_attn_update")
    a = _lib.FwdArgs()
    a.q, a.k, a.v = _ptr(q), _ptr(k), _ptr(v)
    a.h_q, a.h_kv, a.rows_q, a.rows_kv, a.d = h_q, h_kv, rows_q, rows_kv, d
    if acc_in is not None:
        a.o_in, a.m_in, a.l_in = _ptr(acc_in.o), _ptr(acc_in.m), _ptr(acc_in.l)
    flag = None
    if finalize:
        out = AttnOutput(torch.empty(h_q, rows_q, d, dtype=torch.bfloat16, device=q.device),
                         torch.empty(h_q, rows_q, dtype=torch.float32, device=q.device))
        # a caller-owned flag defers the DegenerateRowError check (no stream sync)
        flag = torch.zeros(1, dtype=torch.int32, device=q.device) if degenerate_flag is None else None
        dflag = flag if degenerate_flag is None else degenerate_flag
        a.o_out, a.lse_out, a.degenerate_flag = _ptr(out.o), _ptr(out.lse), _ptr(dflag)
    else:
        out = acc_out if acc_out is not None else AttnAccumulator(
            torch.empty(h_q, rows_q, d, dtype=torch.float32, device=q.device),
            torch.empty(h_q, rows_q, dtype=torch.float32, device=q.device),
            torch.empty(h_q, rows_q, dtype=torch.float32, device=q.device))
        a.o_acc, a.m_acc, a.l_acc = _ptr(out.o), _ptr(out.m), _ptr(out.l)
    a.scale = float(scale) if scale is not None else 0.0
    a.mask = int(mask)
    a.finalize = 1 if finalize else 0
    lib = _lib.lib()
    st = _stream(stream)
    check(lib.da_attn_fwd_chunk(C.byref(a), st))
    if flag is not None:
        check(lib.da_check_degenerate(_ptr(flag), st))
    return out


def block_attn_update(q, k, v, acc: AttnAccumulator | None, mask: MaskMode,
                      scale: float | None = None, *, out: AttnAccumulator | None = None,
                      stream=None) -> AttnAccumulator:
    """flashcore.hpp:135-197: absorb one kv chunk into the accumulator.

    acc=None is AttnAccumulator::fresh; `out` may alias `acc` (in-place update).
    """
    return _fwd(q, k, v, acc, mask, scale, False, out, stream)


def block_attn_update_final(q, k, v, acc: AttnAccumulator | None, mask: MaskMode,
                            scale: float | None = None, stream=None, *,
                            degenerate_flag: torch.Tensor | None = None) -> AttnOutput:
    """block_attn_update followed by finalize in the same kernel (the paper's `last` flag).

    Without `degenerate_flag` a degenerate row raises DegenerateRowError here
    (one stream sync). With a caller-owned int32 device flag the check is
    deferred to ``check_degenerate(flag)``, so pipelined callers never sync.
    """
    return _fwd(q, k, v, acc, mask, scale, True, None, stream, degenerate_flag)


def check_degenerate(flag: torch.Tensor, stream=None) -> None:
    """Raises DegenerateRowError (finalize, flashcore.hpp:233-235) if `flag` was set."""
    check(_lib.lib().da_check_degenerate(_ptr(flag), _stream(stream)))


def rescale(a: AttnAccumulator, b: AttnAccumulator, *, out: AttnAccumulator | None = None,
            stream=None) -> AttnAccumulator:
    """flashcore.hpp:202-224: merge two partial accumulators over disjoint key sets."""
    if a.o.shape != b.o.shape:
        _shape_error("rescale: accumulator shapes disagree")
    h, rows, d = a.o.shape
    _check_acc(a, h, rows, d, "rescale")
    _check_acc(b, h, rows, d, "rescale")
    if out is not None:
        _check_acc(out, h, rows, d, "rescale")
    if out is None:
        out = AttnAccumulator(torch.empty_like(a.o), torch.empty_like(a.m), torch.empty_like(a.l))
    check(_lib.lib().da_attn_merge(_ptr(a.o), _ptr(a.m), _ptr(a.l), _ptr(b.o), _ptr(b.m), _ptr(b.l),
                                   _ptr(out.o), _ptr(out.m), _ptr(out.l), h, rows, d, _stream(stream)))
    return out


def finalize(acc: AttnAccumulator, stream=None) -> AttnOutput:
    """flashcore.hpp:227-240; raises DegenerateRowError when a row absorbed no key."""
    h, rows, d = acc.o.shape
    _check_acc(acc, h, rows, d, "finalize")
    out = AttnOutput(torch.empty(h, rows, d, dtype=torch.bfloat16, device=acc.o.device),
                     torch.empty(h, rows, dtype=torch.float32, device=acc.o.device))
    flag = torch.zeros(1, dtype=torch.int32, device=acc.o.device)
    lib = _lib.lib()
    st = _stream(stream)
    check(lib.da_attn_finalize(_ptr(acc.o), _ptr(acc.m), _ptr(acc.l), _ptr(out.o), _ptr(out.lse),
                               _ptr(flag), h, rows, d, st))
    check(lib.da_check_degenerate(_ptr(flag), st))
    return out


def backward_aux(d_out: torch.Tensor, out: torch.Tensor, stream=None) -> torch.Tensor:
    """flashcore.hpp:250-261: D = rowsum(dO * O), fp32 [heads, rows]."""
    _req(d_out, torch.bfloat16, "d_out"); _req(out, torch.bfloat16, "out")
    if d_out.shape != out.shape or out.dim() != 3:
        _shape_error("backward_aux: shape mismatch")
    h, rows, d = out.shape
    dvec = torch.empty(h, rows, dtype=torch.float32, device=out.device)
    check(_lib.lib().da_attn_bwd_preprocess(_ptr(d_out), _ptr(out), _ptr(dvec), h, rows, d,
                                            _stream(stream)))
    return dvec


def block_attn_backward(q, k, v, out, lse, d_out, mask: MaskMode, scale: float | None = None, *,
                        d_vec: torch.Tensor | None = None, grads: ChunkGrads | None = None,
                        accumulate_kv: bool = False, deterministic: bool = False,
                        stream=None) -> ChunkGrads:
    """flashcore.hpp:269-337: gradient contributions of one (query chunk, kv chunk) pair.

    Returns fp32 ChunkGrads. With `grads` given, dq is accumulated into grads.dq and
    dk/dv are added (accumulate_kv) or overwritten. `d_vec` (backward_aux) is
    computed when not supplied. deterministic=True adds the dq partials in a
    fixed order (bitwise reproducible; dk/dv always are).
    """
    _check_qkv(q, k, v, "block_attn_backward")
    _req(d_out, torch.bfloat16, "d_out")
    _req(lse, torch.float32, "lse")
    h_q, rows_q, d = q.shape
    h_kv, rows_kv, _ = k.shape
    if out is None and d_vec is None:
        from .errors import StateError
        raise StateError("block_attn_backward: needs the forward output (or its D = backward_aux)")
    if out is not None and tuple(out.shape) != (h_q, rows_q, d):
        _shape_error("block_attn_backward: output shape mismatch")
    if tuple(d_out.shape) != (h_q, rows_q, d):
        _shape_error("block_attn_backward: upstream grad shape mismatch")
    if tuple(lse.shape) != (h_q, rows_q):
        _shape_error("block_attn_backward: logsumexp length mismatch")
    if d_vec is not None:
        _req(d_vec, torch.float32, "d_vec")
        if tuple(d_vec.shape) != (h_q, rows_q):
            _shape_error("block_attn_backward: D length mismatch")
    if grads is not None:
        for t, shape, n in ((grads.dq, (h_q, rows_q, d), "dq"), (grads.dk, (h_kv, rows_kv, d), "dk"),
                            (grads.dv, (h_kv, rows_kv, d), "dv")):
            _req(t, torch.float32, n)
            if tuple(t.shape) != shape:
                _shape_error(f"block_attn_backward: {n} accumulator shape mismatch")
    if d_vec is None:
        d_vec = backward_aux(d_out, out, stream)
    if grads is None:
        grads = ChunkGrads(torch.zeros(h_q, rows_q, d, dtype=torch.float32, device=q.device),
                           torch.empty(h_kv, rows_kv, d, dtype=torch.float32, device=q.device),
                           torch.empty(h_kv, rows_kv, d, dtype=torch.float32, device=q.device))
        accumulate_kv = False
    a = _lib.BwdArgs()
    a.q, a.k, a.v, a.d_out = _ptr(q), _ptr(k), _ptr(v), _ptr(d_out)
    a.lse, a.d_vec = _ptr(lse), _ptr(d_vec)
    a.h_q, a.h_kv, a.rows_q, a.rows_kv, a.d = h_q, h_kv, rows_q, rows_kv, d
    a.dq_acc, a.dk_acc, a.dv_acc = _ptr(grads.dq), _ptr(grads.dk), _ptr(grads.dv)
    a.accumulate_kv = 1 if accumulate_kv else 0
    a.scale = float(scale) if scale is not None else 0.0
    a.mask = int(mask)
    a.deterministic = 1 if deterministic else 0
    check(_lib.lib().da_attn_bwd_chunk(C.byref(a), _stream(stream)))
    return grads
