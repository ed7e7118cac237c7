"""Host-buffer attention step with PCIe transfers overlapped per head group.

Thin handle on the C++ host pipeline of the library (csrc/host_pipeline.cu,
C ABI ``da_pipeline_*``): pinned host q/k/v/dO in, pinned host bf16 dQ/dK/dV
out, one full causal forward + backward per call. The heads are split into
groups (whole GQA kv groups); group g+1's copy-in and group g-1's copy-out
overlap group g's compute, and consecutive calls pipeline like the
reference's prefetch (depth 1, runtime.cpp:280-284, 427-431): call i+1's
copy-in of group g waits only for call i's compute of group g. Heads are
independent, so the grouping changes no arithmetic.

Degenerate rows are checked once per joined call through a device flag
(``DegenerateRowError``, flashcore.hpp:233-235).
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from .errors import ShapeError, check


class HostAttention:
    """One causal fwd+bwd over pinned host bf16 tensors q/dO [heads, rows, 128],
    k/v [heads_kv, rows, 128] (heads_kv defaults to heads).

    Device buffers are allocated once (at construction) and reused across
    calls. ``heads_per_group`` trades pipeline fill/drain (smaller groups)
    against wave quantisation of each launch (larger groups); it must cover
    whole kv groups.
    """

    def __init__(self, heads: int, rows: int, d: int = 128, heads_per_group: int = 4,
                 device="cuda", compute_streams: int = 3, heads_kv: int | None = None):
        self.heads, self.rows, self.d, self.hg = heads, rows, d, heads_per_group
        self.heads_kv = heads_kv or heads
        self.device = torch.device(device)
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            check(_lib.lib().da_pipeline_create(heads, self.heads_kv, rows, d, heads_per_group,
                                                compute_streams, C.byref(h)))
        self._h = h

    @property
    def bytes_in(self) -> int:
        return 2 * (self.heads + self.heads_kv) * self.rows * self.d * 2

    @property
    def bytes_out(self) -> int:
        return (self.heads + 2 * self.heads_kv) * self.rows * self.d * 2

    def __call__(self, hq, hk, hv, hdo, hdq, hdk, hdv, *, sync: bool = True, stream=None):
        """q/k/v/dO pinned host bf16 in; dQ/dK/dV pinned host bf16 out.

        Returns after the last device->host copy completed when ``sync``;
        raises DegenerateRowError if any query row attended to no key.
        """
        q_shape = (self.heads, self.rows, self.d)
        kv_shape = (self.heads_kv, self.rows, self.d)
        for t, shape in ((hq, q_shape), (hdo, q_shape), (hdq, q_shape), (hk, kv_shape),
                         (hv, kv_shape), (hdk, kv_shape), (hdv, kv_shape)):
            if tuple(t.shape) != shape or t.dtype != torch.bfloat16 or t.is_cuda \
                    or not t.is_contiguous():
                raise ShapeError("HostAttention: host tensors must be contiguous bf16 "
                                 f"{list(shape)}")
        st = stream or torch.cuda.current_stream(self.device)
        check(_lib.lib().da_pipeline_step(self._h, *(C.c_void_p(t.data_ptr()) for t in
                                                     (hq, hk, hv, hdo, hdq, hdk, hdv)),
                                          1 if sync else 0, C.c_void_p(st.cuda_stream)))
        return hdq, hdk, hdv

    def join(self, stream=None) -> None:
        """Make `stream` (default: current) wait for every call issued so far."""
        st = stream or torch.cuda.current_stream(self.device)
        check(_lib.lib().da_pipeline_join(self._h, C.c_void_p(st.cuda_stream), 0))

    def check(self, stream=None) -> None:
        """Raise DegenerateRowError if any joined call saw a row with no visible key."""
        st = stream or torch.cuda.current_stream(self.device)
        check(_lib.lib().da_pipeline_join(self._h, C.c_void_p(st.cuda_stream), 1))

    def outputs(self, stream=None):
        """The last call's saved O (bf16) and LSE (fp32) — the rematerialisation
        state a later backward would reuse — as fresh device tensors."""
        st = stream or torch.cuda.current_stream(self.device)
        o = torch.empty(self.heads, self.rows, self.d, dtype=torch.bfloat16, device=self.device)
        lse = torch.empty(self.heads, self.rows, dtype=torch.float32, device=self.device)
        check(_lib.lib().da_pipeline_outputs(self._h, C.c_void_p(o.data_ptr()),
                                             C.c_void_p(lse.data_ptr()),
                                             C.c_void_p(st.cuda_stream)))
        return o, lse

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().da_pipeline_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass
