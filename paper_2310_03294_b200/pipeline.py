"""Host-buffer attention step with PCIe transfers overlapped per head group.

The reference's public path takes host matrices (Eigen, runtime.hpp:32-41)
and returns host gradients; its runtime overlaps the next chunk's transfer
with the current chunk's compute (prefetch depth 1, runtime.cpp:280-284,
427-431). ``HostAttention`` applies the same idea to the host<->HBM copies
of a full causal forward+backward on one GPU: the heads are split into
groups, and while group g computes (forward with fused finalize, backward
preprocess, backward, bf16 conversion), group g+1's q/k/v/dO are in flight
host->device on one copy stream and group g-1's dQ/dK/dV device->host on
another. Heads are independent, so the grouping changes no arithmetic: the
result is the same bits as the ungrouped launch on the whole tensor.

Degenerate rows are checked once per call through a shared device flag
(``flashcore.check_degenerate``) instead of one stream sync per group.

Consecutive calls pipeline like the reference's prefetch (depth 1): call
i+1's host->device copy of group g waits only for call i's compute of group
g (not for all of call i), and its compute of group g for call i's
device->host copy of group g. With ``sync=False`` the caller joins the
results onto its stream with ``join()``.
"""
from __future__ import annotations

import torch

from . import _lib
from . import flashcore as F
from .errors import ShapeError, check


class HostAttention:
    """One causal fwd+bwd over pinned host tensors [heads, rows, 128].

    Device buffers are allocated once per shape and reused across calls.
    ``heads_per_group`` trades pipeline fill/drain (smaller groups) against
    wave quantisation of each launch (larger groups).
    """

    def __init__(self, heads: int, rows: int, d: int = 128, heads_per_group: int = 4,
                 device="cuda", compute_streams: int = 3):
        if heads % heads_per_group != 0:
            raise ShapeError(f"heads ({heads}) must be a multiple of heads_per_group "
                             f"({heads_per_group})")
        self.heads, self.rows, self.d, self.hg = heads, rows, d, heads_per_group
        dev = torch.device(device)
        bf = dict(dtype=torch.bfloat16, device=dev)
        f32 = dict(dtype=torch.float32, device=dev)
        self.q, self.k, self.v, self.d_out = (torch.empty(heads, rows, d, **bf) for _ in range(4))
        self.dq = torch.empty(heads, rows, d, **f32)
        self.dk = torch.empty(heads, rows, d, **f32)
        self.dv = torch.empty(heads, rows, d, **f32)
        self.dq16, self.dk16, self.dv16 = (torch.empty(heads, rows, d, **bf) for _ in range(3))
        self.flag = torch.zeros(1, dtype=torch.int32, device=dev)
        self.h2d = torch.cuda.Stream(dev)
        self.d2h = torch.cuda.Stream(dev)
        # groups alternate between compute streams so one group's backward tail
        # overlaps the next group's forward (fills the wave-quantisation gaps)
        self.comp = [torch.cuda.Stream(dev) for _ in range(max(1, compute_streams))]
        self.out = None
        self.lse = None
        # per-group events of the previous call (cross-call pipelining)
        self._prev_comp: list | None = None
        self._prev_d2h: list | None = None
        self._flag_clear = True  # the degenerate flag was checked since it was last set

    @property
    def bytes_in(self) -> int:
        return 4 * self.heads * self.rows * self.d * 2

    @property
    def bytes_out(self) -> int:
        return 3 * self.heads * self.rows * self.d * 2

    def _convert(self, src: torch.Tensor, dst: torch.Tensor, stream) -> None:
        check(_lib.lib().da_convert_f32_bf16(F._ptr(src), F._ptr(dst), src.numel(),
                                             F._stream(stream)))

    def __call__(self, hq, hk, hv, hdo, hdq, hdk, hdv, *, sync: bool = True):
        """q/k/v/dO pinned host bf16 in; dQ/dK/dV pinned host bf16 out.

        Returns after the last device->host copy completed when ``sync``;
        raises DegenerateRowError if any query row attended to no key.
        """
        for t in (hq, hk, hv, hdo, hdq, hdk, hdv):
            if t.shape != (self.heads, self.rows, self.d) or t.dtype != torch.bfloat16:
                raise ShapeError("HostAttention: host tensors must be bf16 "
                                 f"[{self.heads}, {self.rows}, {self.d}]")
        cur = torch.cuda.current_stream()
        if self._flag_clear:  # an unchecked (sync=False) call's flag stays sticky
            self.flag.zero_()
            self._flag_clear = False
        n_groups = self.heads // self.hg
        prev_comp, prev_d2h = self._prev_comp, self._prev_d2h
        fwd_ready = [torch.cuda.Event() for _ in range(n_groups)]  # q, k, v landed
        in_ready = [torch.cuda.Event() for _ in range(n_groups)]  # ... and dO
        out_ready = [torch.cuda.Event() for _ in range(n_groups)]
        # the caller's preceding work (and its timing events) come first
        self.h2d.wait_stream(cur)
        for c in self.comp:
            c.wait_stream(cur)
        comp_done = [torch.cuda.Event() for _ in range(n_groups)]
        d2h_done = [torch.cuda.Event() for _ in range(n_groups)]
        with torch.cuda.stream(self.h2d):
            for g in range(n_groups):
                sl = slice(g * self.hg, (g + 1) * self.hg)
                if prev_comp is not None:  # the previous call's readers of these slices
                    self.h2d.wait_event(prev_comp[g])
                for dst, src in ((self.q, hq), (self.k, hk), (self.v, hv)):
                    dst[sl].copy_(src[sl], non_blocking=True)
                fwd_ready[g].record(self.h2d)
                # dO is first needed by the backward: its copy overlaps the forward
                self.d_out[sl].copy_(hdo[sl], non_blocking=True)
                in_ready[g].record(self.h2d)
        outs, lses = [], []
        for g in range(n_groups):
            sl = slice(g * self.hg, (g + 1) * self.hg)
            comp = self.comp[g % len(self.comp)]
            comp.wait_event(fwd_ready[g])
            if prev_d2h is not None:  # the previous call's copy-out of this group's grads
                comp.wait_event(prev_d2h[g])
            with torch.cuda.stream(comp):
                q, k, v, do = self.q[sl], self.k[sl], self.v[sl], self.d_out[sl]
                out = F.block_attn_update_final(q, k, v, None, F.MaskMode.Diagonal, stream=comp,
                                                degenerate_flag=self.flag)
                comp.wait_event(in_ready[g])
                dvec = F.backward_aux(do, out.o, stream=comp)
                grads = F.ChunkGrads(self.dq[sl], self.dk[sl], self.dv[sl])
                grads.dq.zero_()
                F.block_attn_backward(q, k, v, out.o, out.lse, do, F.MaskMode.Diagonal,
                                      d_vec=dvec, grads=grads, stream=comp)
                for src, dst in ((self.dq, self.dq16), (self.dk, self.dk16), (self.dv, self.dv16)):
                    self._convert(src[sl], dst[sl], comp)
            out_ready[g].record(comp)
            comp_done[g] = out_ready[g]
            self.d2h.wait_event(out_ready[g])
            with torch.cuda.stream(self.d2h):
                for src, dst in ((self.dq16, hdq), (self.dk16, hdk), (self.dv16, hdv)):
                    dst[sl].copy_(src[sl], non_blocking=True)
            d2h_done[g].record(self.d2h)
            outs.append(out.o)
            lses.append(out.lse)
        self._prev_comp, self._prev_d2h = comp_done, d2h_done
        self.out, self.lse = outs, lses  # the rematerialisation state (saved O, LSE) per group
        if sync:
            self.join(cur)
            self.check(cur)
        return hdq, hdk, hdv

    def join(self, stream=None) -> None:
        """Make `stream` (default: current) wait for every call issued so far."""
        stream = stream or torch.cuda.current_stream()
        stream.wait_stream(self.d2h)
        for c in self.comp:
            stream.wait_stream(c)

    def check(self, stream=None) -> None:
        """Raise DegenerateRowError if any joined call saw a row with no visible key."""
        self._flag_clear = True
        F.check_degenerate(self.flag, stream=stream or torch.cuda.current_stream())
