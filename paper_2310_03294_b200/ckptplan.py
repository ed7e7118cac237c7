"""Rematerialization-aware gradient checkpointing on a transformer-layer pipeline.

Mirrors /root/reference/proj/include/distattn/ckptplan.hpp and
src/ckptplan.cpp: the same eight-op layer chain
(norm1, qkv_proj, attention, out_proj, norm2, mlp_up, mlp_act, mlp_down),
the same three strategies and the same segment-wise recomputation algorithm
(ckptplan.cpp:236-305), so plan positions, recompute counts, the cost model
and the saved-scalar accounting equal the reference's (tests/golden/ckpt.json,
dumped from the reference build).

What is real here: the layer is multi-head (d = heads x 128) on the GPU, the
attention op is this library's sm_100a forward (fused finalize -> O, LSE) and
backward kernels, and the projections / MLP are cuBLAS bf16 GEMMs (library
GEMMs: plain matmuls, not the hot path). Under AttentionOutput the backward
consumes the saved O and logsumexp, so the attention forward is never
recomputed (RecomputeTrace.count(Attention) == 0). The backward runs the
attention kernel in its deterministic-dQ mode, and every other op is a
deterministic library call, so gradients are bit-identical across plans —
the reference's cross-plan property (ckptplan.hpp:8-9).
"""
from __future__ import annotations

import enum
import math
from dataclasses import dataclass, field

import torch

from . import flashcore as F
from .errors import ConfigError, ShapeError

HEAD_DIM = 128
NORM_EPS = 1e-6  # ckptplan.cpp:16


class OpKind(enum.IntEnum):
    """ckptplan.hpp:27-36"""
    Norm1 = 0
    QkvProj = 1
    Attention = 2
    OutProj = 3
    Norm2 = 4
    MlpUp = 5
    MlpAct = 6
    MlpDown = 7


OPS_PER_LAYER = 8
NON_ATTENTION_OPS_PER_LAYER = OPS_PER_LAYER - 1
_OP_NAMES = ["norm1", "qkv_proj", "attention", "out_proj", "norm2", "mlp_up", "mlp_act",
             "mlp_down"]


def op_name(k: OpKind) -> str:
    return _OP_NAMES[int(k)]


class CheckpointStrategy(enum.Enum):
    """ckptplan.hpp:60"""
    None_ = "none"
    LayerBoundary = "layer_boundary"
    AttentionOutput = "attention_output"


@dataclass
class LayerWeights:
    wq: torch.Tensor
    wk: torch.Tensor
    wv: torch.Tensor
    wo: torch.Tensor
    w_up: torch.Tensor
    w_down: torch.Tensor


@dataclass
class LayerPipeline:
    """ckptplan.hpp:46-56; d = heads * 128 (the attention op is multi-head)."""
    tokens: int
    heads: int
    d_ff: int
    scale: float
    layers: list = field(default_factory=list)

    @property
    def d(self) -> int:
        return self.heads * HEAD_DIM

    def layer_count(self) -> int:
        return len(self.layers)

    def op_count(self) -> int:
        return self.layer_count() * OPS_PER_LAYER


def make_pipeline(layers: int, tokens: int, heads: int, d_ff: int, seed: int,
                  device="cuda") -> LayerPipeline:
    """ckptplan.cpp:42-65 (weights U[-1/sqrt(d), 1/sqrt(d)], w_down with d_ff),
    drawn from a seeded torch generator and stored bf16 (GEMM operands)."""
    if layers < 1:
        raise ConfigError("pipeline needs at least 1 layer")
    if tokens < 1 or heads < 1 or d_ff < 1:
        raise ConfigError("pipeline dims must be positive")
    d = heads * HEAD_DIM
    g = torch.Generator(device="cpu").manual_seed(seed)

    def u(r, c, w):
        return ((torch.rand(r, c, generator=g, dtype=torch.float64) * 2 - 1) * w).to(
            torch.bfloat16).to(device)

    wd, wff = 1.0 / math.sqrt(d), 1.0 / math.sqrt(d_ff)
    pipe = LayerPipeline(tokens, heads, d_ff, 1.0 / math.sqrt(HEAD_DIM))
    for _ in range(layers):
        pipe.layers.append(LayerWeights(u(d, d, wd), u(d, d, wd), u(d, d, wd), u(d, d, wd),
                                        u(d, d_ff, wd), u(d_ff, d, wff)))
    return pipe


@dataclass
class CheckpointPlan:
    strategy: CheckpointStrategy = CheckpointStrategy.None_
    saved_positions: list = field(default_factory=list)


def plan(pipe: LayerPipeline, strategy: CheckpointStrategy) -> CheckpointPlan:
    """ckptplan.cpp:67-86: value 0 is the input, value i+1 the output of op i."""
    if not pipe.layers:
        raise ConfigError("pipeline needs at least 1 layer")
    p = CheckpointPlan(strategy)
    L = pipe.layer_count()
    if strategy == CheckpointStrategy.None_:
        p.saved_positions = list(range(pipe.op_count() + 1))
    elif strategy == CheckpointStrategy.LayerBoundary:
        p.saved_positions = [l * OPS_PER_LAYER for l in range(L)]
    else:
        p.saved_positions = [0] + [l * OPS_PER_LAYER + int(OpKind.Attention) + 1 for l in range(L)]
    return p


@dataclass
class RecomputeTrace:
    """ckptplan.hpp:74-89"""
    counts: list = field(default_factory=lambda: [0] * OPS_PER_LAYER)

    def count(self, k: OpKind) -> int:
        return self.counts[int(k)]

    def attention_forward_recomputes(self) -> int:
        return self.count(OpKind.Attention)

    def total(self) -> int:
        return sum(self.counts)


@dataclass
class LayerGrads:
    dwq: torch.Tensor = None
    dwk: torch.Tensor = None
    dwv: torch.Tensor = None
    dwo: torch.Tensor = None
    dw_up: torch.Tensor = None
    dw_down: torch.Tensor = None


@dataclass
class PipelineGrads:
    d_input: torch.Tensor = None
    layers: list = field(default_factory=list)


@dataclass
class CkptRunResult:
    output: torch.Tensor
    grads: PipelineGrads
    trace: RecomputeTrace
    attention_forward_launches: int = 0   # forward kernels launched, all phases
    attention_backward_launches: int = 0


# ---------------------------------------------------------------- ops (device)
@dataclass
class _Value:
    """One link of the value chain (ckptplan.cpp:90-95): a/b/c = q/k/v after
    qkv_proj; stat = logsumexp after attention."""
    a: torch.Tensor = None
    b: torch.Tensor = None
    c: torch.Tensor = None
    stat: torch.Tensor = None


def _op_kind(op: int) -> OpKind:
    return OpKind(op % OPS_PER_LAYER)


def _mm(a: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    """bf16 cuBLAS GEMM with fp32 result (activations are kept fp32)."""
    return torch.matmul(a.to(torch.bfloat16), w).float()


def _mm_t(a: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    return torch.matmul(a.to(torch.bfloat16), w.t()).float()


def _wgrad(x: torch.Tensor, g: torch.Tensor) -> torch.Tensor:
    return torch.matmul(x.to(torch.bfloat16).t(), g.to(torch.bfloat16)).float()


def _rms_fwd(x):
    r = torch.rsqrt((x * x).mean(dim=1, keepdim=True) + NORM_EPS)
    return x * r


def _rms_bwd(x, g):
    d = x.shape[1]
    r = torch.rsqrt((x * x).mean(dim=1, keepdim=True) + NORM_EPS)
    gx = (g * x).sum(dim=1, keepdim=True)
    return g * r - x * (gx * r * r * r / d)


def _heads(x: torch.Tensor, h: int) -> torch.Tensor:
    """[tokens, h*128] -> bf16 [h, tokens, 128] (the kernels' layout)."""
    n = x.shape[0]
    return x.view(n, h, HEAD_DIM).permute(1, 0, 2).contiguous().to(torch.bfloat16)


def _tokens(x: torch.Tensor) -> torch.Tensor:
    h, n, _ = x.shape
    return x.permute(1, 0, 2).reshape(n, h * HEAD_DIM).float()


class LocalAttention:
    """The layer's attention op on ONE device: the chunk kernels over the whole
    local sequence (Diagonal mask, fused finalize; deterministic dQ)."""

    def forward(self, q, k, v, scale):
        o = F.block_attn_update_final(q, k, v, None, F.MaskMode.Diagonal, scale)
        return o.o, o.lse

    def backward(self, q, k, v, o, lse, d_out, scale):
        g = F.block_attn_backward(q, k, v, o, lse, d_out, F.MaskMode.Diagonal, scale,
                                  deterministic=True)
        return g.dq, g.dk, g.dv


class SeqParallelAttention:
    """The layer's attention op as DistFlashAttn: the sequence is sharded over
    the ranks of a rank.RankRuntime (one process per GPU), each rank holding
    its contiguous token chunk of every activation; attention runs the
    schedule-driven distributed forward / backward. The
    backward re-installs the layer's saved (q, k, v, O, LSE) — under
    AttentionOutput those are the checkpointed forward outputs, so the
    attention forward is never recomputed (ckptplan.cpp:146-155, 198-206).
    The runtime must be created with deterministic=True for the reference's
    bitwise cross-plan property (ckptplan.hpp:8-9). Every call is collective:
    all ranks run the same plan, so the calls line up."""

    def __init__(self, runtime, fwd_schedule: str = "balanced", bwd_schedule: str = "balanced"):
        self.rt, self.fwd_schedule, self.bwd_schedule = runtime, fwd_schedule, bwd_schedule

    def forward(self, q, k, v, scale):
        if abs(scale - 1.0 / math.sqrt(HEAD_DIM)) > 1e-12:
            raise ConfigError("the per-rank runtime uses scale 1/sqrt(128)")
        out, lse, _ = self.rt.forward(q, k, v, self.fwd_schedule)
        return out, lse

    def backward(self, q, k, v, o, lse, d_out, scale):
        dq, dk, dv, _ = self.rt.backward(d_out, self.bwd_schedule, saved=(q, k, v, o, lse))
        return dq, dk, dv


class _Exec:
    def __init__(self, pipe: LayerPipeline, attention=None):
        self.pipe = pipe
        self.attention = attention if attention is not None else LocalAttention()
        self.fwd_launches = 0
        self.bwd_launches = 0

    def forward(self, op: int, v: _Value) -> _Value:
        """ckptplan.cpp:126-167"""
        pipe = self.pipe
        lw = pipe.layers[op // OPS_PER_LAYER]
        k = _op_kind(op)
        out = _Value()
        if k in (OpKind.Norm1, OpKind.Norm2):
            out.a = _rms_fwd(v.a)
        elif k == OpKind.QkvProj:
            out.a, out.b, out.c = _mm(v.a, lw.wq), _mm(v.a, lw.wk), _mm(v.a, lw.wv)
        elif k == OpKind.Attention:
            h = pipe.heads
            o, lse = self.attention.forward(_heads(v.a, h), _heads(v.b, h), _heads(v.c, h),
                                            pipe.scale)
            self.fwd_launches += 1
            out.a, out.stat = _tokens(o), lse
        elif k == OpKind.OutProj:
            out.a = _mm(v.a, lw.wo)
        elif k == OpKind.MlpUp:
            out.a = _mm(v.a, lw.w_up)
        elif k == OpKind.MlpAct:
            out.a = v.a * torch.sigmoid(v.a)
        else:
            out.a = _mm(v.a, lw.w_down)
        return out

    def backward(self, op: int, vin: _Value, vout: _Value, g: _Value, lg: LayerGrads) -> _Value:
        """ckptplan.cpp:170-229"""
        pipe = self.pipe
        lw = pipe.layers[op // OPS_PER_LAYER]
        k = _op_kind(op)
        dx = _Value()
        if k in (OpKind.Norm1, OpKind.Norm2):
            dx.a = _rms_bwd(vin.a, g.a)
        elif k == OpKind.QkvProj:
            lg.dwq, lg.dwk, lg.dwv = _wgrad(vin.a, g.a), _wgrad(vin.a, g.b), _wgrad(vin.a, g.c)
            dx.a = _mm_t(g.a, lw.wq)
            dx.a += _mm_t(g.b, lw.wk)
            dx.a += _mm_t(g.c, lw.wv)
        elif k == OpKind.Attention:
            # consumes the op's OUTPUT value (O, logsumexp): saved under
            # AttentionOutput, recomputed under LayerBoundary
            h = pipe.heads
            dq, dk, dv = self.attention.backward(_heads(vin.a, h), _heads(vin.b, h),
                                                 _heads(vin.c, h), _heads(vout.a, h), vout.stat,
                                                 _heads(g.a, h), pipe.scale)
            self.bwd_launches += 1
            dx.a, dx.b, dx.c = _tokens(dq), _tokens(dk), _tokens(dv)
        elif k == OpKind.OutProj:
            lg.dwo = _wgrad(vin.a, g.a)
            dx.a = _mm_t(g.a, lw.wo)
        elif k == OpKind.MlpUp:
            lg.dw_up = _wgrad(vin.a, g.a)
            dx.a = _mm_t(g.a, lw.w_up)
        elif k == OpKind.MlpAct:
            s = torch.sigmoid(vin.a)
            dx.a = g.a * (s * (1.0 + vin.a * (1.0 - s)))
        else:
            lg.dw_down = _wgrad(vin.a, g.a)
            dx.a = _mm_t(g.a, lw.w_down)
        return dx


def run_with_checkpointing(pipe: LayerPipeline, p: CheckpointPlan, x: torch.Tensor,
                           d_out: torch.Tensor, executor=None, attention=None) -> CkptRunResult:
    """ckptplan.cpp:236-305: forward keeping only the plan's values, then the
    backward segment by segment, recomputing each from its checkpoint; a
    segment-final attention whose output was saved (AttentionOutput) is not
    recomputed. `executor` (forward/backward per op) defaults to the device
    ops; tests substitute a recording stub to check the control flow on CPU.
    `attention`: LocalAttention (default) or SeqParallelAttention — then x /
    d_out are this rank's token shard and pipe.tokens the shard's rows, and
    the weight gradients are this rank's partial sums (all-reduce them)."""
    if not pipe.layers:
        raise ConfigError("pipeline needs at least 1 layer")
    if tuple(x.shape) != (pipe.tokens, pipe.d):
        raise ShapeError("pipeline input must be tokens x d")
    if tuple(d_out.shape) != (pipe.tokens, pipe.d):
        raise ShapeError("pipeline d_out must be tokens x d")
    if not p.saved_positions or p.saved_positions[0] != 0:
        raise ConfigError("plan must anchor at the pipeline input")
    n_ops = pipe.op_count()
    saved = [False] * (n_ops + 1)
    for pos in p.saved_positions:
        if pos < 0 or pos > n_ops:
            raise ConfigError("saved position out of range")
        saved[pos] = True
    ex = executor if executor is not None else _Exec(pipe, attention)
    store: dict[int, _Value] = {0: _Value(a=x.float())}
    cur = store[0]
    for op in range(n_ops):
        cur = ex.forward(op, cur)
        if saved[op + 1] or op + 1 == n_ops:
            store[op + 1] = cur
    trace = RecomputeTrace()
    grads = PipelineGrads(layers=[LayerGrads() for _ in range(pipe.layer_count())])
    bounds = sorted(p.saved_positions)
    if bounds[-1] != n_ops:
        bounds.append(n_ops)
    g = _Value(a=d_out.float())
    for bi in range(len(bounds) - 1, 0, -1):
        begin, end = bounds[bi - 1], bounds[bi]
        vals = [None] * (end - begin + 1)
        vals[0] = store[begin]
        for op in range(begin, end):
            boundary_attention = (op + 1 == end and saved[op + 1] and
                                  _op_kind(op) == OpKind.Attention)
            if p.strategy == CheckpointStrategy.AttentionOutput and boundary_attention:
                vals[op + 1 - begin] = store[op + 1]
                continue
            if p.strategy == CheckpointStrategy.None_:
                vals[op + 1 - begin] = store[op + 1]
                continue
            vals[op + 1 - begin] = ex.forward(op, vals[op - begin])
            trace.counts[int(_op_kind(op))] += 1
        for op in range(end - 1, begin - 1, -1):
            g = ex.backward(op, vals[op - begin], vals[op + 1 - begin], g,
                            grads.layers[op // OPS_PER_LAYER])
    grads.d_input = g.a
    return CkptRunResult(store[n_ops].a, grads, trace, getattr(ex, "fwd_launches", 0),
                         getattr(ex, "bwd_launches", 0))


# ---------------------------------------------------------------- cost model
@dataclass
class CkptCostModel:
    """ckptplan.hpp:112-120"""
    f_attn: float = 0.0
    f_rest: float = 0.0
    backward: float = 0.0

    def check(self):
        if self.f_attn < 0 or self.f_rest < 0 or self.backward < 0:
            raise ConfigError("checkpoint cost model entries must be non-negative")
        if self.f_attn + self.f_rest <= 0:
            raise ConfigError("checkpoint cost model needs a positive forward cost")


def iteration_time_model(costs: CkptCostModel, layers: int, strategy: CheckpointStrategy) -> float:
    """ckptplan.cpp:314-329"""
    costs.check()
    if layers < 1:
        raise ConfigError("need at least 1 layer")
    fwd = layers * (costs.f_attn + costs.f_rest)
    bwd = layers * costs.backward
    if strategy == CheckpointStrategy.None_:
        return fwd + bwd
    if strategy == CheckpointStrategy.LayerBoundary:
        return fwd + layers * (costs.f_attn + costs.f_rest) + bwd
    return fwd + layers * costs.f_rest + bwd


def recompute_time(trace: RecomputeTrace, costs: CkptCostModel) -> float:
    """ckptplan.cpp:331-341"""
    costs.check()
    t = 0.0
    for k in range(OPS_PER_LAYER):
        per = costs.f_attn if k == int(OpKind.Attention) else costs.f_rest / NON_ATTENTION_OPS_PER_LAYER
        t += per * trace.counts[k]
    return t


def saved_activation_scalars(p: CheckpointPlan, pipe: LayerPipeline) -> int:
    """ckptplan.cpp:343-358"""
    per_layer = pipe.tokens * pipe.d
    if p.strategy == CheckpointStrategy.None_:
        return pipe.layer_count() * (6 * per_layer + 2 * pipe.tokens * pipe.d_ff + 2 * per_layer)
    return pipe.layer_count() * per_layer


def saved_statistic_scalars(p: CheckpointPlan, pipe: LayerPipeline) -> int:
    """ckptplan.cpp:360-364 (the logsumexp rows; x heads in the multi-head layer)."""
    if p.strategy != CheckpointStrategy.AttentionOutput:
        return 0
    return pipe.layer_count() * pipe.tokens * pipe.heads
