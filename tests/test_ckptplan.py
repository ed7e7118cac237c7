"""Rematerialization-aware checkpointing, mirroring
/root/reference/proj/tests/test_ckptplan.cpp.

CPU: plan positions, recompute counts of the segment algorithm, the cost model
and saved-scalar accounting equal the reference build's (tests/golden/ckpt.json,
dumped by oracle/ref_driver ckpt). GPU: the multi-head layer pipeline on the
sm_100a attention kernels — bit-identical gradients across the three plans,
no attention forward recompute under AttentionOutput, and agreement with a
plain PyTorch fp32 autograd reference of the same pipeline.
"""
import json
import math
from pathlib import Path

import pytest
import torch

from paper_2310_03294_b200 import ckptplan as K
from paper_2310_03294_b200.errors import ConfigError, ShapeError

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "ckpt.json").read_text())
STRATS = {"none": K.CheckpointStrategy.None_, "layer_boundary": K.CheckpointStrategy.LayerBoundary,
          "attention_output": K.CheckpointStrategy.AttentionOutput}


class _Stub:
    """Records the op calls; values are placeholders (control flow only)."""

    def __init__(self):
        self.fwd_launches = 0
        self.bwd_launches = 0

    def forward(self, op, v):
        if op % K.OPS_PER_LAYER == K.OpKind.Attention:
            self.fwd_launches += 1
        return K._Value(a=v.a)

    def backward(self, op, vin, vout, g, lg):
        if op % K.OPS_PER_LAYER == K.OpKind.Attention:
            self.bwd_launches += 1
        return K._Value(a=g.a)


def _host_pipe(L):
    return K.LayerPipeline(tokens=12, heads=1, d_ff=8, scale=1.0, layers=[None] * L)


@pytest.mark.parametrize("case", GOLD["cases"], ids=lambda c: f"L{c['layers']}-{c['strategy']}")
def test_plans_counts_and_cost_model_equal_reference(case):
    L, st = case["layers"], STRATS[case["strategy"]]
    pipe = _host_pipe(L)
    p = K.plan(pipe, st)
    assert p.saved_positions == case["positions"]
    x = torch.zeros(12, pipe.d)
    r = K.run_with_checkpointing(pipe, p, x, x, executor=_Stub())
    assert r.trace.counts == case["counts"]
    cost = K.CkptCostModel(*GOLD["cost"])
    assert K.iteration_time_model(cost, L, st) == case["iteration_time"]
    assert K.recompute_time(r.trace, cost) == pytest.approx(case["recompute_time"], abs=1e-12)
    # the reference's per-layer tensor is tokens x d with its toy d = 4, d_ff = 8
    d_ref, per = 4, 12 * 4
    expect = case["saved_activation_scalars"]
    ours = K.saved_activation_scalars(p, pipe)
    if st == K.CheckpointStrategy.None_:
        assert expect == L * (8 * per + 2 * 12 * 8)
        assert ours == L * (8 * 12 * pipe.d + 2 * 12 * 8)
    else:
        assert expect == L * 12 * d_ref and ours == L * 12 * pipe.d
    # attention forward is launched once per layer in the forward pass, plus the
    # recomputes of the plan; the backward launches it once per layer
    assert r.attention_forward_launches == L + r.trace.attention_forward_recomputes()
    assert r.attention_backward_launches == L


def test_errors_mirror_reference():
    pipe = _host_pipe(1)
    with pytest.raises(ConfigError):
        K.plan(K.LayerPipeline(12, 1, 8, 1.0, []), K.CheckpointStrategy.None_)
    with pytest.raises(ConfigError):
        K.run_with_checkpointing(pipe, K.CheckpointPlan(K.CheckpointStrategy.None_, [1]),
                                 torch.zeros(12, 128), torch.zeros(12, 128), executor=_Stub())
    with pytest.raises(ShapeError):
        K.run_with_checkpointing(pipe, K.plan(pipe, K.CheckpointStrategy.None_),
                                 torch.zeros(11, 128), torch.zeros(12, 128), executor=_Stub())
    with pytest.raises(ConfigError):
        K.iteration_time_model(K.CkptCostModel(-1, 1, 1), 1, K.CheckpointStrategy.None_)
    with pytest.raises(ConfigError):
        K.iteration_time_model(K.CkptCostModel(0, 0, 1), 1, K.CheckpointStrategy.None_)


def test_attention_output_saves_one_forward_per_layer():
    cost = K.CkptCostModel(f_attn=2.0, f_rest=3.0, backward=9.0)
    for L in (1, 4, 32):
        lb = K.iteration_time_model(cost, L, K.CheckpointStrategy.LayerBoundary)
        ao = K.iteration_time_model(cost, L, K.CheckpointStrategy.AttentionOutput)
        assert lb - ao == L * cost.f_attn


# ---------------------------------------------------------------- GPU
def _torch_reference(pipe, x, d_out):
    """The same pipeline in fp32 PyTorch autograd (weights = the bf16 values)."""
    x = x.detach().clone().requires_grad_(True)
    ws = [[w.float().detach().clone().requires_grad_(True) for w in
           (lw.wq, lw.wk, lw.wv, lw.wo, lw.w_up, lw.w_down)] for lw in pipe.layers]
    h, n = pipe.heads, pipe.tokens
    cur = x
    for wq, wk, wv, wo, wu, wdn in ws:
        cur = cur * torch.rsqrt((cur * cur).mean(1, keepdim=True) + K.NORM_EPS)
        q, k, v = cur @ wq, cur @ wk, cur @ wv
        sh = lambda t: t.view(n, h, 128).permute(1, 0, 2)  # noqa: E731
        s = sh(q) @ sh(k).transpose(1, 2) * pipe.scale
        s = s.masked_fill(torch.ones(n, n, dtype=torch.bool, device=x.device).triu(1), -math.inf)
        o = (torch.softmax(s, -1) @ sh(v)).permute(1, 0, 2).reshape(n, h * 128)
        cur = o @ wo
        cur = cur * torch.rsqrt((cur * cur).mean(1, keepdim=True) + K.NORM_EPS)
        u = cur @ wu
        cur = (u * torch.sigmoid(u)) @ wdn
    cur.backward(d_out)
    return cur.detach(), x.grad, [[w.grad for w in lw] for lw in ws]


def _rel(a, b):
    return float((a.float() - b.float()).abs().max() / b.float().abs().max().clamp_min(1e-30))


@pytest.mark.gpu
def test_gpu_layer_pipeline_bitwise_across_plans(cuda):
    L, n, heads, d_ff = 2, 384, 2, 512
    pipe = K.make_pipeline(L, n, heads, d_ff, seed=3)
    g = torch.Generator().manual_seed(4)
    x = (torch.rand(n, pipe.d, generator=g) * 2 - 1).to(cuda)
    d_out = (torch.rand(n, pipe.d, generator=g) * 2 - 1).to(cuda)
    runs = {s: K.run_with_checkpointing(pipe, K.plan(pipe, s), x, d_out)
            for s in K.CheckpointStrategy}
    torch.cuda.synchronize()
    base = runs[K.CheckpointStrategy.None_]
    for s, r in runs.items():
        assert torch.equal(r.output, base.output)
        assert torch.equal(r.grads.d_input, base.grads.d_input), s
        for la, lb in zip(r.grads.layers, base.grads.layers):
            for f in ("dwq", "dwk", "dwv", "dwo", "dw_up", "dw_down"):
                assert torch.equal(getattr(la, f), getattr(lb, f)), (s, f)
    ao = runs[K.CheckpointStrategy.AttentionOutput]
    lb = runs[K.CheckpointStrategy.LayerBoundary]
    assert ao.trace.attention_forward_recomputes() == 0 and ao.attention_forward_launches == L
    assert lb.trace.attention_forward_recomputes() == L and lb.attention_forward_launches == 2 * L
    out_r, dx_r, dws_r = _torch_reference(pipe, x, d_out)
    assert _rel(ao.output, out_r) < 2e-2
    assert _rel(ao.grads.d_input, dx_r) < 3e-2
    for lg, wr in zip(ao.grads.layers, dws_r):
        for f, ref in zip(("dwq", "dwk", "dwv", "dwo", "dw_up", "dw_down"), wr):
            assert _rel(getattr(lg, f), ref) < 3e-2, f
