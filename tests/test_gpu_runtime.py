"""GPU parity of the full sequence-parallel path (P logical workers on one
B200) against the C oracle (bit-exact with the reference CPU implementation,
see test_oracle.py) on the same seeded inputs.

Tolerances (north_star): O, dQ, dK, dV max-abs error / max|ref| <= 2e-2;
logsumexp max-abs <= 1e-3. Schedules / index maps / counters: exact.
"""
import json
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import oracle as O
from torch_ref import rel_err

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"
TOL, LSE_TOL = 2e-2, 1e-3


def _np(t):
    return t.detach().float().cpu().numpy().astype(np.float64)


def _cat(shards, name):
    return torch.cat([getattr(s, name) for s in shards], dim=1)


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def test_device_make_shards_is_the_reference_index_map(cuda):
    from paper_2310_03294_b200.runtime import make_parity_shards
    shards = make_parity_shards(0, 4, 512, 2, 128)
    q, k, v, do = O.make_inputs(0, 4, 512, 128, 2, bf16=True)
    assert np.array_equal(_np(_cat(shards, "q")), q)
    assert np.array_equal(_np(_cat(shards, "k")), k)
    assert np.array_equal(_np(_cat(shards, "v")), v)
    assert np.array_equal(_np(_cat(shards, "d_out")), do)


def _check_against_oracle(shards, P, n, sched, heads, trace_f=None, trace_b=None, heads_kv=None,
                          bwd="ring"):
    heads_kv = heads_kv or heads
    group = heads // heads_kv
    q, k, v, do = (_np(_cat(shards, f)) for f in ("q", "k", "v", "d_out"))
    out, lse = _np(_cat(shards, "out")), _np(_cat(shards, "lse"))
    dq, dk, dv = (_np(_cat(shards, f)) for f in ("dq", "dk", "dv"))
    dk_ref = np.zeros_like(dk)
    dv_ref = np.zeros_like(dv)
    for h in range(heads):
        hk = h // group
        o_r, l_r, cf = O.run_forward(q[h], k[hk], v[hk], P, sched)
        if bwd == "ring":
            dq_r, dk_r, dv_r, cb = O.run_backward(q[h], k[hk], v[hk], o_r, l_r, do[h], P)
        else:
            dq_r, dk_r, dv_r, cb = O.run_backward_sched(q[h], k[hk], v[hk], o_r, l_r, do[h], P, bwd)
        assert _rel(out[h], o_r) < TOL, ("out", h)
        assert np.abs(lse[h] - l_r).max() < LSE_TOL, ("lse", h)
        assert _rel(dq[h], dq_r) < TOL, ("dq", h)
        dk_ref[hk] += dk_r
        dv_ref[hk] += dv_r
        if trace_f is not None and heads == 1:
            c = trace_f.counters
            assert [c.kv_scalars, c.q_scalars, c.partial_scalars, c.grad_scalars, c.kv_messages,
                    c.q_messages, c.partial_messages, c.grad_messages] == cf[:8]
            assert trace_f.attention_kernel_calls == cf[8]
            c = trace_b.counters
            assert [c.kv_scalars, c.q_scalars, c.partial_scalars, c.grad_scalars, c.kv_messages,
                    c.q_messages, c.partial_messages, c.grad_messages] == cb[:8]
            assert trace_b.attention_kernel_calls == cb[8]
    assert _rel(dk, dk_ref) < TOL and _rel(dv, dv_ref) < TOL


@pytest.mark.parametrize("sched", ["balanced", "ring"])
def test_cfg1_single_head_4096_p4(cuda, sched):
    """BASELINE.json configs[0]: 1 head, seq 4096, d=128, P=4 simulated workers."""
    from paper_2310_03294_b200.runtime import make_parity_shards, run_backward, run_forward
    shards = make_parity_shards(0, 4, 4096, 1, 128)
    tf = run_forward(shards, sched)
    tb = run_backward(shards)
    torch.cuda.synchronize()
    _check_against_oracle(shards, 4, 4096, sched, 1, tf, tb)


@pytest.mark.parametrize("P,n,heads", [(1, 512, 2), (2, 1024, 1), (8, 2048, 1), (3, 384, 2),
                                       (6, 768, 1), (4, 200, 1)])
def test_worker_counts_balanced(cuda, P, n, heads):
    from paper_2310_03294_b200.runtime import make_parity_shards, run_backward, run_forward
    shards = make_parity_shards(11, P, n, heads, 128)
    tf = run_forward(shards, "balanced")
    tb = run_backward(shards)
    torch.cuda.synchronize()
    _check_against_oracle(shards, P, n, "balanced", heads, tf, tb)


@pytest.mark.parametrize("P,n", [(4, 4096), (5, 1280), (8, 2048)])
def test_balanced_backward(cuda, P, n):
    """Load-balanced backward (extension): same gradients, balanced pairs."""
    from paper_2310_03294_b200.runtime import make_parity_shards, run_backward, run_forward
    shards = make_parity_shards(2, P, n, 1, 128)
    tf = run_forward(shards, "balanced")
    tb = run_backward(shards, "balanced")
    torch.cuda.synchronize()
    _check_against_oracle(shards, P, n, "balanced", 1, tf, tb, bwd="balanced")


def test_gqa_4q_2kv(cuda):
    from paper_2310_03294_b200.runtime import make_parity_shards, run_backward, run_forward
    shards = make_parity_shards(3, 2, 1024, 4, 128, heads_kv=2)
    run_forward(shards, "balanced")
    run_backward(shards)
    torch.cuda.synchronize()
    _check_against_oracle(shards, 2, 1024, "balanced", 4, heads_kv=2)


def test_golden_fixture_from_reference_build(cuda):
    """tests/golden/numerics_d128.npz was produced by the reference's own code."""
    from paper_2310_03294_b200.runtime import make_parity_shards, run_backward, run_forward
    gold = np.load(GOLD / "numerics_d128.npz")
    meta = json.loads((GOLD / "numerics_d128.json").read_text())["heads"][0]
    shards = make_parity_shards(0, 4, 512, 1, 128)
    tf = run_forward(shards, "balanced")
    run_backward(shards)
    torch.cuda.synchronize()
    assert _rel(_np(_cat(shards, "out"))[0], gold["out"]) < TOL
    assert np.abs(_np(_cat(shards, "lse"))[0] - gold["lse"]).max() < LSE_TOL
    for f in ("dq", "dk", "dv"):
        assert _rel(_np(_cat(shards, f))[0], gold[f]) < TOL, f
    c = tf.counters
    assert [c.kv_scalars, c.q_scalars, c.partial_scalars, c.grad_scalars, c.kv_messages,
            c.q_messages, c.partial_messages, c.grad_messages] == meta["fwd_counters"]


def test_ring_and_balanced_agree_and_state_errors(cuda):
    from paper_2310_03294_b200.errors import StateError
    from paper_2310_03294_b200.runtime import make_parity_shards, run_backward, run_forward
    a = make_parity_shards(5, 8, 1024, 2, 128)
    b = make_parity_shards(5, 8, 1024, 2, 128)
    run_forward(a, "ring")
    run_forward(b, "balanced")
    for x, y in zip(a, b):
        assert (x.out.float() - y.out.float()).abs().max().item() <= 2 ** -7
        assert (x.lse - y.lse).abs().max().item() < 1e-4
    c = make_parity_shards(5, 2, 256, 1, 128)
    with pytest.raises(StateError):
        run_backward(c)


@pytest.mark.parametrize("P,n,heads,heads_kv", [(4, 4096, 1, 1), (2, 1024, 1, 1), (8, 2048, 2, 2),
                                                (6, 1500, 1, 1), (4, 1024, 4, 2)])
def test_balanced_split_forward(cuda, P, n, heads, heads_kv):
    """Even-P last-step split (extension): half-pair tasks on packed kv row
    halves, the same results as the oracle stepper running the same table;
    counters equal (H=1) — half KV messages are counted at their size."""
    from paper_2310_03294_b200.runtime import make_parity_shards, run_backward, run_forward
    shards = make_parity_shards(5, P, n, heads, 128, heads_kv=heads_kv)
    tf = run_forward(shards, "balanced_split")
    tb = run_backward(shards)
    torch.cuda.synchronize()
    _check_against_oracle(shards, P, n, "balanced_split", heads, tf, tb, heads_kv=heads_kv)


@pytest.mark.parametrize("P,n,heads,heads_kv", [(4, 4096, 1, 1), (2, 1002, 1, 1), (8, 2048, 2, 2),
                                                (4, 1024, 4, 2), (5, 1280, 1, 1)])
def test_balanced_split_backward(cuda, P, n, heads, heads_kv):
    """Backward of the split schedule (extension): the split step's halves on
    packed kv rows, their dk/dv folded into the kv owner's rows; gradients and
    counters (H=1) equal to the oracle running the same table; odd P is the
    balanced backward."""
    from paper_2310_03294_b200.runtime import make_parity_shards, run_backward, run_forward
    shards = make_parity_shards(6, P, n, heads, 128, heads_kv=heads_kv)
    tf = run_forward(shards, "balanced_split")
    tb = run_backward(shards, "balanced_split")
    torch.cuda.synchronize()
    _check_against_oracle(shards, P, n, "balanced_split", heads, tf, tb, heads_kv=heads_kv,
                          bwd="balanced_split")


def test_p1_backward_is_the_single_chunk_kernel(cuda):
    """test_runtime.cpp:201-213: with one worker the runtime backward is one
    block_attn_backward call (dk/dv bitwise; dq to fp32 reduction order)."""
    from paper_2310_03294_b200.flashcore import MaskMode, block_attn_backward
    from paper_2310_03294_b200.runtime import make_parity_shards, run_backward, run_forward
    shards = make_parity_shards(9, 1, 1024, 2, 128)
    run_forward(shards, "ring")
    run_backward(shards)
    s = shards[0]
    g = block_attn_backward(s.q, s.k, s.v, s.out, s.lse, s.d_out, MaskMode.Diagonal)
    torch.cuda.synchronize()
    assert torch.equal(g.dk, s.dk) and torch.equal(g.dv, s.dv)
    assert float((g.dq - s.dq).abs().max() / g.dq.abs().max()) < 1e-5


def test_invalid_schedule_and_mismatched_shards_are_rejected(cuda):
    """test_runtime.cpp:278-287"""
    from paper_2310_03294_b200 import schedule as S
    from paper_2310_03294_b200.errors import ScheduleError, ShapeError
    from paper_2310_03294_b200.runtime import make_parity_shards, run_forward
    shards = make_parity_shards(1, 4, 512, 1, 128)
    bad = S.build_ring_schedule(4)
    bad.steps[1][1] = S.Task(S.TaskKind.Idle, 2)
    with pytest.raises(ScheduleError):
        run_forward(shards, bad)
    small = make_parity_shards(1, 4, 512, 1, 128)
    small[2].q = small[2].q[:, :64].contiguous()
    with pytest.raises(ShapeError):
        run_forward(small, "ring")


def test_runtime_takes_any_valid_schedule_table(cuda):
    """run_forward / run_backward accept a Schedule object, not only a kind
    (runtime.hpp:106-118 take `const Schedule&`): a valid table that is none
    of the built-ins (ring with steps 1 and 2 swapped) runs through
    da_run_forward_table; the built-in tables passed as objects give the same
    bits as the kind entry points."""
    import dataclasses

    from paper_2310_03294_b200 import schedule as S
    from paper_2310_03294_b200.runtime import make_parity_shards, run_backward, run_forward

    def outs(sh):
        return [torch.cat([getattr(x, f) for x in sh], 1).clone() for f in ("out", "lse")]

    base = make_parity_shards(3, 4, 1024, 2, 128)
    run_forward(base, "ring")
    run_backward(base, "ring")
    ref = outs(base)
    ref_g = [torch.cat([getattr(x, f) for x in base], 1).clone() for f in ("dq", "dk", "dv")]

    same = make_parity_shards(3, 4, 1024, 2, 128)
    run_forward(same, S.build_ring_schedule(4))
    run_backward(same, S.build_ring_backward_schedule(4))
    got = outs(same)
    assert torch.equal(got[0], ref[0]) and torch.equal(got[1], ref[1])
    for f, r in zip(("dq", "dk", "dv"), ref_g):  # dq: unordered fp32 reductions by default
        g = torch.cat([getattr(x, f) for x in same], 1)
        assert (torch.equal(g, r) if f != "dq" else rel_err(g, r) < 1e-5), f

    custom = S.build_ring_schedule(4)
    custom.steps[1], custom.steps[2] = custom.steps[2], custom.steps[1]
    custom.messages = sorted((dataclasses.replace(m, step=3 - m.step) if m.step in (1, 2) else m
                              for m in custom.messages), key=lambda m: (m.step, m.from_))
    assert S.validate(custom) == []
    other = make_parity_shards(3, 4, 1024, 2, 128)
    run_forward(other, custom)
    o = outs(other)
    assert rel_err(o[0], ref[0]) < 1e-2 and (o[1] - ref[1]).abs().max().item() < 1e-4
