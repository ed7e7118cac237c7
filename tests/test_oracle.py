"""Pins the C oracle (oracle/distattn_oracle.c) to the reference.

Sources of truth, in order: the golden vectors committed under tests/golden/
(produced by the unmodified reference build, oracle/make_golden.py), the
reference's own unit-test constants (cited), and — when oracle/_ref exists in
this checkout — a live run of the reference build.
"""
import json
import math
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O

GOLD = Path(__file__).resolve().parent / "golden"


def test_rng_known_answers():
    # test_numerics.cpp:100-105
    r = O.Rng(0)
    assert [r.next_u64() for _ in range(3)] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4,
                                                0x06C45D188009454F]
    g = json.loads((GOLD / "rng.json").read_text())
    r = O.Rng(0)
    assert [str(r.next_u64()) for _ in range(8)] == g["seed0_u64"]
    r = O.Rng(12345)
    assert [r.next_unit() for _ in range(8)] == g["seed12345_unit"]
    r = O.Rng(7)
    child = r.fork()
    assert str(child.next_u64()) == g["fork7_child_u64"]
    assert str(r.next_u64()) == g["fork7_parent_next"]


@pytest.mark.parametrize("kind", ["ring", "balanced"])
def test_schedules_field_exact(kind):
    g = json.loads((GOLD / "schedules.json").read_text())[kind]
    for ref in g:
        steps, tasks, msgs = O.schedule_flat(ref["P"], kind)
        assert steps == ref["steps"]
        assert tasks == ref["tasks"]
        assert msgs == ref["messages"]


def _small_cases():
    meta = json.loads((GOLD / "numerics_small.json").read_text())
    return sorted(meta)


@pytest.mark.parametrize("key", _small_cases())
def test_runtime_bit_exact_vs_reference_goldens(key):
    meta = json.loads((GOLD / "numerics_small.json").read_text())[key]
    gold = np.load(GOLD / "numerics_small.npz")
    P = int(key.split("_")[0][1:])
    N = int(key.split("_")[1][1:])
    d = int(key.split("_")[2][1:])
    sched = key.split("_")[3]
    q, k, v, do = O.make_inputs(0, P, N, d, 1, bf16=False)
    out, lse, cf = O.run_forward(q[0], k[0], v[0], P, sched)
    dq, dk, dv, cb = O.run_backward(q[0], k[0], v[0], out, lse, do[0], P)
    for name, arr in (("out", out), ("lse", lse), ("dq", dq), ("dk", dk), ("dv", dv)):
        assert np.array_equal(arr, gold[f"{key}/{name}"]), name
    assert cf[:8] == meta["fwd_counters"]
    assert cb[:8] == meta["bwd_counters"]
    assert cf[8] == meta["fwd_kernel_calls"] and cb[8] == meta["bwd_kernel_calls"]


def test_d128_bf16_fixture():
    gold = np.load(GOLD / "numerics_d128.npz")
    meta = json.loads((GOLD / "numerics_d128.json").read_text())
    q, k, v, do = O.make_inputs(0, 4, 512, 128, 1, bf16=True)
    out, lse, cf = O.run_forward(q[0], k[0], v[0], 4, "balanced")
    dq, dk, dv, cb = O.run_backward(q[0], k[0], v[0], out, lse, do[0], 4)
    for name, arr in (("out", out), ("lse", lse), ("dq", dq), ("dk", dk), ("dv", dv)):
        assert np.array_equal(arr.astype(np.float32), gold[name]), name
    assert cf[:8] == meta["heads"][0]["fwd_counters"]


def test_blockwise_matches_dense_and_rescale_identity():
    # test_flashcore.cpp:54-126 style properties
    q, k, v, do = O.make_inputs(3, 1, 48, 8, 1, bf16=False)
    q, k, v, do = q[0], k[0], v[0], do[0]
    scale = 1 / math.sqrt(8)
    ref_o, ref_lse = O.dense_oracle(q, k, v, True, scale)
    acc = O.block_attn_update(q, k, v, None, "diagonal", scale, (5, 7))
    o, lse = O.finalize(acc)
    assert np.abs(o - ref_o).max() < 1e-12 and np.abs(lse - ref_lse).max() < 1e-12
    fresh = (np.zeros_like(acc[0]), np.full(48, -np.inf), np.zeros(48))
    same = O.rescale(fresh, acc)
    assert all(np.array_equal(a, b) for a, b in zip(same, acc))
    empty = O.block_attn_update(q, k, v, acc, "empty", scale)
    assert all(np.array_equal(a, b) for a, b in zip(empty, acc))
    # chunked backward contributions add up to the dense gradient (test_flashcore.cpp:312-334)
    dq_ref, dk_ref, dv_ref = O.dense_backward(q, k, v, do, True, scale)
    dq, dk, dv = O.block_attn_backward(q, k, v, ref_o, ref_lse, do, "diagonal", scale, (4, 6))
    for a, b in ((dq, dq_ref), (dk, dk_ref), (dv, dv_ref)):
        assert np.abs(a - b).max() < 1e-10


def test_degenerate_row_is_an_error():
    acc = (np.zeros((2, 4)), np.full(2, -np.inf), np.zeros(2))
    with pytest.raises(O.OracleError):
        O.finalize(acc)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built in this checkout")
def test_live_reference_bit_exact():
    ref, meta = O.ref_run(64, 8, 2, 16, 5, "balanced", bf16=True)
    q, k, v, do = O.make_inputs(5, 8, 64, 16, 2, bf16=True)
    assert np.array_equal(q, ref["q"]) and np.array_equal(do, ref["d_out"])
    for h in range(2):
        out, lse, cf = O.run_forward(q[h], k[h], v[h], 8, "balanced")
        dq, dk, dv, _ = O.run_backward(q[h], k[h], v[h], out, lse, do[h], 8)
        assert np.array_equal(out, ref["out"][h]) and np.array_equal(lse, ref["lse"][h])
        assert np.array_equal(dq, ref["dq"][h]) and np.array_equal(dk, ref["dk"][h])
        assert np.array_equal(dv, ref["dv"][h])
        assert cf[:8] == meta["heads"][h]["fwd_counters"]
