"""Native schedules (libdistattn_b200.so, csrc/schedule.cpp) against the reference.

Mirrors /root/reference/proj/tests/test_schedule.cpp; tables must be
field-exact with the goldens produced by the reference build.
"""
import json
from fractions import Fraction
from pathlib import Path

import pytest

from paper_2310_03294_b200 import schedule as S
from paper_2310_03294_b200.errors import ConfigError

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.mark.parametrize("kind", ["ring", "balanced"])
def test_tables_field_exact_vs_reference(kind):
    build = S.build_ring_schedule if kind == "ring" else S.build_balanced_schedule
    for ref in json.loads((GOLD / "schedules.json").read_text())[kind]:
        s = build(ref["P"])
        tasks, msgs = s.flat()
        assert s.step_count() == ref["steps"]
        assert [tasks[i:i + 6] for i in range(0, len(tasks), 6)] == ref["tasks"]
        assert [msgs[i:i + 4] for i in range(0, len(msgs), 4)] == ref["messages"]
        assert s.attention_task_count() == ref["attention"]
        assert s.idle_slot_count() == ref["idle"]
        assert s.merge_count() == ref["merges"]
        assert S.idle_fraction(s) == Fraction(*ref["idle_fraction"])
        assert S.expected_speedup(s) == Fraction(*ref["speedup"])


def test_exact_counts_p8():
    # test_schedule.cpp:50-85
    r = S.build_ring_schedule(8)
    assert (r.step_count(), r.attention_task_count(), r.idle_slot_count()) == (8, 36, 28)
    assert S.idle_fraction(r) == Fraction(7, 16) and S.expected_speedup(r) == Fraction(9, 2)
    b = S.build_balanced_schedule(8)
    assert (b.step_count(), b.attention_task_count(), b.idle_slot_count(), b.merge_count()) == \
        (5, 36, 4, 6)
    assert len(b.messages) == 34
    assert S.idle_fraction(b) == Fraction(1, 10) and S.expected_speedup(b) == Fraction(36, 5)
    b7 = S.build_balanced_schedule(7)
    assert (b7.step_count(), b7.idle_slot_count()) == (4, 0)


def test_validate_clean_p_le_64_and_closed_forms():
    for p in range(1, 65):
        assert S.validate(S.build_ring_schedule(p)) == []
        assert S.validate(S.build_balanced_schedule(p)) == []
        assert S.idle_fraction(S.build_ring_schedule(p)) == S.ring_idle_fraction_formula(p)
        assert S.build_balanced_schedule(p).step_count() == (p + 2) // 2
        if p % 2 == 1:
            assert S.idle_fraction(S.build_balanced_schedule(p)) == 0
        elif p >= 4:
            sim = S.idle_fraction(S.build_balanced_schedule(p))
            assert sim == Fraction(1, p + 2) and sim != S.balanced_idle_fraction_reference(p)
        if p >= 2:
            assert S.expected_speedup(S.build_balanced_schedule(p)) >= \
                S.expected_speedup(S.build_ring_schedule(p))


def test_completeness_one_task_per_step():
    for p in range(1, 33):
        for s in (S.build_ring_schedule(p), S.build_balanced_schedule(p)):
            pairs = set()
            for step in s.steps:
                per = {}
                for t in step:
                    if t.is_attention():
                        per[t.worker] = per.get(t.worker, 0) + 1
                        pairs.add((t.query_owner, t.kv_owner))
                assert max(per.values()) <= 1
            assert pairs == {(q, kv) for q in range(1, p + 1) for kv in range(1, q + 1)}


def test_validator_flags_injected_faults():
    # test_schedule.cpp:159-199
    bad = S.build_ring_schedule(3)
    bad.steps[2].append(S.Task(S.TaskKind.RemoteAttn, 3, 3, 2, 0))
    bad.messages.append(S.ScheduleMessage(2, 2, 3, S.PayloadKind.KV))
    v = S.validate(bad)
    assert any("computed 2 times" in m for m in v) and any("primary tasks" in m for m in v)

    s = S.build_balanced_schedule(8)
    for step in s.steps:
        idx = [i for i, t in enumerate(step) if t.kind == S.TaskKind.RescaleMerge]
        if idx:
            del step[idx[0]]
            break
    assert any("never merged" in m for m in S.validate(s))

    s = S.build_ring_schedule(4)
    del s.messages[0]
    assert any("never sent" in m for m in S.validate(s))


def test_fuzz_validator_1000_runs():
    from oracle import oracle as O
    rng = O.Rng(2024)
    for _ in range(1000):
        p = 1 + rng.next_u64() % 32
        balanced = (rng.next_u64() & 1) != 0
        s = S.build_balanced_schedule(p) if balanced else S.build_ring_schedule(p)
        assert S.validate(s) == []


def test_config_errors():
    with pytest.raises(ConfigError):
        S.build_ring_schedule(0)
    with pytest.raises(ConfigError):
        S.build_balanced_schedule(-1)
    with pytest.raises(ConfigError):
        S.ring_idle_fraction_formula(0)


def test_json_csv_shape():
    s = S.build_balanced_schedule(4)
    j = json.loads(S.schedule_to_json(s))
    assert j["P"] == 4 and len(j["steps"]) == 3 and len(j["messages"]) == 7
    assert j["steps"][1][0] == {"task": {"kind": "remote_attn", "kv_owner": 1, "query_owner": 4},
                                "worker": 1}
    csv = S.schedule_to_csv(s).splitlines()
    assert csv[0] == "step,worker,task,query_owner,kv_owner,helper"
    assert "1,4,rescale_merge,,,1" in csv


def test_backward_schedules():
    """Ring backward = the reference run_backward order; balanced backward is
    the extension: same tasks as the balanced forward plus
    GradKV returns, validated with the reference invariants + GradKV coverage."""
    for p in range(1, 33):
        rb = S.build_ring_backward_schedule(p)
        bb = S.build_balanced_backward_schedule(p)
        assert S.validate_backward(rb) == [] and S.validate_backward(bb) == []
        # task tables are the forward ones
        assert rb.steps == S.build_ring_schedule(p).steps
        assert bb.steps == S.build_balanced_schedule(p).steps
        grads = [m for m in bb.messages if m.kind == S.PayloadKind.GradKV]
        direct = [t for st in bb.steps for t in st
                  if t.kind == S.TaskKind.RemoteAttn and t.worker == t.query_owner]
        assert len(grads) == len(direct)
    b8 = S.build_balanced_backward_schedule(8)
    assert S.expected_speedup(b8) == Fraction(36, 5)
    assert S.expected_speedup(S.build_ring_backward_schedule(8)) == Fraction(9, 2)
    # message accounting at P=6 (reference ring backward: 15 GradKV, test_runtime.cpp:234-268)
    r6 = S.build_ring_backward_schedule(6)
    assert sum(1 for m in r6.messages if m.kind == S.PayloadKind.GradKV) == 15


def test_backward_validator_flags_missing_grad():
    s = S.build_balanced_backward_schedule(6)
    idx = [i for i, m in enumerate(s.messages) if m.kind == S.PayloadKind.GradKV][0]
    del s.messages[idx]
    assert any("never returned" in m for m in S.validate_backward(s))
    # and the forward validator rejects stray GradKV messages
    assert any("grad_kv" in m for m in S.validate(S.build_ring_backward_schedule(3)))
