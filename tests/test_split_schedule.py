"""Even-P last-step split of the balanced schedule (extension).

Not in the reference: its balanced schedule idles helpers 1..P/2 at t = P/2
(schedule.cpp:95-97). The split mode gives each of them the low half of the kv
rows of the pair (p + P/2, p) and the owner the high half. Pinned here by:
hand tables (P = 2, 4), the native builder == the C oracle restatement, the
reference validator's invariants extended to half coverage, and the oracle
stepper reproducing the dense causal attention.
"""
from fractions import Fraction

import numpy as np
import pytest

from oracle import oracle as O
from paper_2310_03294_b200 import schedule as S

K = S.TaskKind


def _rows(s):
    return [(t.worker, int(t.kind), t.query_owner, t.kv_owner, t.helper) for t in s.steps[-1]]


def test_hand_tables_p2_p4():
    s2 = S.build_balanced_split_schedule(2)
    assert s2.step_count() == 2
    # t1: w1 helps owner 2 on kv1 low half; w2 direct on kv1 high half; merge at w2
    assert _rows(s2) == [(1, 1, 2, 1, 1), (2, 1, 2, 1, 2), (2, 2, 0, 0, 1)]
    assert [(m.from_, m.to, int(m.kind)) for m in s2.messages] == [(2, 1, 1), (1, 2, 2), (1, 2, 4)]
    s4 = S.build_balanced_split_schedule(4)
    assert s4.step_count() == 3 and s4.idle_slot_count() == 0
    assert _rows(s4) == [(1, 1, 3, 1, 1), (2, 1, 4, 2, 1), (3, 1, 3, 1, 2), (4, 1, 4, 2, 2),
                         (3, 2, 0, 0, 1), (4, 2, 0, 0, 2)]
    # steps before the last are the reference's balanced steps
    b4 = S.build_balanced_schedule(4)
    assert s4.steps[:2] == b4.steps[:2]


@pytest.mark.parametrize("P", [1, 2, 3, 4, 5, 6, 7, 8, 12, 16])
def test_native_builder_equals_oracle_restatement(P):
    steps, tasks, msgs = O.schedule_flat(P, "balanced_split")
    s = S.build_balanced_split_schedule(P)
    t, m = s.flat()
    assert steps == s.step_count()
    assert [x for r in tasks for x in r] == t and [x for r in msgs for x in r] == m


def test_odd_p_is_the_reference_balanced_schedule():
    for P in (1, 3, 5, 7, 9, 31):
        assert S.build_balanced_split_schedule(P).flat() == S.build_balanced_schedule(P).flat()


def test_validate_clean_and_no_idle_p_le_64():
    for P in range(1, 65):
        s = S.build_balanced_split_schedule(P)
        assert S.validate(s) == [], P
        assert s.idle_slot_count() == 0
        assert s.step_count() == P // 2 + 1


def test_validator_half_coverage_faults():
    s = S.build_balanced_split_schedule(4)
    # drop the owner's high half: pair (3, 1) only partly computed, KVHalf unconsumed
    bad = S.Schedule(s.workers, [list(st) for st in s.steps], list(s.messages))
    i = next(i for i, t in enumerate(bad.steps[2]) if t.worker == 3)
    bad.steps[2][i] = S.Task(K.Idle, 3)
    v = S.validate(bad)
    assert any("pair (q=3, kv=1) is only partly computed (low half)" in x for x in v)
    assert any("kv_half) is never consumed" in x for x in v)
    # the owner takes the whole chunk as well: the low half is computed twice
    bad2 = S.Schedule(s.workers, [list(st) for st in s.steps], list(s.messages))
    bad2.steps[2][i] = S.Task(K.RemoteAttn, 3, 3, 1, 0)
    v2 = S.validate(bad2)
    assert any("pair (q=3, kv=1) computed 2 times" in x for x in v2)
    # unknown part
    bad3 = S.Schedule(s.workers, [list(st) for st in s.steps], list(s.messages))
    bad3.steps[2][i] = S.Task(K.RemoteAttn, 3, 3, 1, 7)
    assert any("unknown kv part 7" in x for x in S.validate(bad3))


def test_weighted_speedup_ceilings():
    half = Fraction(1, 2)
    ring, bal, split = (S.build_ring_schedule(8), S.build_balanced_schedule(8),
                        S.build_balanced_split_schedule(8))
    assert S.weighted_makespan(ring, half) == Fraction(15, 2)
    assert S.weighted_makespan(bal, half) == Fraction(9, 2)
    assert S.weighted_makespan(split, half) == 4
    # balanced over ring 5/3 (the reference ceiling), split over ring 15/8
    assert S.weighted_makespan(ring, half) / S.weighted_makespan(bal, half) == Fraction(5, 3)
    assert S.weighted_makespan(ring, half) / S.weighted_makespan(split, half) == Fraction(15, 8)
    for P in range(2, 33, 2):
        assert S.weighted_makespan(S.build_balanced_split_schedule(P), half) == \
            S.weighted_makespan(S.build_balanced_schedule(P), half) - half


def test_json_marks_the_half_tasks():
    j = S.schedule_to_json(S.build_balanced_split_schedule(2))
    assert '"kv_part": "low"' in j and '"kv_part": "high"' in j and '"kv_half"' in j


@pytest.mark.parametrize("P,n", [(2, 64), (4, 128), (6, 96), (8, 256), (4, 132)])
def test_oracle_stepper_split_matches_dense_and_balanced(P, n):
    q, k, v, _ = O.make_inputs(3, P, n, 16, 1)
    q, k, v = q[0], k[0], v[0]
    out_s, lse_s, c_s = O.run_forward(q, k, v, P, "balanced_split")
    out_b, lse_b, c_b = O.run_forward(q, k, v, P, "balanced")
    o_ref, lse_ref = O.dense_oracle(q, k, v, True, 1.0 / np.sqrt(16))
    assert np.abs(out_s - o_ref).max() < 1e-10 and np.abs(lse_s - lse_ref).max() < 1e-10
    assert np.abs(out_s - out_b).max() < 1e-12
    rows = n // P
    # counters (runtime.cpp:50-83 accounting): the split step moves half a KV
    # chunk per owner instead of a whole one, plus one Q and one Partial each
    assert c_s[0] == c_b[0] - (P // 2) * 2 * rows * 16 + (P // 2) * 2 * (rows - rows // 2) * 16
    assert c_s[1] == c_b[1] + (P // 2) * rows * 16
    assert c_s[2] == c_b[2] + (P // 2) * rows * 18
    assert c_s[8] == c_b[8] + P // 2  # attention kernel calls


def test_split_backward_table():
    """Backward of the split schedule (DA_SCHEDULE_BALANCED_SPLIT_BWD): the split
    task table plus one GradKV per direct task (the half's for the split step),
    valid under the backward invariants, no idle slot; odd P = balanced backward."""
    for P in range(1, 33):
        s = S.build_balanced_split_backward_schedule(P)
        assert S.validate_backward(s) == [], P
        assert s.steps == S.build_balanced_split_schedule(P).steps
        assert s.idle_slot_count() == 0
        grads = sorted((m.step, m.from_, m.to) for m in s.messages
                       if m.kind == S.PayloadKind.GradKV)
        direct = sorted((t_, t.worker, t.kv_owner) for t_, st in enumerate(s.steps) for t in st
                        if t.kind == K.RemoteAttn and t.worker == t.query_owner)
        assert grads == direct
        if P % 2:
            assert s.flat() == S.build_balanced_backward_schedule(P).flat()
    # P = 4, t = 2: owners 3 / 4 take the high halves of kv 1 / 2 (KVHalf in, GradKV
    # of the half back); helpers 1 / 2 the low halves (Q bundle in, dq Partial back)
    s4 = S.build_balanced_split_backward_schedule(4)
    last = sorted((m.from_, m.to, m.kind.name) for m in s4.messages if m.step == 2)
    assert last == [(1, 3, "KVHalf"), (1, 3, "PartialResult"), (2, 4, "KVHalf"),
                    (2, 4, "PartialResult"), (3, 1, "GradKV"), (3, 1, "Q"), (4, 2, "GradKV"),
                    (4, 2, "Q")]


@pytest.mark.parametrize("P,n", [(2, 64), (4, 128), (6, 96), (8, 256), (4, 132), (3, 96)])
def test_oracle_split_backward_matches_ring(P, n):
    """The oracle's backward over the split table gives the reference ring
    backward's gradients (fp64, to summation order); counters: the split step
    moves half a KV chunk and half a GradKV per owner, plus a Q bundle and a dq
    Partial per helper."""
    q, k, v, do = O.make_inputs(4, P, n, 16, 1)
    q, k, v, do = q[0], k[0], v[0], do[0]
    out, lse, _ = O.run_forward(q, k, v, P, "balanced")
    dq_r, dk_r, dv_r, _ = O.run_backward(q, k, v, out, lse, do, P)
    dq_s, dk_s, dv_s, c_s = O.run_backward_sched(q, k, v, out, lse, do, P, "balanced_split")
    _, _, _, c_b = O.run_backward_sched(q, k, v, out, lse, do, P, "balanced")
    for a, b in ((dq_s, dq_r), (dk_s, dk_r), (dv_s, dv_r)):
        assert np.abs(a - b).max() < 1e-12
    rows, half = n // P, (P // 2 if P % 2 == 0 else 0)
    hi = rows - rows // 2
    assert c_s[0] == c_b[0] - half * 2 * rows * 16 + half * 2 * hi * 16   # KV / KVHalf
    assert c_s[3] == c_b[3] - half * 2 * rows * 16 + half * 2 * hi * 16   # GradKV halves
    assert c_s[1] == c_b[1] + half * rows * (2 * 16 + 2)                  # Q bundles
    assert c_s[8] == c_b[8] + half                                         # kernel calls
