"""The per-rank runtime's message protocol (csrc/rank_runtime.cu), on CPU.

Every rank derives its sends and receives from the same schedule table, one
pass = a fixed global sequence of phases (operands(t), results(t)). For the
NCCL transport each phase is one ncclGroupStart/Send/Recv/GroupEnd, so the
protocol is deadlock-free and correct exactly when, in every phase, the keys
rank a sends to rank b are the keys b receives from a, in the same order; the
IPC transport's per-pair ready/done counters rely on the same pairing. This
checks that property for every built-in schedule up to P = 16, through the
library's own program builder (da_rank_protocol), without a device.
"""
import ctypes as C
from collections import defaultdict

import pytest

from paper_2310_03294_b200 import _lib
from paper_2310_03294_b200.errors import check

FWD = {"ring": 0, "balanced": 1, "balanced_split": 4}
BWD = {"ring": 2, "balanced": 3, "balanced_split": 5}
KEYS = ["k", "v", "q", "part", "k_hi", "v_hi", "d_out", "lse", "d_vec", "gk0", "gv0", "gk1",
        "gv1", "gq0", "gq1", "gk_half", "gv_half"]


def protocol(world, rank, fwd, bwd):
    lib = _lib.lib()
    n = C.c_int64(0)
    check(lib.da_rank_protocol(world, rank, FWD[fwd], BWD[bwd], None, 0, C.byref(n)))
    buf = (C.c_int32 * max(1, 5 * n.value))()
    check(lib.da_rank_protocol(world, rank, FWD[fwd], BWD[bwd], buf, n.value, C.byref(n)))
    return [tuple(buf[5 * i:5 * i + 5]) for i in range(n.value)]


@pytest.mark.parametrize("fwd,bwd", [("ring", "ring"), ("balanced", "balanced"),
                                     ("balanced_split", "ring"), ("balanced_split", "balanced"),
                                     ("balanced_split", "balanced_split")])
@pytest.mark.parametrize("world", list(range(1, 17)))
def test_every_send_meets_its_receive_in_the_same_phase(world, fwd, bwd):
    sends = defaultdict(list)  # (pass, phase, src, dst) -> keys in issue order
    recvs = defaultdict(list)
    for r in range(world):
        for pas, phase, direction, peer, key in protocol(world, r, fwd, bwd):
            assert 0 <= peer < world and peer != r
            (sends if direction == 0 else recvs)[(pas, phase, r, peer) if direction == 0
                                                 else (pas, phase, peer, r)].append(key)
    assert set(sends) == set(recvs)
    for k in sends:
        assert sends[k] == recvs[k], (k, [KEYS[x] for x in sends[k]], [KEYS[x] for x in recvs[k]])


def test_message_volume_matches_the_schedule():
    """balanced P=8 forward: 22 KV messages (k + v each), 6 Q, 6 partials
    (SURVEY Appendix A); ring P=8 backward: 28 KV refetches + 28 GradKV."""
    per = defaultdict(int)
    for r in range(8):
        for pas, _, direction, _, key in protocol(8, r, "balanced", "ring"):
            if direction == 0:
                per[(pas, KEYS[key])] += 1
    assert per[(0, "k")] == per[(0, "v")] == 22
    assert per[(0, "q")] == 6 and per[(0, "part")] == 6
    assert per[(1, "k")] == 28
    assert per[(1, "gk0")] + per[(1, "gk1")] == 28


def test_protocol_rejects_bad_arguments():
    from paper_2310_03294_b200.errors import ConfigError
    n = C.c_int64(0)
    with pytest.raises(ConfigError):
        check(_lib.lib().da_rank_protocol(4, 4, 1, 2, None, 0, C.byref(n)))
    with pytest.raises(ConfigError):
        check(_lib.lib().da_rank_protocol(4, 0, 9, 2, None, 0, C.byref(n)))
