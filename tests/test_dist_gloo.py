"""Multi-process host logic of the distributed runtime (dist.py) on CPU.

world_size 2/3/4 over gloo with a TEST-ONLY compute backend built on the C
oracle: the per-worker op order of DistRuntime is the reference's, so the
results must be bit-identical to the oracle's single-process stepper (itself
bit-exact with the reference build). The production path swaps in the sm_100a
backend and NCCL; this test pins plan decoding, message routing, prefetch,
partial merges and GradKV folding.
"""
import math
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

from oracle import oracle as O


class OracleBackend:
    acc_dtype = torch.float64
    grad_dtype = torch.float64

    def __init__(self, d):
        self.scale = 1.0 / math.sqrt(d)

    def new_acc(self, h, rows, d, packed=None):
        if packed is None:
            packed = torch.empty(h * rows * (d + 2), dtype=torch.float64)
        o = packed[: h * rows * d].view(h, rows, d)
        m = packed[h * rows * d: h * rows * (d + 1)].view(h, rows)
        l = packed[h * rows * (d + 1):].view(h, rows)
        return (o, m, l), packed

    def update(self, q, k, v, acc_in, mask, out_acc):
        h, hk = q.shape[0], k.shape[0]
        for i in range(h):
            prev = None if acc_in is None else tuple(x[i].numpy() for x in acc_in)
            o, m, l = O.block_attn_update(q[i].numpy(), k[i * hk // h].numpy(),
                                          v[i * hk // h].numpy(), prev, mask, self.scale)
            out_acc[0][i].copy_(torch.from_numpy(o))
            out_acc[1][i].copy_(torch.from_numpy(m))
            out_acc[2][i].copy_(torch.from_numpy(l))
        return out_acc

    def merge(self, acc, part):
        for i in range(acc[0].shape[0]):
            o, m, l = O.rescale(tuple(x[i].numpy() for x in acc), tuple(x[i].numpy() for x in part))
            acc[0][i].copy_(torch.from_numpy(o))
            acc[1][i].copy_(torch.from_numpy(m))
            acc[2][i].copy_(torch.from_numpy(l))
        return acc

    def finalize(self, acc):
        outs, lses = [], []
        for i in range(acc[0].shape[0]):
            o, lse = O.finalize(tuple(x[i].numpy() for x in acc))
            outs.append(torch.from_numpy(o))
            lses.append(torch.from_numpy(lse))
        return torch.stack(outs), torch.stack(lses)

    def bwd_aux(self, d_out, out):
        return torch.stack([torch.from_numpy(O.backward_aux(d_out[i].numpy(), out[i].numpy()))
                            for i in range(out.shape[0])])

    def grads(self, q, k, v, lse, d_out, d_vec, mask, dq, dk, dv, accumulate_kv):
        h, hk = q.shape[0], k.shape[0]
        if not accumulate_kv:
            dk.zero_()
            dv.zero_()
        for i in range(h):
            j = i * hk // h
            gq, gk, gv = O.block_attn_backward_with_d(q[i].numpy(), k[j].numpy(), v[j].numpy(),
                                                      d_vec[i].numpy(), lse[i].numpy(),
                                                      d_out[i].numpy(), mask, self.scale)
            dq[i] += torch.from_numpy(gq)
            dk[j] += torch.from_numpy(gk)
            dv[j] += torch.from_numpy(gv)

    def add_(self, dst, src):
        dst.add_(src)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, d, heads, schedule, bwd_schedule, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2310_03294_b200.dist import DistRuntime, Transport
        q, k, v, do = O.make_inputs(0, world, n, d, heads, bf16=True)
        rows = n // world
        sl = slice(rank * rows, (rank + 1) * rows)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a[:, sl]))  # noqa: E731
        rt = DistRuntime(rank, world, backend=OracleBackend(d), transport=Transport(),
                         device=torch.device("cpu"))
        out, lse = rt.forward(t(q), t(k), t(v), schedule)
        dq, dk, dv = rt.backward(t(do), bwd_schedule)
        np.savez(os.path.join(outdir, f"r{rank}.npz"), out=out.numpy(), lse=lse.numpy(),
                 dq=dq.numpy(), dk=dk.numpy(), dv=dv.numpy(),
                 held=rt.trace["max_remote_chunks_held"])
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("world,schedule,bwd", [(2, "balanced", "ring"), (3, "balanced", "balanced"),
                                                (4, "balanced", "balanced"), (4, "ring", "ring"),
                                                (5, "balanced", "balanced"),
                                                (2, "balanced_split", "ring"),
                                                (4, "balanced_split", "balanced")])
def test_dist_runtime_gloo_bit_exact(world, schedule, bwd):
    n, d, heads = 16 * world, 8, 2
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_worker, args=(world, _free_port(), n, d, heads, schedule, bwd, td), nprocs=world,
                 join=True)
        res = [np.load(os.path.join(td, f"r{r}.npz")) for r in range(world)]
    q, k, v, do = O.make_inputs(0, world, n, d, heads, bf16=True)
    for h in range(heads):
        out, lse, _ = O.run_forward(q[h], k[h], v[h], world, schedule)
        if bwd == "ring":  # the reference's own order
            dq, dk, dv, _ = O.run_backward(q[h], k[h], v[h], out, lse, do[h], world)
        else:
            dq, dk, dv, _ = O.run_backward_sched(q[h], k[h], v[h], out, lse, do[h], world, bwd)
        got = {f: np.concatenate([r[f][h] for r in res], 0) for f in ("out", "lse", "dq", "dk", "dv")}
        assert np.array_equal(got["out"], out)
        assert np.array_equal(got["lse"], lse)
        assert np.array_equal(got["dq"], dq)
        assert np.array_equal(got["dk"], dk)
        assert np.array_equal(got["dv"], dv)
    assert max(int(r["held"]) for r in res) <= 2  # residency bound with prefetch


def _trace_worker(rank, world, port, n, d, heads, heads_kv, schedule, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2310_03294_b200.dist import DistRuntime, Transport, trace_to_json
        q, k, v, do = O.make_inputs(1, world, n, d, heads, bf16=True)
        rows = n // world
        sl = slice(rank * rows, (rank + 1) * rows)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a[:, sl]))  # noqa: E731
        rt = DistRuntime(rank, world, backend=OracleBackend(d), transport=Transport(),
                         device=torch.device("cpu"))
        rt.forward(t(q), t(k[:heads_kv]), t(v[:heads_kv]), schedule, trace=True)
        rt.backward(t(do), schedule, trace=True)
        tf, tb = rt.forward_trace(), rt.backward_trace()
        if rank == 0:
            with open(os.path.join(outdir, "fwd.json"), "w") as fh:
                fh.write(trace_to_json(tf))
            with open(os.path.join(outdir, "bwd.json"), "w") as fh:
                fh.write(trace_to_json(tb))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("world,schedule,heads,heads_kv", [(4, "ring", 2, 2), (6, "balanced", 4, 2)])
def test_wall_clock_trace_schema_and_counters(world, schedule, heads, heads_kv):
    """wall-clock trace in the reference schema (runtime.cpp:752-782)
    with byte-exact counters; the measured forward KV volume equals the analyzer's
    seq_parallel_forward_kv_volume_nd (analyzer.cpp:39-44) exactly."""
    import json
    from fractions import Fraction
    from paper_2310_03294_b200 import schedule as S
    n, d = 8 * world, 8
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_trace_worker, args=(world, _free_port(), n, d, heads, heads_kv, schedule, td),
                 nprocs=world, join=True)
        tf = json.loads(open(os.path.join(td, "fwd.json")).read())
        tb = json.loads(open(os.path.join(td, "bwd.json")).read())
    for tr in (tf, tb):
        assert set(tr) >= {"workers", "messages", "counters", "attention_kernel_calls",
                           "max_remote_chunks_held", "makespan"}
        assert [w["worker"] for w in tr["workers"]] == list(range(1, world + 1))
        for w in tr["workers"]:
            for e in w["events"]:
                assert 0.0 <= e["t0"] <= e["t1"] <= tr["makespan"] + 1e-6
        for m in tr["messages"]:
            assert m["t_issue"] <= m["t_arrive"] + 0.5  # host clocks of one machine
        assert tr["attention_kernel_calls"] == world * (world + 1) // 2
    sched = S.build_ring_schedule(world) if schedule == "ring" else S.build_balanced_schedule(world)
    kinds = {0: "kv", 1: "q", 2: "partial", 3: "grad_kv"}
    want = sorted((kinds[int(m.kind)], m.from_, m.to) for m in sched.messages)
    assert sorted((m["kind"], m["from"], m["to"]) for m in tf["messages"]) == want
    c = tf["counters"]
    rows = n // world
    # scalars per the reference's payload sizes (runtime.cpp:50-59) times heads
    assert c["kv_scalars"] == c["kv_messages"] * 2 * rows * d * heads_kv
    assert c["q_scalars"] == c["q_messages"] * rows * d * heads
    assert c["partial_scalars"] == c["partial_messages"] * rows * (d + 2) * heads
    assert c["kv_bytes"] == 8 * c["kv_scalars"]  # float64 payloads in this CPU test
    if schedule == "ring":
        vol = Fraction(c["kv_scalars"], world * n * d * heads)
        assert vol == Fraction(world - 1, world) * Fraction(heads_kv, heads)
    gradkv = sum(1 for m in tb["messages"] if m["kind"] == "grad_kv")
    direct = sum(1 for st in sched.steps for t_ in st
                 if t_.kind == S.TaskKind.RemoteAttn and t_.worker == t_.query_owner)
    assert gradkv == direct == tb["counters"]["grad_messages"]
