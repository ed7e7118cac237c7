"""The C++ per-rank runtime (csrc/rank_runtime.cu, da_rank_*) with one process
per rank on one GPU: copy-engine pulls from the other processes' memory
(CUDA IPC) ordered by device-side counters. Checked against the C oracle and
the forward bitwise against the single-process device executor."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

from oracle import oracle as O

pytestmark = pytest.mark.gpu
TOL, LSE_TOL = 2e-2, 1e-3


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, heads, fwd, bwd, outdir, heads_kv=None, transport="ipc",
            deterministic=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2310_03294_b200.rank import RankRuntime
        q, k, v, do = O.make_inputs(0, world, n, 128, heads, bf16=True)
        rows = n // world
        sl = slice(rank * rows, (rank + 1) * rows)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a[:, sl])).cuda().to(torch.bfloat16)  # noqa: E731
        rt = RankRuntime(rank, world, transport=transport, deterministic=deterministic)
        hk = heads_kv or heads
        qq, kk, vv, dd = t(q), t(k[:hk]), t(v[:hk]), t(do)
        first = None
        for _ in range(2):  # second pass: cached mappings, running counters
            out, lse, cf = rt.forward(qq, kk, vv, fwd)
            dq, dk, dv, cb = rt.backward(dd, bwd)
            torch.cuda.synchronize()
            if first is None:
                first = [x.clone() for x in (out, lse, dq, dk, dv)]
        same = all(torch.equal(a, b) for a, b in zip(first, (out, lse, dq, dk, dv)))
        np.savez(os.path.join(outdir, f"r{rank}.npz"), out=out.float().cpu().numpy(),
                 lse=lse.cpu().numpy(), dq=dq.cpu().numpy(), dk=dk.cpu().numpy(),
                 dv=dv.cpu().numpy(), cf=np.array(list(cf.__dict__.values())),
                 cb=np.array(list(cb.__dict__.values())), same=np.array(same))
        tdist.barrier()
        rt.close()
        tdist.barrier()
    finally:
        tdist.destroy_process_group()


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


@pytest.mark.parametrize("world,n,heads,fwd,bwd,heads_kv", [
    (2, 1024, 2, "balanced", "ring", None), (4, 2048, 1, "balanced", "balanced", None),
    (3, 768, 2, "ring", "balanced", None), (4, 1024, 2, "balanced_split", "ring", None),
    (1, 512, 2, "balanced", "ring", None), (2, 1002, 1, "balanced_split", "balanced", None),
    (4, 1024, 4, "balanced", "balanced", 2), (8, 2048, 2, "balanced_split", "balanced", None),
    (8, 2048, 4, "balanced", "ring", 1), (2, 1002, 1, "balanced_split", "balanced_split", None),
    (4, 1024, 2, "balanced_split", "balanced_split", None),
    (4, 1024, 4, "balanced_split", "balanced_split", 2),
    (8, 2048, 2, "balanced_split", "balanced_split", None),
    (3, 768, 2, "balanced", "balanced_split", None)])
def test_native_rank_runtime(cuda, world, n, heads, fwd, bwd, heads_kv):
    """Worlds 1-4 and 8 (the SCALE run's P), ring / balanced / split forward,
    ring / balanced / split backward, odd chunk rows (split halves 250 / 251),
    GQA (4 q / 2 kv and 4 q / 1 kv heads)."""
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_worker, args=(world, _port(), n, heads, fwd, bwd, td, heads_kv), nprocs=world,
                 join=True)
        res = [np.load(os.path.join(td, f"r{r}.npz")) for r in range(world)]
    got = {f: np.concatenate([r[f] for r in res], axis=1) for f in ("out", "lse", "dq", "dk", "dv")}
    q, k, v, do = O.make_inputs(0, world, n, 128, heads, bf16=True)
    hk = heads_kv or heads
    group = heads // hk
    dk_ref = np.zeros((hk, n, 128))
    dv_ref = np.zeros((hk, n, 128))
    for h in range(heads):
        j = h // group  # GQA parity: MHA with the group's K/V replicated
        o_r, l_r, c_f = O.run_forward(q[h], k[j], v[j], world, fwd)
        if bwd == "ring":
            dq_r, dk_r, dv_r, c_b = O.run_backward(q[h], k[j], v[j], o_r, l_r, do[h], world)
        else:
            dq_r, dk_r, dv_r, c_b = O.run_backward_sched(q[h], k[j], v[j], o_r, l_r, do[h], world,
                                                         bwd)
        assert _rel(got["out"][h], o_r) < TOL
        assert np.abs(got["lse"][h] - l_r).max() < LSE_TOL
        assert _rel(got["dq"][h], dq_r) < TOL
        dk_ref[j] += dk_r
        dv_ref[j] += dv_r
    assert _rel(got["dk"], dk_ref) < TOL and _rel(got["dv"], dv_ref) < TOL
    if heads_kv:
        return
    # per-rank counters summed = the reference's CommCounters (x heads for scalars)
    cf = sum(r["cf"] for r in res)
    cb = sum(r["cb"] for r in res)
    assert list(cf[:4]) == [x * heads for x in c_f[:4]] and list(cf[4:8]) == list(c_f[4:8])
    assert list(cb[:4]) == [x * heads for x in c_b[:4]] and list(cb[4:8]) == list(c_b[4:8])
    from paper_2310_03294_b200.runtime import make_parity_shards, run_forward
    shards = make_parity_shards(0, world, n, heads, 128)
    run_forward(shards, fwd)
    torch.cuda.synchronize()
    assert np.array_equal(got["out"], torch.cat([s.out for s in shards], 1).float().cpu().numpy())
    assert np.array_equal(got["lse"], torch.cat([s.lse for s in shards], 1).cpu().numpy())


@pytest.mark.parametrize("world,fwd,bwd", [(3, "balanced", "balanced"), (4, "balanced_split", "ring"),
                                           (4, "balanced_split", "balanced_split")])
def test_native_rank_runtime_deterministic_backward(cuda, world, fwd, bwd):
    """deterministic=True: the distributed backward repeats bit for bit (the
    reference's executors do, runtime.hpp:7-9) and still matches the oracle."""
    n, heads = 256 * world, 2
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_worker, args=(world, _port(), n, heads, fwd, bwd, td, None, "ipc", True),
                 nprocs=world, join=True)
        res = [np.load(os.path.join(td, f"r{r}.npz")) for r in range(world)]
    assert all(bool(r["same"]) for r in res)
    got = {f: np.concatenate([r[f] for r in res], axis=1) for f in ("dq", "dk", "dv")}
    q, k, v, do = O.make_inputs(0, world, n, 128, heads, bf16=True)
    for h in range(heads):
        o_r, l_r, _ = O.run_forward(q[h], k[h], v[h], world, fwd)
        g = (O.run_backward(q[h], k[h], v[h], o_r, l_r, do[h], world) if bwd == "ring" else
             O.run_backward_sched(q[h], k[h], v[h], o_r, l_r, do[h], world, bwd))
        for name, ref in zip(("dq", "dk", "dv"), g[:3]):
            assert _rel(got[name][h], ref) < TOL, name


def test_native_rank_runtime_nccl_transport_world1(cuda):
    """The NCCL transport at one rank (the only NCCL world one GPU allows:
    NCCL refuses two ranks on one device): communicator bootstrap through the
    allgather, the pass with an empty protocol, results = the oracle. The
    multi-rank message protocol itself is checked on CPU for P <= 16
    (tests/test_rank_protocol.py)."""
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_worker, args=(1, _port(), 512, 2, "balanced", "ring", td, None, "nccl"),
                 nprocs=1, join=True)
        r = np.load(os.path.join(td, "r0.npz"))
    q, k, v, do = O.make_inputs(0, 1, 512, 128, 2, bf16=True)
    for h in range(2):
        o_r, l_r, _ = O.run_forward(q[h], k[h], v[h], 1, "balanced")
        assert _rel(r["out"][h], o_r) < TOL


def test_native_rank_runtime_nocomm_arm_runs(cuda):
    """transport="none": the same kernels on local buffers (no transfers), the
    denominator of the exposed-communication measurement; it completes at
    world 3 without waiting on any peer."""
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_worker, args=(3, _port(), 768, 2, "balanced", "balanced", td, None, "none"),
                 nprocs=3, join=True)
        res = [np.load(os.path.join(td, f"r{r}.npz")) for r in range(3)]
    # rank 0 (worker 1) only ever uses its own chunk: still exact
    q, k, v, do = O.make_inputs(0, 3, 768, 128, 2, bf16=True)
    o_r, _, _ = O.run_forward(q[0], k[0], v[0], 3, "balanced")
    assert _rel(res[0]["out"][0], o_r[:256]) < TOL


def _trace_worker(rank, world, port, outdir, fwd, bwd):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import json
        from paper_2310_03294_b200.rank import RankRuntime
        n, heads = 512 * world, 2
        q, k, v, do = O.make_inputs(0, world, n, 128, heads, bf16=True)
        rows = n // world
        sl = slice(rank * rows, (rank + 1) * rows)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a[:, sl])).cuda().to(torch.bfloat16)  # noqa: E731
        rt = RankRuntime(rank, world, transport="ipc")
        _, _, cf = rt.forward(t(q), t(k), t(v), fwd, trace=True)
        _, _, _, cb = rt.backward(t(do), bwd, trace=True)
        tf = rt.gather_trace("forward", cf, cf.max_remote_chunks_held)
        tb = rt.gather_trace("backward", cb, cb.max_remote_chunks_held)
        if rank == 0:
            with open(os.path.join(outdir, "trace.json"), "w") as f:
                json.dump({"fwd": tf, "bwd": tb}, f)
        tdist.barrier()
        rt.close()
        tdist.barrier()
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("world,fwd,bwd", [(4, "balanced", "ring"), (4, "balanced_split", "balanced"),
                                           (4, "balanced_split", "balanced_split")])
def test_native_runtime_wall_clock_trace(cuda, world, fwd, bwd):
    """SURVEY §8(f)4 on the product path: the native runtime's CUDA-event trace
    in the reference's ExecutionTrace schema (runtime.cpp:752-782): one event
    per attention task and merge, one message per schedule message with the
    schedule's (kind, from, to), arrivals after issues, counters summed."""
    import json

    from paper_2310_03294_b200 import schedule as S
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_trace_worker, args=(world, _port(), td, fwd, bwd), nprocs=world, join=True)
        tr = json.load(open(os.path.join(td, "trace.json")))
    builders = {"balanced": S.build_balanced_schedule, "ring": S.build_ring_schedule,
                "balanced_split": S.build_balanced_split_schedule}
    kinds = {0: "kv", 1: "q", 2: "partial", 3: "grad_kv", 4: "kv_half"}
    sched = builders[fwd](world)
    tf, tb = tr["fwd"], tr["bwd"]
    for t_ in (tf, tb):
        assert set(t_) >= {"workers", "messages", "counters", "attention_kernel_calls",
                           "max_remote_chunks_held", "makespan"}
        assert [w["worker"] for w in t_["workers"]] == list(range(1, world + 1))
        for w in t_["workers"]:
            for e in w["events"]:
                assert 0.0 <= e["t0"] <= e["t1"] <= t_["makespan"] + 1e-3
        for m in t_["messages"]:
            # issue and arrival come from different ranks' clocks (origins recorded
            # after one barrier); the ranks here share ONE GPU, whose contexts
            # time-slice, so the origins can be milliseconds apart
            assert m["t_issue"] >= 0.0 and 0.0 <= m["t_arrive"] <= t_["makespan"] + 50.0
    assert sorted((m["kind"], m["from"], m["to"]) for m in tf["messages"]) == \
        sorted((kinds[int(m.kind)], m.from_, m.to) for m in sched.messages)
    assert tf["attention_kernel_calls"] == sched.attention_task_count()
    merges = sum(1 for st in sched.steps for x in st if x.kind == S.TaskKind.RescaleMerge)
    assert sum(1 for w in tf["workers"] for e in w["events"]
               if e["task"].startswith("rescale_merge")) == merges
    bsched = {"ring": S.build_ring_backward_schedule,
              "balanced": S.build_balanced_backward_schedule,
              "balanced_split": S.build_balanced_split_backward_schedule}[bwd](world)
    assert sorted((m["kind"], m["from"], m["to"]) for m in tb["messages"]) == \
        sorted((kinds[int(m.kind)], m.from_, m.to) for m in bsched.messages)
    assert tf["counters"]["kv_messages"] == sum(1 for m in sched.messages if int(m.kind) in (0, 4))


def _table_worker(rank, world, port, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import dataclasses
        torch.cuda.set_device(0)
        from paper_2310_03294_b200 import schedule as S
        from paper_2310_03294_b200.rank import RankRuntime
        n, heads = 256 * world, 2
        q, k, v, do = O.make_inputs(0, world, n, 128, heads, bf16=True)
        rows = n // world
        sl = slice(rank * rows, (rank + 1) * rows)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a[:, sl])).cuda().to(torch.bfloat16)  # noqa: E731
        custom = S.build_ring_schedule(world)  # a valid table none of the built-ins: steps 1, 2 swapped
        custom.steps[1], custom.steps[2] = custom.steps[2], custom.steps[1]
        custom.messages = sorted((dataclasses.replace(m, step=3 - m.step) if m.step in (1, 2) else m
                                  for m in custom.messages), key=lambda m: (m.step, m.from_))
        rt = RankRuntime(rank, world, transport="ipc")
        out, lse, _ = rt.forward(t(q), t(k), t(v), custom)
        dq, dk, dv, _ = rt.backward(t(do), S.build_ring_backward_schedule(world))
        torch.cuda.synchronize()
        np.savez(os.path.join(outdir, f"r{rank}.npz"), out=out.float().cpu().numpy(),
                 lse=lse.cpu().numpy(), dq=dq.cpu().numpy())
        tdist.barrier()
        rt.close()
        tdist.barrier()
    finally:
        tdist.destroy_process_group()


def test_native_runtime_takes_schedule_tables(cuda):
    """da_rank_forward_table / da_rank_backward_table: any validated table (here
    ring with steps 1 and 2 swapped, and the ring backward as an object) runs
    on the per-rank runtime and matches the oracle's ring results."""
    world = 4
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_table_worker, args=(world, _port(), td), nprocs=world, join=True)
        res = [np.load(os.path.join(td, f"r{r}.npz")) for r in range(world)]
    got = {f: np.concatenate([r[f] for r in res], axis=1) for f in ("out", "lse", "dq")}
    q, k, v, do = O.make_inputs(0, world, 256 * world, 128, 2, bf16=True)
    for h in range(2):
        o_r, l_r, _ = O.run_forward(q[h], k[h], v[h], world, "ring")
        dq_r = O.run_backward(q[h], k[h], v[h], o_r, l_r, do[h], world)[0]
        assert _rel(got["out"][h], o_r) < TOL and np.abs(got["lse"][h] - l_r).max() < LSE_TOL
        assert _rel(got["dq"][h], dq_r) < TOL
