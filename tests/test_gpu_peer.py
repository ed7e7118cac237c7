"""The sequence-parallel runtime with REAL kernels and one process per rank
(dist.DistRuntime + CudaBackend + PeerTransport), on one GPU.

Each rank is a separate process; K/V, Q, partials and gradients move by
copy-engine pulls from the other processes' device memory (CUDA IPC
mappings) ordered by device-side counters (csrc/peer.cu) — the same code
that runs over NVLink between GPUs, here with all ranks sharing cuda:0.
Checked against the C oracle (bit-exact with the reference build) on the
same seeded inputs, and the forward bitwise against the single-process
device executor (runtime.cu) running the same schedule.
"""
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


def _worker(rank, world, port, n, heads, fwd, bwd, outdir, heads_kv=None):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        from paper_2310_03294_b200.dist import CudaBackend, DistRuntime, PeerTransport
        q, k, v, do = O.make_inputs(0, world, n, 128, heads, bf16=True)
        rows = n // world
        sl = slice(rank * rows, (rank + 1) * rows)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a[:, sl])).to(dev).to(torch.bfloat16)  # noqa: E731
        rt = DistRuntime(rank, world, backend=CudaBackend(dev), transport=PeerTransport(device=dev),
                         device=dev)
        hk = heads_kv or heads
        for _ in range(2):  # the second pass reuses the published buffers and counters
            out, lse = rt.forward(t(q), t(k[:hk]), t(v[:hk]), fwd)
            dq, dk, dv = rt.backward(t(do), bwd)
        torch.cuda.synchronize()
        np.savez(os.path.join(outdir, f"r{rank}.npz"), out=out.float().cpu().numpy(),
                 lse=lse.cpu().numpy(), dq=dq.cpu().numpy(), dk=dk.cpu().numpy(),
                 dv=dv.cpu().numpy())
        tdist.barrier()
    finally:
        tdist.destroy_process_group()


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


@pytest.mark.parametrize("world,n,heads,fwd,bwd,heads_kv", [
    (2, 1024, 2, "balanced", "ring", None), (4, 2048, 1, "balanced", "balanced", None),
    (3, 768, 2, "ring", "balanced", None), (4, 1024, 2, "balanced_split", "ring", None),
    (2, 8192, 2, "balanced", "balanced", None), (4, 1024, 4, "balanced", "balanced", 2)])
def test_peer_runtime_one_process_per_rank(cuda, world, n, heads, fwd, bwd, heads_kv):
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_worker, args=(world, _port(), n, heads, fwd, bwd, td, heads_kv), nprocs=world,
                 join=True)
        res = [np.load(os.path.join(td, f"r{r}.npz")) for r in range(world)]
    got = {f: np.concatenate([r[f] for r in res], axis=1) for f in ("out", "lse", "dq", "dk", "dv")}
    q, k, v, do = O.make_inputs(0, world, n, 128, heads, bf16=True)
    hk_n = heads_kv or heads
    group = heads // hk_n
    dk_ref = np.zeros((hk_n, n, 128))
    dv_ref = np.zeros((hk_n, n, 128))
    for h in range(heads):
        j = h // group  # GQA parity: MHA with the group's K/V replicated
        o_r, l_r, _ = O.run_forward(q[h], k[j], v[j], world, fwd)
        if bwd == "ring":
            dq_r, dk_r, dv_r, _ = O.run_backward(q[h], k[j], v[j], o_r, l_r, do[h], world)
        else:
            dq_r, dk_r, dv_r, _ = O.run_backward_sched(q[h], k[j], v[j], o_r, l_r, do[h], world, bwd)
        assert _rel(got["out"][h], o_r) < TOL
        assert np.abs(got["lse"][h] - l_r).max() < LSE_TOL
        assert _rel(got["dq"][h], dq_r) < TOL
        dk_ref[j] += dk_r
        dv_ref[j] += dv_r
    assert _rel(got["dk"], dk_ref) < TOL
    assert _rel(got["dv"], dv_ref) < TOL
    if heads_kv:
        return
    # forward bitwise equal to the single-process device executor (same kernels, same order)
    from paper_2310_03294_b200.runtime import make_parity_shards, run_forward
    shards = make_parity_shards(0, world, n, heads, 128)
    run_forward(shards, fwd)
    torch.cuda.synchronize()
    out_dev = torch.cat([s.out for s in shards], 1).float().cpu().numpy()
    lse_dev = torch.cat([s.lse for s in shards], 1).cpu().numpy()
    assert np.array_equal(got["out"], out_dev)
    assert np.array_equal(got["lse"], lse_dev)
