"""Runtime contract checks mirrored from /root/reference/proj/tests/test_runtime.cpp
that need no GPU: ragged splits, and the overlap/residency properties of the
per-rank runtime (dist.py) under gloo with the oracle compute backend."""
import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2310_03294_b200.errors import ConfigError
from paper_2310_03294_b200.runtime import Rng, make_shards

from test_dist_gloo import OracleBackend, _free_port


def test_make_shards_rejects_ragged_splits():
    # test_runtime.cpp:57-69
    with pytest.raises(ConfigError):
        make_shards(3, 32, 8, Rng(3))
    with pytest.raises(ConfigError):
        make_shards(0, 32, 8, Rng(3))
    with pytest.raises(ConfigError):
        make_shards(2, 0, 8, Rng(3))


def _overlap_worker(rank, world, port, n, d, heads, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2310_03294_b200.dist import DistRuntime, Transport
        q, k, v, do = O.make_inputs(2, world, n, d, heads, bf16=True)
        rows = n // world
        sl = slice(rank * rows, (rank + 1) * rows)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a[:, sl]))  # noqa: E731
        res = {}
        for overlap in (True, False):
            rt = DistRuntime(rank, world, backend=OracleBackend(d), transport=Transport(),
                             device=torch.device("cpu"))
            out, lse = rt.forward(t(q), t(k), t(v), "balanced", overlap=overlap)
            dq, dk, dv = rt.backward(t(do), "ring", overlap=overlap)
            res[overlap] = [x.numpy().copy() for x in (out, lse, dq, dk, dv)] + \
                [rt.trace["max_remote_chunks_held"]]
        np.savez(os.path.join(outdir, f"r{rank}.npz"),
                 **{f"{o}_{i}": a for o, v_ in res.items() for i, a in enumerate(v_)})
    finally:
        tdist.destroy_process_group()


def test_overlap_changes_timing_only_and_residency():
    """test_runtime.cpp:130-164: prefetch changes no bit of the results; one
    remote chunk is held without prefetch, at most two with it."""
    world, n, d, heads = 4, 64, 8, 1
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_overlap_worker, args=(world, _free_port(), n, d, heads, td), nprocs=world,
                 join=True)
        res = [np.load(os.path.join(td, f"r{r}.npz")) for r in range(world)]
    for r in res:
        for i in range(5):
            assert np.array_equal(r[f"True_{i}"], r[f"False_{i}"])
    assert max(int(r["False_5"]) for r in res) == 1
    assert max(int(r["True_5"]) for r in res) == 2
