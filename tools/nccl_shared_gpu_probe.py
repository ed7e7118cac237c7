"""Probe: the native runtime's NCCL transport with 2+ ranks on ONE GPU.

NCCL refuses it ("Duplicate GPU detected", ncclInvalidUsage at
ncclCommInitRankConfig; gpurun_out/nccl_try.txt of the r2 probe), which is
why the multi-rank GPU tests use the IPC transport and the NCCL protocol is
verified on CPU (tests/test_rank_protocol.py). Kept to re-check on a box with
several GPUs:  python tools/nccl_shared_gpu_probe.py [world]
"""
import os, sys, tempfile
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch, torch.multiprocessing as mp
import test_gpu_rank_native as T
from oracle import oracle as O
if __name__ == "__main__":
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(T._worker, args=(world, T._port(), 256 * world, 2, "balanced", "balanced", td, None, "nccl"), nprocs=world, join=True)
        res = [np.load(os.path.join(td, f"r{r}.npz")) for r in range(world)]
    got = np.concatenate([r["out"] for r in res], axis=1)
    q, k, v, do = O.make_inputs(0, world, 256 * world, 128, 2, bf16=True)
    o_r, l_r, _ = O.run_forward(q[0], k[0], v[0], world, "balanced")
    print("NCCL world", world, "rel err O:", np.abs(got[0] - o_r).max() / np.abs(o_r).max())
