"""Feasibility probe: CUDA IPC tensors + stream-memop signals between two
processes on one GPU (the single-GPU stand-in for NVLink peers)."""
import ctypes as C
import os
import socket
import sys
from pathlib import Path

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def worker(rank, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    from torch.multiprocessing.reductions import reduce_tensor
    from paper_2310_03294_b200 import _lib
    lib = _lib.lib()
    torch.cuda.set_device(0)
    t = torch.full((1 << 22,), float(rank + 1), device="cuda")
    flags = torch.zeros(64, dtype=torch.int32, device="cuda")
    mine = (reduce_tensor(t), reduce_tensor(flags))
    allr = [None, None]
    dist.all_gather_object(allr, mine)
    peer = 1 - rank
    (ft, at), (ff, af) = allr[peer]
    pt, pf = ft(*at), ff(*af)
    s = torch.cuda.Stream()
    if rank == 0:
        with torch.cuda.stream(s):
            torch.cuda._sleep(200_000_000)  # ~0.1 s of spinning before producing
            t.fill_(42.0)
            assert lib.da_stream_write_u32(C.c_void_p(s.cuda_stream), C.c_void_p(flags.data_ptr()), 1) == 0
    else:
        local = torch.empty_like(t)
        with torch.cuda.stream(s):
            assert lib.da_stream_wait_u32_geq(C.c_void_p(s.cuda_stream), C.c_void_p(pf.data_ptr()), 1) == 0
            local.copy_(pt, non_blocking=True)
        s.synchronize()
        ok = bool((local == 42.0).all().item())
        print("rank1 pulled producer data after signal:", ok, flush=True)
    torch.cuda.synchronize()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    sk = socket.socket(); sk.bind(("127.0.0.1", 0)); port = sk.getsockname()[1]; sk.close()
    mp.spawn(worker, args=(port,), nprocs=2, join=True)
