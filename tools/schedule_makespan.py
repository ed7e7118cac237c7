"""Schedule makespans from MEASURED chunk-kernel times on one B200 (projection).

Times each task kind of the sequence-parallel schedules at the real per-GPU
chunk size (seq N over P GPUs -> c = N/P rows, 32 heads, d=128) with CUDA
events: the causal diagonal chunk, a full chunk pair, a half pair (split
step), the partial merge, and the backward pair kernels. The makespan of a
schedule is then sum over steps of max over workers (primary task + the
owner's merges), i.e. the compute critical path with communication fully
overlapped — the quantity the reference's virtual-time analyzer computes with
unit costs (analyzer.cpp), here with measured costs. Prints one JSON line.

    python tools/schedule_makespan.py [N] [P ...]
"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2310_03294_b200 import flashcore as F  # noqa: E402
from paper_2310_03294_b200 import schedule as S  # noqa: E402

H, D = 32, 128
HKV = H  # set by argv: python tools/schedule_makespan.py N [P ...] [--kv HKV]


def timed(fn, iters=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def task_times(c):
    dev = "cuda"
    rnd = lambda *sh: (torch.rand(*sh, device=dev) * 2 - 1).to(torch.bfloat16)  # noqa: E731
    q, do = rnd(H, c, D), rnd(H, c, D)
    k, v = rnd(HKV, c, D), rnd(HKV, c, D)
    kh, vh = k[:, : c // 2].contiguous(), v[:, : c // 2].contiguous()
    acc = F.block_attn_update(q, k, v, None, F.MaskMode.Diagonal)
    part = F.block_attn_update(q, k, v, None, F.MaskMode.Full)
    out = F.finalize(acc)
    dvec = F.backward_aux(do, out.o)
    g = F.ChunkGrads(torch.zeros(H, c, D, device=dev), torch.zeros(HKV, c, D, device=dev),
                     torch.zeros(HKV, c, D, device=dev))
    t = {
        "fwd_diag": timed(lambda: F.block_attn_update(q, k, v, acc, F.MaskMode.Diagonal, out=acc)),
        "fwd_full": timed(lambda: F.block_attn_update(q, k, v, acc, F.MaskMode.Full, out=acc)),
        "fwd_half": timed(lambda: F.block_attn_update(q, kh, vh, acc, F.MaskMode.Full, out=acc)),
        "merge": timed(lambda: F.rescale(acc, part, out=acc)),
        "finalize": timed(lambda: F.finalize(acc)),
        "bwd_diag": timed(lambda: F.block_attn_backward(q, k, v, out.o, out.lse, do,
                                                        F.MaskMode.Diagonal, d_vec=dvec, grads=g,
                                                        accumulate_kv=True)),
        "bwd_full": timed(lambda: F.block_attn_backward(q, k, v, out.o, out.lse, do,
                                                        F.MaskMode.Full, d_vec=dvec, grads=g,
                                                        accumulate_kv=True)),
    }
    return t


def makespan(s, t, fwd=True):
    pre = "fwd_" if fwd else "bwd_"
    total = 0.0
    for step in s.steps:
        per = {}
        for task in step:
            if task.kind == S.TaskKind.LocalAttn:
                per[task.worker] = per.get(task.worker, 0.0) + t[pre + "diag"]
            elif task.kind == S.TaskKind.RemoteAttn:
                key = "full" if task.kv_part == S.KVPart.Whole else "half"
                if not fwd:
                    key = "full"
                per[task.worker] = per.get(task.worker, 0.0) + t[pre + key]
            elif task.kind == S.TaskKind.RescaleMerge:
                per[task.worker] = per.get(task.worker, 0.0) + (t["merge"] if fwd else 0.0)
        total += max(per.values(), default=0.0)
    return total


def main():
    global HKV
    args = sys.argv[1:]
    if "--kv" in args:
        i = args.index("--kv")
        HKV = int(args[i + 1])
        args = args[:i] + args[i + 2:]
    n = int(args[0]) if args else 131072
    ps = [int(x) for x in args[1:]] or [2, 4, 8]
    res = {"seq": n, "heads": H, "heads_kv": HKV, "d": D, "note": "compute critical path from measured chunk "
           "kernels on one B200; communication assumed overlapped (projection, not a "
           "multi-GPU measurement)", "P": {}}
    for P in ps:
        c = n // P
        t = task_times(c)
        fr, fb, fs = (makespan(S.build_ring_schedule(P), t), makespan(S.build_balanced_schedule(P), t),
                      makespan(S.build_balanced_split_schedule(P), t))
        br = makespan(S.build_ring_backward_schedule(P), t, fwd=False)
        bb = makespan(S.build_balanced_backward_schedule(P), t, fwd=False)
        res["P"][P] = {"chunk_rows": c, "task_ms": t,
                       "fwd_ms": {"ring": fr, "balanced": fb, "balanced_split": fs},
                       "bwd_ms": {"ring": br, "balanced": bb},
                       "speedup_vs_ring": {"fwd_balanced": fr / fb, "fwd_split": fr / fs,
                                           "fwdbwd_balanced": (fr + br) / (fb + bb),
                                           "fwdbwd_split": (fr + br) / (fs + bb)},
                       "fwdbwd_tflops_per_gpu_split": 7.0 * n * n * D * H / P /
                       ((fs + bb) * 1e-3) / 1e12}
        print(json.dumps({str(P): res["P"][P]["speedup_vs_ring"]}), flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
