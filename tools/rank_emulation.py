"""Per-rank compute times of an N-GPU run, measured one rank at a time on ONE B200.

Each rank r of a world-W run is the native per-rank runtime (csrc/rank_runtime.cu,
``rank.RankRuntime``) with the "none" transport: the same schedule, the same
kernels at the same per-rank chunk sizes (rows = seq / W), the same merges,
folds and conversions, only the transfers are replaced by one local fill of each
receive slot. Run alone, rank r's fwd+bwd step time T_r is the compute on its
critical path with communication fully hidden, so max_r T_r is a lower bound of
the real W-GPU step (the analyzer's makespan with measured costs,
analyzer.cpp:20-64), and the ring/balanced ratio of max_r T_r is the
balanced-schedule speed-up the compute alone allows. It is a MEASUREMENT of
every rank's work on the production code path, but not of NVLink: exposed
communication needs the W-GPU run (bench.py --gpus W, nocomm leg).

    python tools/rank_emulation.py --config cfg3 --world 8 [--steps 2]
prints one JSON line.
"""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import CONFIGS, flops_fwd_bwd, peaks, ClockSampler  # noqa: E402
from paper_2310_03294_b200.rank import RankRuntime  # noqa: E402

D = 128
LEGS = (("ring+ring", "ring", "ring"), ("balanced+balanced", "balanced", "balanced"),
        ("balanced_split+balanced", "balanced_split", "balanced"),
        ("balanced_split+balanced_split", "balanced_split", "balanced_split"))


def rank_time(r, world, rows, heads, hkv, fwd, bwd, steps, warmup):
    torch.manual_seed(1234 + r)

    def rnd(h):
        return (torch.rand(h, rows, D, device="cuda") * 2 - 1).to(torch.bfloat16)

    q, k, v, do = rnd(heads), rnd(hkv), rnd(hkv), rnd(heads)
    rt = RankRuntime(r, world, transport="none")
    try:
        def step():
            rt.forward(q, k, v, fwd)
            rt.backward(do, bwd)

        for _ in range(warmup):
            step()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(steps):
            step()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / steps
    finally:
        rt.close()
        del q, k, v, do
        torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--world", type=int, default=8)
    ap.add_argument("--seq", type=int, default=0)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--legs", default="all", help="comma list of leg names, or all")
    a = ap.parse_args()
    seq, heads, hkv, idx = CONFIGS[a.config]
    seq = a.seq or seq
    W = a.world
    rows = seq // W
    fl = flops_fwd_bwd(seq, heads)
    peak, peak_sus, src = peaks()
    legs = [l for l in LEGS if a.legs == "all" or l[0] in a.legs.split(",")]
    out = {"tool": "tools/rank_emulation.py", "config": a.config, "baseline_index": idx,
           "seq": seq, "heads": heads, "heads_kv": hkv, "world": W, "rows_per_rank": rows,
           "steps": a.steps, "warmup": a.warmup, "legs": {}}
    with ClockSampler(0) as clk:
        clk.timed(True)
        for name, f, b in legs:
            if f == "balanced_split" and W % 2:
                continue
            t = [rank_time(r, W, rows, heads, hkv, f, b, a.steps, a.warmup) for r in range(W)]
            mx = max(t)
            out["legs"][name] = {
                "rank_ms": t, "max_ms": mx, "mean_ms": sum(t) / W,
                "imbalance": mx / (sum(t) / W),
                "tflops_per_gpu_at_max": fl / W / (mx * 1e-3) / 1e12,
                "frac_of_burst_peak": fl / W / (mx * 1e-3) / 1e12 / peak,
                "tokens_per_s_at_max": seq / (mx * 1e-3)}
        clk.timed(False)
    ring = out["legs"].get("ring+ring", {}).get("max_ms")
    for name, leg in out["legs"].items():
        leg["speedup_vs_ring"] = ring / leg["max_ms"] if ring else None
    out["peak_tflops"], out["peak_source"] = peak, src
    out["clocks"] = clk.summary()
    out["reading"] = ("max_ms = slowest rank's fwd+bwd with transfers replaced by local fills: "
                      "the W-GPU step's compute critical path (lower bound of the real step); "
                      "NVLink exposure is not included")
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
