"""Benchmark: causal attention forward+backward (DistFlashAttn hot path) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N=1 workload = BASELINE.json configs[1]: Llama-7B attention layer (32 heads,
d=128), causal fwd+bwd at seq 32K on one B200, synthetic U[-1,1) bf16 inputs
generated on the device. One step = one forward (block_attn_update with the
fused finalize) + backward_aux + block_attn_backward over the full sequence.
N>1 runs the sequence-parallel runtime (paper_2310_03294_b200/dist.py): the
sequence is split into N contiguous chunks, one per rank (32K tokens per GPU),
balanced forward + balanced backward schedules, messages pulled by the copy
engines from the peers' HBM (--transport peer, default) or NCCL send/recv.

Metric: whole-job attention fwd+bwd TFLOP/s (algorithmic causal FLOPs
7·N²·d·H per step, no recompute counted), with tokens/s and per-GPU TFLOP/s
beside it. Inputs (4 × 268 MB at 32K) exceed the 126 MB L2, so no flush is
needed between steps.

--impl reference times the reference's own CPU implementation (the
unmodified sources compiled into oracle/_ref/ref_driver) on a bounded sample
of the same workload, with every host core.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

H, D, SEQ = 32, 128, 32768
PEAKS_FILE = ROOT / "MEASURED_PEAKS.json"
FALLBACK_PEAK = 1590.0  # B200_PROFILING.md fallback (TFLOP/s, burst)


def flops_fwd_bwd(n: int, heads: int, d: int = D) -> float:
    return 7.0 * n * n * d * heads


def peaks():
    try:
        p = json.loads(PEAKS_FILE.read_text())
        return float(p["bf16_tflops"]), float(p.get("bf16_tflops_sustained", p["bf16_tflops"])), "measured"
    except Exception:
        return FALLBACK_PEAK, 1400.0, "fallback"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + clock-event reasons sampled every ~5 ms by NVML in a thread
    (nvidia-smi as a fallback). `timed(True/False)` brackets the timed region:
    the summary's median covers those samples only (all samples if none)."""
    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int = 0, period_s: float = 0.005):
        self.index = index
        self.period = period_s
        self.proc = None
        self.thread = None
        self.samples = []  # (in_timed_region, sm_mhz, max_mhz, reasons)
        self._timed = False
        self._stop = False

    def _nvml_handle(self):
        import pynvml as N
        N.nvmlInit()
        try:  # match the CUDA device by PCI address (CUDA and NVML orders may differ)
            import torch
            p = torch.cuda.get_device_properties(self.index)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            return N, N.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return N, N.nvmlDeviceGetHandleByIndex(self.index)

    def _run_nvml(self, N, h):
        bits = {"hw_slowdown": N.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": N.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": N.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": N.nvmlClocksEventReasonSwPowerCap}
        mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
        while not self._stop:
            try:
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((self._timed, float(sm), float(mx),
                                     {n for n, b in bits.items() if r & b}))
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        try:
            import threading
            N, h = self._nvml_handle()
            self.thread = threading.Thread(target=self._run_nvml, args=(N, h), daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.thread = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def timed(self, on: bool):
        self._timed = on

    def __exit__(self, *a):
        self._stop = True
        if self.thread is not None:
            self.thread.join(timeout=2)
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out, _ = self.proc.communicate()
            for ln in out.splitlines():
                parts = [p.strip() for p in ln.split(",")]
                try:
                    self.samples.append((False, float(parts[0]), float(parts[1]),
                                         {n for n, v in zip(self.NAMES, parts[2:])
                                          if v.lower() == "active"}))
                except (ValueError, IndexError):
                    continue

    def summary(self):
        inside = [x for x in self.samples if x[0]] or self.samples
        sm = [x[1] for x in inside]
        mx = max((x[2] for x in self.samples), default=0.0)
        reasons = set().union(*(x[3] for x in inside)) if inside else set()
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvml" if self.thread is not None else "nvidia-smi"}


# ----------------------------------------------------------------------------- reference arm
def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def reference_sample(threads: int, n: int = 8192, workers: int = 8, heads: int = 1,
                     schedule: str = "balanced") -> dict:
    """The reference CPU path (oracle/_ref/ref_driver: unmodified sources) on a
    bounded sample of the workload: `heads` heads of seq n, P=workers threads
    per head (concurrent executor), balanced forward + ring backward."""
    from oracle import oracle as O
    if not O.ref_available():
        raise RuntimeError("oracle/_ref/ref_driver missing (build with `make -C oracle ref`)")
    r = O.ref_time(n, workers, heads, D, schedule, threads)
    return {"seconds": r["seconds"], "tflops": r["tflops"], "threads": r["threads"],
            "sample": f"{heads} head(s) x seq {n} x d {D}, P={workers} concurrent workers "
                      f"({schedule} fwd + ring bwd), bf16-rounded fp64 inputs"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = cpu_threads()
    vals = []
    for i in range(args.warmup + args.steps):
        s = reference_sample(threads)
        if i >= args.warmup:
            vals.append(s)
    v = statistics.median(x["tflops"] for x in vals)
    secs = statistics.median(x["seconds"] for x in vals)
    line = {
        "impl": "reference", "metric": "attn fwd+bwd TFLOP/s", "value": v, "unit": "TFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": secs * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "llama7b-attn causal fwd+bwd (reference CPU, bounded sample)",
                   "heads": H, "d": D, "seq_len": SEQ},
        "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": vals[0]["threads"],
                         "kind": "reference", "sample": vals[0]["sample"]},
        "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- our arm, N=1
def _profile_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu capture."""
    f = ROOT / "profiles" / "roofline_traffic.json"
    try:
        return json.loads(f.read_text())
    except Exception:
        return {}


def run_single(args):
    import torch
    from paper_2310_03294_b200 import flashcore as F

    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    n = args.seq
    heads = args.heads
    stream = torch.cuda.current_stream()

    def rnd(*shape):
        return (torch.rand(*shape, device=dev) * 2 - 1).to(torch.bfloat16)

    torch.manual_seed(0)
    q, k, v, d_out = rnd(heads, n, D), rnd(heads, n, D), rnd(heads, n, D), rnd(heads, n, D)
    grads = F.ChunkGrads(torch.zeros(heads, n, D, device=dev), torch.empty(heads, n, D, device=dev),
                         torch.empty(heads, n, D, device=dev))

    ev = {k_: [] for k_ in ("fwd", "aux", "bwd")}
    dflag = torch.zeros(1, dtype=torch.int32, device=dev)  # checked once after the timed loop

    def step(record=False):
        if record:
            e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            e[0].record(stream)
        out = F.block_attn_update_final(q, k, v, None, F.MaskMode.Diagonal, degenerate_flag=dflag)
        if record:
            e[1].record(stream)
        dvec = F.backward_aux(d_out, out.o)
        if record:
            e[2].record(stream)
        grads.dq.zero_()
        F.block_attn_backward(q, k, v, out.o, out.lse, d_out, F.MaskMode.Diagonal, d_vec=dvec,
                              grads=grads)
        if record:
            e[3].record(stream)
            ev["fwd"].append((e[0], e[1]))
            ev["aux"].append((e[1], e[2]))
            ev["bwd"].append((e[2], e[3]))
        return out

    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:  # started before the warm-up
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        clk.timed(True)
        start.record(stream)
        for _ in range(args.steps):
            step(record=True)
        end.record(stream)
        torch.cuda.synchronize()
        clk.timed(False)
    ms = start.elapsed_time(end) / args.steps
    F.check_degenerate(dflag)
    fl = flops_fwd_bwd(n, heads)
    tflops = fl / (ms * 1e-3) / 1e12
    t_fwd = statistics.mean(a.elapsed_time(b) for a, b in ev["fwd"])
    t_bwd = statistics.mean(a.elapsed_time(b) for a, b in ev["bwd"])
    t_aux = statistics.mean(a.elapsed_time(b) for a, b in ev["aux"])

    # ---- e2e: host (pinned) inputs -> device -> fwd+bwd -> bf16 grads -> host,
    # through the public host-buffer API (copies overlapped per head group)
    from paper_2310_03294_b200.pipeline import HostAttention
    hq, hk, hv, hdo = (t.cpu().pin_memory() for t in (q, k, v, d_out))
    hdq, hdk, hdv = (torch.empty(heads, n, D, dtype=torch.bfloat16).pin_memory() for _ in range(3))
    del grads
    ha = HostAttention(heads, n, D, heads_per_group=args.heads_per_group, device=dev)

    def e2e_step():
        ha(hq, hk, hv, hdo, hdq, hdk, hdv, sync=False)

    for _ in range(max(3, args.warmup)):
        e2e_step()
    ha.join(stream)
    torch.cuda.synchronize()
    e_steps = max(2, args.steps)  # the same K as the device-timed steps
    s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s2.record(stream)
    for _ in range(e_steps):
        e2e_step()
    ha.join(stream)  # consecutive steps overlap (prefetch); the end event sees all of them
    e2.record(stream)
    torch.cuda.synchronize()
    ha.check(stream)
    ms_e2e = s2.elapsed_time(e2) / e_steps
    h2d = ha.bytes_in
    d2h = ha.bytes_out

    peak, peak_sus, src = peaks()
    # dominant kernel: the backward chunk kernel
    dom = "bwd" if t_bwd >= t_fwd else "fwd"
    t_dom = t_bwd if dom == "bwd" else t_fwd
    dom_flops = (5.0 if dom == "bwd" else 2.0) * n * n * D * heads
    achieved = dom_flops / (t_dom * 1e-3) / 1e12
    traffic = _profile_traffic().get(f"{dom}_dram_bytes_per_launch")
    line = {
        "metric": "attn fwd+bwd TFLOP/s", "value": tflops, "unit": "TFLOP/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": "llama7b-attn causal fwd+bwd, 32 heads, d=128, seq 32K, 1 B200 "
                               "(BASELINE configs[1])",
                   "heads": heads, "d": D, "seq_len": n, "mask": "causal", "workers": 1,
                   "l2": "inputs (4 x %d MB) exceed L2; no flush" % (heads * n * D * 2 >> 20)},
        "tokens_per_s": n / (ms * 1e-3),
        "tflops_per_gpu": tflops,
        "frac_of_peak": tflops / peak,
        "kernel_ms": {"fwd": t_fwd, "bwd_preprocess": t_aux, "bwd": t_bwd},
        "kernel_tflops": {"fwd": 2.0 * n * n * D * heads / (t_fwd * 1e-3) / 1e12,
                          "bwd": 5.0 * n * n * D * heads / (t_bwd * 1e-3) / 1e12},
        "roofline": {"bound": "tensor", "kernel": f"attn_{dom}_kernel", "achieved": achieved,
                     "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                     "frac_of_sustained": achieved / peak_sus, "peak_source": src,
                     "traffic": traffic,
                     "algorithmic_flops_per_launch": dom_flops},
        "e2e": {"value": fl / (ms_e2e * 1e-3) / 1e12, "unit": "TFLOP/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": ms_e2e,
                "path": "pipeline.HostAttention (flashcore.block_attn_update_final + backward_aux + "
                        "block_attn_backward over the C ABI): pinned-host q/k/v/dO in, bf16 "
                        "dQ/dK/dV out, copies overlapped per group of %d heads, 3 compute streams; consecutive "
                        "steps overlap (step i+1's H2D of a group waits only for step i's compute of it)"
                        % args.heads_per_group},
        "gpu_launches": 3 * args.steps,
        "clocks": clk.summary(),
    }
    if not args.no_cpu_baseline:
        try:
            s = reference_sample(cpu_threads())
            line["cpu_baseline"] = {"value": s["tflops"], "unit": "TFLOP/s", "cores": s["threads"],
                                    "kind": "reference", "sample": s["sample"],
                                    "seconds": s["seconds"]}
        except Exception as exc:  # pragma: no cover - reported, not fatal
            line["cpu_baseline"] = {"value": None, "unit": "TFLOP/s", "cores": cpu_threads(),
                                    "kind": "reference", "sample": f"unavailable: {exc}"}
    print(json.dumps(line), flush=True)
    return 0


def run_multi(args):
    from paper_2310_03294_b200 import dist
    return dist.bench_main(args)


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seq", type=int, default=SEQ)
    ap.add_argument("--heads", type=int, default=H)
    ap.add_argument("--heads-per-group", type=int, default=2)  # e2e copy/compute granularity (A/B: 2 >= 1 by ~0.5-1%)
    ap.add_argument("--fwd-schedule", default="balanced", choices=["ring", "balanced", "balanced_split"])
    ap.add_argument("--bwd-schedule", default="balanced", choices=["ring", "balanced"])
    ap.add_argument("--runtime", default="native", choices=["native", "python"],
                    help="N>1: the C++ per-rank runtime (da_rank_*) or dist.DistRuntime")
    ap.add_argument("--transport", default="peer", choices=["peer", "nccl"],
                    help="--runtime python: copy-engine pulls from peer HBM or NCCL send/recv")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--force-dist", action="store_true",
                    help="run the torchrun/NCCL path even at one rank (tests the N>1 code)")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus > 1 or world > 1 or args.force_dist:
        return run_multi(args)
    return run_single(args)


if __name__ == "__main__":
    sys.exit(main())
