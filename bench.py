"""Benchmark: causal attention forward+backward (DistFlashAttn hot path) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg2|cfg2gqa|cfg3|cfg4|cfg5]

N=1 workload = BASELINE.json configs[1] (cfg2): Llama-7B attention layer (32
heads, d=128), causal fwd+bwd at seq 32K on one B200, synthetic U[-1,1) bf16
inputs generated on the device. One step = one forward (block_attn_update
with the fused finalize) + backward_aux + block_attn_backward over the full
sequence. `--config cfg2gqa` is the same with 8 kv heads (cfg5's ratio).

N>1 (configs[2..4]; default cfg3 = 128K tokens over N GPUs, strong scaling)
runs the native per-rank runtime (csrc/rank_runtime.cu), one process per GPU:
plain `python bench.py --gpus N` spawns its N ranks itself (torchrun works
too). The headline leg is the balanced forward with the even-P split +
balanced backward; the same line carries the ring/ring and balanced/balanced
legs (the north_star balanced-vs-ring speed-up) and a no-communication leg
(same kernels on local buffers) from which exposed communication is
computed as the reference's comm_overhead_pct (analyzer.cpp:60-64).
Transport: NCCL send/recv on a side stream when the ranks sit on distinct
GPUs, CUDA-IPC copy-engine pulls when they share one (--share-gpu, tests).

Metric: whole-job attention fwd+bwd TFLOP/s (algorithmic causal FLOPs
7·N²·d·H per step, no recompute counted), with tokens/s and per-GPU TFLOP/s
beside it. Inputs exceed the 126 MB L2 at every config, so no flush is needed
between steps.

--impl reference times the reference's own CPU implementation (the
unmodified sources compiled into oracle/_ref/ref_driver) on a bounded sample
of the same workload, with every host core busy.
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


def reference_sample(threads: int, n: int = 8192, workers: int = 8, heads: int | None = None,
                     schedule: str = "balanced") -> dict:
    """The reference CPU path (oracle/_ref/ref_driver: unmodified sources) on a
    bounded sample of the workload: `heads` heads of seq n run concurrently,
    P=workers threads each (the reference's concurrent executor,
    runtime.cpp:481-484), balanced forward + ring backward. By default
    heads = threads // workers so every host core is busy; `threads` in the
    result is the number of threads that actually ran."""
    from oracle import oracle as O
    if not O.ref_available():
        raise RuntimeError("oracle/_ref/ref_driver missing (build with `make -C oracle ref`)")
    if heads is None:
        heads = max(1, threads // workers)
    r = O.ref_time(n, workers, heads, D, schedule, threads)
    return {"seconds": r["seconds"], "tflops": r["tflops"], "threads": r["threads"],
            "sample": f"{heads} head(s) x seq {n} x d {D} concurrently, P={workers} worker "
                      f"threads each ({schedule} fwd + ring bwd, reference concurrent executor), "
                      "bf16-rounded fp64 inputs"}


def cpu_baseline(threads: int) -> dict:
    """BASELINE.md's CPU anchors: the 16K sample (all cores) as the value,
    BASELINE configs[0] (seq 4096, d=128, P=4, one head) timed in full beside
    it. Larger configs are N^2 * H extrapolations of the anchor, labelled so."""
    s = reference_sample(threads, n=16384, workers=8)
    c1 = reference_sample(threads, n=4096, workers=4, heads=1)
    per_head_s = s["seconds"] * (threads // 8 or 1) / max(1, s["threads"] // 8)
    return {"value": s["tflops"], "unit": "TFLOP/s", "cores": s["threads"], "kind": "reference",
            "sample": s["sample"], "seconds": s["seconds"],
            "cfg1_seconds": c1["seconds"], "cfg1_threads": c1["threads"],
            "cfg1": "BASELINE configs[0] in full: 1 head x seq 4096 x d 128, P=4 (balanced fwd + "
                    "ring bwd), reference concurrent executor",
            "cfg2_extrapolated_s": s["seconds"] * (32768 / 16384) ** 2 * 32 / max(1, s["threads"] // 8),
            "extrapolation": "cfg2 (32 heads x 32K) from the 16K anchor by N^2 * H over the "
                             "concurrently running heads (not measured)",
            "per_head_s_16k": per_head_s}


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
        "ms_per_step": secs * 1e3, "higher_is_better": True,
        "scaling": "weak" if args.gpus == 1 else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "llama7b-attn causal fwd+bwd (reference CPU, bounded sample of "
                               + _cfg(args)["name"] + ")",
                   "heads": _cfg(args)["heads"], "d": D, "seq_len": _cfg(args)["seq"]},
        "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": vals[0]["threads"],
                         "kind": "reference", "sample": vals[0]["sample"]},
        "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


CONFIGS = {
    # name: (total seq, q heads, kv heads, BASELINE configs[] index)
    "cfg2": (32768, 32, 32, 1),
    "cfg2gqa": (32768, 32, 8, 4),
    "cfg3": (131072, 32, 32, 2),
    "cfg4": (524288, 32, 32, 3),
    "cfg5": (262144, 32, 8, 4),
}


def _cfg(args) -> dict:
    name = args.config or ("cfg2" if args.gpus == 1 else "cfg3")
    seq, hq, hkv, idx = CONFIGS[name]
    if args.seq:
        seq = args.seq
    if args.heads:
        hq = args.heads
        hkv = min(hkv, hq) if hkv != CONFIGS[name][1] else hq
    return {"name": name, "seq": seq, "heads": hq, "heads_kv": hkv, "baseline_index": idx}


# ----------------------------------------------------------------------------- our arm, N=1
def _profile_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu capture."""
    f = ROOT / "profiles" / "roofline_traffic.json"
    try:
        return json.loads(f.read_text())
    except Exception:
        return {}


# Shared-memory bytes each kernel moves per (query tile, kv tile) pair of 128 x 128
# (DESIGN.md §4): the bound both kernels actually run against.
#   forward  (per tile pair; a CTA owns two query tiles): S = Q K^T operands 64 KB,
#            PV operands (P from smem) 64 KB, K/V TMA writes 32 KB, P stores 32 KB
#   backward: MMA operands 256 KB (S 64, dP 64, dV 32, dK 32, dQ^T 64), Q/dO TMA
#            writes 64 KB, dS stores 32 KB, dQ partial staging 128 KB (stores +
#            TMA reads), -lse / -D broadcast loads 32 KB (8 warps x 32 x 128 B)
SMEM_BYTES_PER_PAIR = {"fwd": 196608, "bwd": 524288}
SMEM_B_PER_CLK_PER_SM = 128.0  # B300_MICROARCH.md "smem crossbar BW" (same SM design on B200)
N_SM = 148


def smem_roofline(n: int, heads: int, t_fwd_ms: float, t_bwd_ms: float, mhz) -> dict:
    """Achieved shared-memory bandwidth per SM of both chunk kernels (causal
    32K: n_t (n_t + 1) / 2 tile pairs per head) against 128 B/clk/SM."""
    nt = (n + 127) // 128
    pairs = heads * nt * (nt + 1) // 2
    out = {"peak_B_per_clk_per_SM": SMEM_B_PER_CLK_PER_SM, "tile_pairs_per_launch": pairs,
           "bytes_per_tile_pair": SMEM_BYTES_PER_PAIR, "clock_mhz": mhz}
    if not mhz:
        return out
    for k, t in (("fwd", t_fwd_ms), ("bwd", t_bwd_ms)):
        b = pairs * SMEM_BYTES_PER_PAIR[k] / (t * 1e-3 * mhz * 1e6 * N_SM)
        out[k] = {"achieved_B_per_clk_per_SM": b, "frac": b / SMEM_B_PER_CLK_PER_SM}
    return out


def run_single(args):
    import torch
    from paper_2310_03294_b200 import flashcore as F

    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    cfg = _cfg(args)
    n, heads, hkv = cfg["seq"], cfg["heads"], cfg["heads_kv"]
    stream = torch.cuda.current_stream()

    def rnd(*shape):
        return (torch.rand(*shape, device=dev) * 2 - 1).to(torch.bfloat16)

    torch.manual_seed(0)
    q, k, v, d_out = rnd(heads, n, D), rnd(hkv, n, D), rnd(hkv, n, D), rnd(heads, n, D)
    grads = F.ChunkGrads(torch.zeros(heads, n, D, device=dev), torch.empty(hkv, n, D, device=dev),
                         torch.empty(hkv, n, D, device=dev))

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
    hdq, hdk, hdv = (torch.empty(*t.shape, dtype=torch.bfloat16).pin_memory() for t in (q, k, v))
    del grads
    hpg = max(args.heads_per_group, heads // hkv)
    ha = HostAttention(heads, n, D, heads_per_group=hpg, device=dev, heads_kv=hkv)

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
    clocks = clk.summary()
    smem = smem_roofline(n, heads, t_fwd, t_bwd, clocks.get("sm_mhz"))
    # roofline denominator (B200_PROFILING.md): the sustained cuBLAS figure for
    # a kernel timed inside a long step under the power cap, the burst figure
    # for a kernel timed alone; the timed region here is the repeated step, so
    # it is the sustained one whenever the power cap held the clock there
    long_step = "sw_power_cap" in clocks.get("reasons", [])
    peak_used = peak_sus if long_step else peak
    line = {
        "metric": "attn fwd+bwd TFLOP/s", "value": tflops, "unit": "TFLOP/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": f"llama7b-attn causal fwd+bwd, {heads} q / {hkv} kv heads, d=128, "
                               f"seq {n}, 1 B200 (BASELINE configs[{cfg['baseline_index']}]"
                               + (" shape per GPU)" if cfg["name"] != "cfg2" else ")"),
                   "name": cfg["name"], "heads": heads, "heads_kv": hkv, "d": D, "seq_len": n,
                   "mask": "causal", "workers": 1,
                   "l2": "inputs (4 x %d MB) exceed L2; no flush" % (heads * n * D * 2 >> 20)},
        "tokens_per_s": n / (ms * 1e-3),
        "tflops_per_gpu": tflops,
        "frac_of_peak": tflops / peak,
        "kernel_ms": {"fwd": t_fwd, "bwd_preprocess": t_aux, "bwd": t_bwd},
        "kernel_tflops": {"fwd": 2.0 * n * n * D * heads / (t_fwd * 1e-3) / 1e12,
                          "bwd": 5.0 * n * n * D * heads / (t_bwd * 1e-3) / 1e12},
        "roofline": {"bound": "tensor", "kernel": f"attn_{dom}_kernel", "achieved": achieved,
                     "peak": peak_used, "unit": "TFLOP/s", "frac": achieved / peak_used,
                     "peak_basis": ("sustained (kernel timed inside the repeated step under "
                                    "sw_power_cap)" if long_step else "burst"),
                     "frac_of_burst": achieved / peak, "frac_of_sustained": achieved / peak_sus,
                     "peak_source": src,
                     "traffic": traffic if cfg["name"] == "cfg2" else None,
                     "algorithmic_flops_per_launch": dom_flops,
                     "smem": smem},
        "e2e": {"value": fl / (ms_e2e * 1e-3) / 1e12, "unit": "TFLOP/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": ms_e2e,
                "path": "pipeline.HostAttention -> C++ host pipeline (da_pipeline_step: fwd with "
                        "fused finalize + backward_aux + backward + bf16 conversion per head group): "
                        "pinned-host q/k/v/dO in, bf16 dQ/dK/dV out, copies overlapped per group of "
                        "%d heads, 3 compute streams; consecutive steps overlap (step i+1's H2D of a "
                        "group waits only for step i's compute of it)" % hpg},
        "gpu_launches": 3 * args.steps,
        "clocks": clocks,
    }
    if not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(cpu_threads())
        except Exception as exc:  # pragma: no cover - reported, not fatal
            line["cpu_baseline"] = {"value": None, "unit": "TFLOP/s", "cores": cpu_threads(),
                                    "kind": "reference", "sample": f"unavailable: {exc}"}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- our arm, N>1
NVLINK_GBS = 770.0  # measured peer copy per direction per GPU (B200_PROFILING.md; 900 nominal)


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def spawn_ranks(args, argv) -> int:
    """`python bench.py --gpus N` without torchrun: start the N ranks (one
    process per GPU, rank 0 prints the line) and return the worst exit code."""
    port = _free_port()
    procs = []
    for r in range(args.gpus):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(args.gpus),
                   LOCAL_WORLD_SIZE=str(args.gpus), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, str(Path(__file__).resolve()), *argv],
                                      env=env, stdout=None if r == 0 else subprocess.DEVNULL))
    rcs = [None] * len(procs)
    while any(rc is None for rc in rcs):
        for i, p in enumerate(procs):
            if rcs[i] is None:
                rcs[i] = p.poll()
        if any(rc not in (None, 0) for rc in rcs):  # one rank failed: the others would hang
            for i, p in enumerate(procs):
                if rcs[i] is None:
                    p.kill()
                    rcs[i] = p.wait()
            break
        time.sleep(0.2)
    return max(abs(rc) for rc in rcs)


def received_bytes(cf, cb, nq: int) -> int:
    """Bytes this rank received in one fwd+bwd step, from the runtime's counters
    (counted by the receiver, runtime.cpp:50-83 x heads): KV bf16, Q bf16,
    forward partials fp32 (o | m | l), GradKV fp32, the backward (q, dO, lse,
    D) bundle (q_scalars = nq * 258 -> nq * 520 bytes) and dq partials fp32."""
    fwd = 2 * cf.kv_scalars + 2 * cf.q_scalars + 4 * cf.partial_scalars
    bwd = 2 * cb.kv_scalars + 4 * cb.grad_scalars + 4 * cb.partial_scalars
    bwd += cb.q_scalars * 520 // 258
    return int(fwd + bwd)


def run_multi(args):
    """One rank of the N-GPU run (torchrun or spawn_ranks): the native per-rank
    runtime, device-timed legs, max over ranks, rank 0 prints the line."""
    import torch
    import torch.distributed as tdist
    from paper_2310_03294_b200.rank import RankRuntime

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    if world != args.gpus:
        raise SystemExit(f"WORLD_SIZE={world} but --gpus {args.gpus}")
    ndev = torch.cuda.device_count()
    if ndev < world and not args.share_gpu:
        raise SystemExit(f"--gpus {world} needs {world} visible GPUs (found {ndev}); "
                         "--share-gpu runs every rank on cuda:0 (tests)")
    dev_index = 0 if args.share_gpu else local % ndev
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    # host bootstrap + timing reductions; the data plane is the runtime's own
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    transport = args.transport
    if transport == "auto":
        transport = "ipc" if args.share_gpu else "nccl"
    cfg = _cfg(args)
    seq, heads, hkv = cfg["seq"], cfg["heads"], cfg["heads_kv"]
    if seq % world:
        raise SystemExit(f"seq {seq} does not divide over {world} ranks")
    rows = seq // world
    torch.manual_seed(1234 + rank)

    def rnd(h):
        return (torch.rand(h, rows, D, device=dev) * 2 - 1).to(torch.bfloat16)

    q, k, v, do = rnd(heads), rnd(hkv), rnd(hkv), rnd(heads)
    runtimes = {}

    def runtime(tr):
        if tr not in runtimes:
            runtimes[tr] = RankRuntime(rank, world, transport=tr,
                                       nccl_max_ctas=args.nccl_max_ctas)
        return runtimes[tr]

    fallback = None
    if transport == "nccl":
        # NCCL must load on every rank before any rank enters the collective
        # communicator init; if it cannot, every rank uses the IPC pulls instead
        from paper_2310_03294_b200.errors import Error as DaError
        ok = torch.tensor([1.0])
        try:
            import ctypes as _C
            _C.CDLL("libnccl.so.2", mode=_C.RTLD_GLOBAL)
        except OSError as exc:
            ok[0], fallback = 0.0, f"libnccl.so.2 not loadable: {exc}"
        tdist.all_reduce(ok, op=tdist.ReduceOp.MIN)
        if ok.item() > 0:
            try:
                runtime("nccl")
            except DaError as exc:  # the communicator init itself failed (collective)
                ok[0], fallback = 0.0, f"NCCL init failed: {exc}"
            tdist.all_reduce(ok, op=tdist.ReduceOp.MIN)
        if ok.item() == 0:
            for rt_ in runtimes.values():
                rt_.close()
            runtimes.clear()
            transport, fallback = "ipc", fallback or "NCCL failed on another rank"

    def timed(fwd, bwd, tr, steps, clk=None):
        rt = runtime(tr)
        res = {}

        def step():
            _, _, res["cf"] = rt.forward(q, k, v, fwd)
            res["cb"] = rt.backward(do, bwd)[3]

        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        tdist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if clk:
            clk.timed(True)
        s.record()
        for _ in range(steps):
            step()
        e.record()
        torch.cuda.synchronize()
        if clk:
            clk.timed(False)
        tdist.barrier()
        ms = torch.tensor([s.elapsed_time(e) / steps])
        tdist.all_reduce(ms, op=tdist.ReduceOp.MAX)
        return ms.item(), res["cf"], res["cb"]

    fl = flops_fwd_bwd(seq, heads)
    head_fwd, head_bwd = args.fwd_schedule, args.bwd_schedule
    with ClockSampler(dev_index) as clk:  # started before the warm-up
        ms, cf, cb = timed(head_fwd, head_bwd, transport, args.steps, clk)
    legs = {f"{head_fwd}+{head_bwd}": {"ms": ms, "tflops": fl / (ms * 1e-3) / 1e12,
                                       "transport": transport}}
    if not args.no_legs:
        leg_steps = max(2, args.leg_steps)
        for name, f, b, tr in (("ring+ring", "ring", "ring", transport),
                               ("balanced+balanced", "balanced", "balanced", transport),
                               ("nocomm", head_fwd, head_bwd, "none")):
            if name in legs:
                continue
            lms = timed(f, b, tr, leg_steps)[0]
            legs[name] = {"ms": lms, "tflops": fl / (lms * 1e-3) / 1e12, "transport": tr,
                          "fwd": f, "bwd": b}
    nbytes = torch.tensor([float(received_bytes(cf, cb, heads * rows))])
    tdist.all_reduce(nbytes, op=tdist.ReduceOp.MAX)
    launches = torch.tensor([float(cf.attention_kernel_calls + cf.partial_messages + 1 + 1 +
                                   cb.attention_kernel_calls + 2 * cb.grad_messages +
                                   cb.partial_messages)])
    tdist.all_reduce(launches, op=tdist.ReduceOp.SUM)

    # e2e through the same public API with host buffers: each rank's shard is
    # copied in from pinned host memory and its bf16 gradients out, inside the
    # timed region; step j+1's copy-in and step j's copy-out overlap compute
    rt = runtime(transport)
    host_in = [t.cpu().pin_memory() for t in (q, k, v, do)]
    host_out = [torch.empty(*t.shape, dtype=torch.bfloat16).pin_memory() for t in (q, k, v)]
    dev_in = [[torch.empty_like(t) for t in (q, k, v, do)] for _ in range(2)]
    cur = torch.cuda.current_stream()
    h2d, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    freed = [None, None]

    def load(j):
        slot = j % 2
        with torch.cuda.stream(h2d):
            if freed[slot] is not None:
                h2d.wait_event(freed[slot])
            for dst, src in zip(dev_in[slot], host_in):
                dst.copy_(src, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(h2d)
        return ev

    def e2e_run(n_steps):
        h2d.wait_stream(cur)
        ready = load(0)
        for j in range(n_steps):
            nxt = load(j + 1) if j + 1 < n_steps else None  # prefetch
            cur.wait_event(ready)
            x = dev_in[j % 2]
            rt.forward(x[0], x[1], x[2], head_fwd)
            grads = rt.backward(x[3], head_bwd)[:3]
            g16 = [g.to(torch.bfloat16) for g in grads]
            done = torch.cuda.Event()
            done.record(cur)
            freed[j % 2] = done
            d2h.wait_event(done)
            with torch.cuda.stream(d2h):
                for src, dst in zip(g16, host_out):
                    dst.copy_(src, non_blocking=True)
                    src.record_stream(d2h)
            ready = nxt
        cur.wait_stream(d2h)

    e2e_run(2)
    torch.cuda.synchronize()
    tdist.barrier()
    e_steps = max(2, args.steps)
    s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s2.record()
    e2e_run(e_steps)
    e2.record()
    torch.cuda.synchronize()
    tdist.barrier()
    ms_e2e = torch.tensor([s2.elapsed_time(e2) / e_steps])
    tdist.all_reduce(ms_e2e, op=tdist.ReduceOp.MAX)
    ms_e2e = ms_e2e.item()
    for rt_ in runtimes.values():
        rt_.close()

    if rank == 0:
        peak, peak_sus, src = peaks()
        clocks = clk.summary()
        long_step = "sw_power_cap" in clocks.get("reasons", [])  # see run_single
        peak_used = peak_sus if long_step else peak
        per_gpu = fl / (ms * 1e-3) / 1e12 / world
        t_tensor = fl / world / (peak_used * 1e12)
        t_link = nbytes.item() / (NVLINK_GBS * 1e9)
        t_roof = max(t_tensor, t_link)
        ring = legs.get("ring+ring", {}).get("ms")
        nocomm = legs.get("nocomm", {}).get("ms")
        line = {
            "metric": "attn fwd+bwd TFLOP/s", "value": fl / (ms * 1e-3) / 1e12, "unit": "TFLOP/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"llama7b-attn causal fwd+bwd, {heads} q / {hkv} kv heads, "
                                   f"d=128, seq {seq} over {world} B200 (BASELINE configs"
                                   f"[{cfg['baseline_index']}]), {head_fwd} fwd + {head_bwd} bwd, "
                                   f"native per-rank runtime, {transport} transport",
                       "name": cfg["name"], "heads": heads, "heads_kv": hkv, "d": D,
                       "seq_len": seq, "tokens_per_gpu": rows, "fwd_schedule": head_fwd,
                       "bwd_schedule": head_bwd, "transport": transport,
                       "shared_gpu": bool(args.share_gpu),
                       "transport_fallback": fallback,
                       "l2": "inputs exceed L2; no flush"},
            "tokens_per_s": seq / (ms * 1e-3),
            "tflops_per_gpu": per_gpu,
            "legs": legs,
            "balanced_speedup_vs_ring": (ring / ms) if ring else None,
            "exposed_comm_pct": (100.0 * (ms - nocomm) / nocomm) if nocomm else None,
            "exposed_comm_definition": "(t - t_nocomm) / t_nocomm, t_nocomm = same kernels and "
                                       "schedule on local buffers (analyzer.cpp:60-64)",
            "roofline": {"bound": "tensor" if t_tensor >= t_link else "nvlink",
                         "kernel": "whole step per GPU (compute + exposed NVLink)",
                         "achieved": per_gpu, "peak": peak_used, "unit": "TFLOP/s",
                         "peak_basis": "sustained (power-capped step)" if long_step else "burst",
                         "frac_of_burst_tensor": per_gpu / peak,
                         "frac": t_roof / (ms * 1e-3), "t_roof_ms": t_roof * 1e3,
                         "t_tensor_ms": t_tensor * 1e3, "t_nvlink_ms": t_link * 1e3,
                         "nvlink_bytes_per_gpu": nbytes.item(), "nvlink_gbs": NVLINK_GBS,
                         "peak_source": src, "frac_of_sustained_tensor": per_gpu / peak_sus,
                         "traffic": None},
            "e2e": {"value": fl / (ms_e2e * 1e-3) / 1e12, "unit": "TFLOP/s",
                    "h2d_bytes_per_step": sum(t.numel() * 2 for t in host_in) * world,
                    "d2h_bytes_per_step": sum(t.numel() * 2 for t in host_out) * world,
                    "ms_per_step": ms_e2e,
                    "path": "rank.RankRuntime (C++ da_rank_*) forward/backward with pinned-host "
                            "shards in and bf16 grads out, every rank; step j+1's copy-in and "
                            "step j's copy-out overlap compute (two input sets, two copy streams)"},
            "gpu_launches": int(launches.item()) * args.steps,
            "clocks": clocks,
            "cpu_baseline_note": "the reference CPU path is timed at N=1 only (bench contract)",
        }
        print(json.dumps(line), flush=True)
    tdist.destroy_process_group()
    return 0


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help="default: cfg2 at N=1, cfg3 (128K over N) at N>1")
    ap.add_argument("--seq", type=int, default=0, help="override the config's total tokens")
    ap.add_argument("--heads", type=int, default=0, help="override the config's query heads")
    ap.add_argument("--heads-per-group", type=int, default=2)  # e2e copy/compute granularity (A/B: 2 >= 1 by ~0.5-1%)
    ap.add_argument("--fwd-schedule", default="balanced_split",
                    choices=["ring", "balanced", "balanced_split"])
    ap.add_argument("--bwd-schedule", default="balanced_split",
                    choices=["ring", "balanced", "balanced_split"])
    ap.add_argument("--transport", default="auto", choices=["auto", "nccl", "ipc"],
                    help="N>1: NCCL send/recv (distinct GPUs) or CUDA-IPC pulls (shared GPU)")
    ap.add_argument("--nccl-max-ctas", type=int, default=0)
    ap.add_argument("--share-gpu", action="store_true",
                    help="N>1 on one GPU (every rank on cuda:0; tests the multi-rank path)")
    ap.add_argument("--no-legs", action="store_true", help="N>1: headline leg only")
    ap.add_argument("--leg-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1:
        if "WORLD_SIZE" not in os.environ:
            return spawn_ranks(args, argv)
        return run_multi(args)
    return run_single(args)


if __name__ == "__main__":
    sys.exit(main())
