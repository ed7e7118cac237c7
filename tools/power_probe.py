"""SM clock and board power of each kernel under the 1000 W cap (development tool).

Runs the 32-head x 32K causal forward alone, the backward alone and the whole
bench step back to back for a few seconds each, with uniform [-1, 1) inputs
and with all-zero inputs, sampling NVML (SM clock, power) in a thread; prints
one line per case: median clock, median power, ms per launch and the energy
per TFLOP. Numbers under this tool are diagnostics, not bench values.

    python tools/power_probe.py [seconds]
"""
import statistics
import sys
import threading
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2310_03294_b200 import flashcore as F  # noqa: E402

H, N, D = 32, 32768, 128
secs = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0


def sampler(out, stop):
    import pynvml as nv
    nv.nvmlInit()
    h = nv.nvmlDeviceGetHandleByIndex(0)
    while not stop[0]:
        out.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                    nv.nvmlDeviceGetPowerUsage(h) / 1000.0))
        time.sleep(0.01)


def run(name, fn, flops):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    samples, stop = [], [False]
    th = threading.Thread(target=sampler, args=(samples, stop), daemon=True)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 0
    t0 = time.time()
    s.record()
    th.start()
    while time.time() - t0 < secs:
        fn()
        n += 1
        if n % 8 == 0:
            torch.cuda.synchronize()
    e.record()
    torch.cuda.synchronize()
    stop[0] = True
    th.join()
    ms = s.elapsed_time(e) / n
    clk = statistics.median(x[0] for x in samples)
    pw = statistics.median(x[1] for x in samples)
    tf = flops / (ms * 1e-3) / 1e12
    print(f"{name:28s} {ms:8.3f} ms  {tf:7.1f} TFLOP/s  clock {clk:6.0f} MHz  power {pw:6.0f} W  "
          f"{pw / tf:6.3f} J per TFLOP  ({clk / tf:5.3f} MHz per TFLOP/s)", flush=True)


def main():
    for label, scale in (("uniform[-1,1)", 1.0), ("zeros", 0.0)):
        torch.manual_seed(0)
        q, k, v, do = [((torch.rand(H, N, D, device="cuda") * 2 - 1) * scale).to(torch.bfloat16)
                       for _ in range(4)]
        out = F.block_attn_update_final(q, k, v, None, F.MaskMode.Diagonal)
        dvec = F.backward_aux(do, out.o)
        grads = F.ChunkGrads(torch.zeros(H, N, D, device="cuda"), torch.empty(H, N, D, device="cuda"),
                             torch.empty(H, N, D, device="cuda"))

        def fwd():
            F.block_attn_update_final(q, k, v, None, F.MaskMode.Diagonal)

        def bwd():
            F.block_attn_backward(q, k, v, out.o, out.lse, do, F.MaskMode.Diagonal, d_vec=dvec,
                                  grads=grads)

        def step():
            o = F.block_attn_update_final(q, k, v, None, F.MaskMode.Diagonal)
            dv_ = F.backward_aux(do, o.o)
            grads.dq.zero_()
            F.block_attn_backward(q, k, v, o.o, o.lse, do, F.MaskMode.Diagonal, d_vec=dv_,
                                  grads=grads)

        run(f"forward   {label}", fwd, 2.0 * N * N * D * H)
        run(f"backward  {label}", bwd, 5.0 * N * N * D * H)
        run(f"step      {label}", step, 7.0 * N * N * D * H)


if __name__ == "__main__":
    main()
