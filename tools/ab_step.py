"""Sustained A/B of library variants on the bench step (development tool).

    python tools/ab_step.py LIB [seconds]
Runs the bench.py N=1 step (forward with fused finalize + backward_aux +
backward, 32 heads x 32K) back to back for `seconds` after a warm-up, with
the library at LIB (DISTATTN_B200_LIB), and prints mean fwd / bwd / step ms
and the median SM clock under load (NVML)."""
import os
import statistics
import sys
import threading
import time
from pathlib import Path

lib = sys.argv[1]
os.environ["DISTATTN_B200_LIB"] = lib
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2310_03294_b200 import flashcore as F  # noqa: E402

secs = float(sys.argv[2]) if len(sys.argv) > 2 else 3.0
H, N = 32, 32768
torch.manual_seed(0)
q, k, v, do = [(torch.rand(H, N, 128, device="cuda") * 2 - 1).to(torch.bfloat16) for _ in range(4)]
grads = F.ChunkGrads(torch.zeros(H, N, 128, device="cuda"), torch.empty(H, N, 128, device="cuda"),
                     torch.empty(H, N, 128, device="cuda"))
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream()
clocks = []
stop = False


def sampler():
    import pynvml as nv
    nv.nvmlInit()
    h = nv.nvmlDeviceGetHandleByIndex(0)
    while not stop:
        clocks.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
        time.sleep(0.01)


def step(ev):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(st)
    out = F.block_attn_update_final(q, k, v, None, F.MaskMode.Diagonal, degenerate_flag=flag)
    e[1].record(st)
    dvec = F.backward_aux(do, out.o)
    grads.dq.zero_()
    F.block_attn_backward(q, k, v, out.o, out.lse, do, F.MaskMode.Diagonal, d_vec=dvec, grads=grads)
    e[2].record(st)
    ev.append(e)


for _ in range(5):
    step([])
torch.cuda.synchronize()
th = threading.Thread(target=sampler, daemon=True)
th.start()
ev = []
t0 = time.time()
while time.time() - t0 < secs:
    step(ev)
    if len(ev) % 10 == 0:
        torch.cuda.synchronize()
torch.cuda.synchronize()
stop = True
fwd = statistics.mean(a.elapsed_time(b) for a, b, _ in ev)
bwd = statistics.mean(b.elapsed_time(c) for _, b, c in ev)
print(f"{Path(lib).name}: fwd {fwd:.3f} ms  bwd {bwd:.3f} ms  step {fwd + bwd:.3f} ms  "
      f"({7 * N * N * 128 * H / ((fwd + bwd) * 1e-3) / 1e12:.1f} TFLOP/s)  "
      f"clock {statistics.median(clocks) if clocks else 0:.0f} MHz  n={len(ev)}", flush=True)
