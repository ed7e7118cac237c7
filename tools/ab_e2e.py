"""Sustained A/B of the host-buffer pipeline (bench.py's e2e leg) across
library variants (development tool).

    python tools/ab_e2e.py LIB [seconds] [heads_per_group]
32 heads x 32K causal fwd+bwd from pinned host buffers through
pipeline.HostAttention, back-to-back calls (sync=False) for `seconds`;
prints ms per step and TFLOP/s."""
import os
import sys
import time
from pathlib import Path

os.environ["DISTATTN_B200_LIB"] = sys.argv[1]
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2310_03294_b200.pipeline import HostAttention  # noqa: E402

secs = float(sys.argv[2]) if len(sys.argv) > 2 else 4.0
hpg = int(sys.argv[3]) if len(sys.argv) > 3 else 2
H, N = 32, 32768
torch.manual_seed(0)
host = [((torch.rand(H, N, 128) * 2 - 1).to(torch.bfloat16)).pin_memory() for _ in range(4)]
outs = [torch.empty(H, N, 128, dtype=torch.bfloat16).pin_memory() for _ in range(3)]
ha = HostAttention(H, N, heads_per_group=hpg)
st = torch.cuda.current_stream()
for _ in range(3):
    ha(*host, *outs, sync=False)
ha.check()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(st)
n = 0
t0 = time.time()
while time.time() - t0 < secs:
    ha(*host, *outs, sync=False)
    n += 1
    if n % 8 == 0:
        ha.join()
        torch.cuda.synchronize()
ha.join()
e.record(st)
torch.cuda.synchronize()
ms = s.elapsed_time(e) / n
print(f"{Path(sys.argv[1]).name}: e2e {ms:.3f} ms/step  {7 * N * N * 128 * H / (ms * 1e-3) / 1e12:.1f} "
      f"TFLOP/s  n={n}", flush=True)
