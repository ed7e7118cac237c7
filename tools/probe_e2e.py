"""e2e (pinned host in/out) timing of pipeline.HostAttention per heads_per_group."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2310_03294_b200.pipeline import HostAttention  # noqa: E402

h, n = 32, int(sys.argv[1]) if len(sys.argv) > 1 else 32768
host = [(torch.rand(h, n, 128) * 2 - 1).to(torch.bfloat16).pin_memory() for _ in range(4)]
outs = [torch.empty(h, n, 128, dtype=torch.bfloat16).pin_memory() for _ in range(3)]
fl = 7 * n * n * 128 * h
for spec in (sys.argv[2] if len(sys.argv) > 2 else "2x1,2x2,4x2").split(","):
    hpg, cs = (int(x) for x in spec.split("x"))
    ha = HostAttention(h, n, 128, heads_per_group=hpg, compute_streams=cs)
    for _ in range(2):
        ha(*host, *outs)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(4):
        ha(*host, *outs, sync=False)
    ha.join()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 4
    print(f"hpg {hpg:2d} streams {cs}: {ms:.2f} ms  {fl / ms / 1e9:.1f} TFLOP/s e2e", flush=True)
    del ha
    torch.cuda.empty_cache()
