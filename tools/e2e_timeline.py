"""Kernel timeline of the host-buffer pipeline (pipeline.HostAttention) under
torch.profiler: busy fraction of the GPU over K steps and the largest idle gaps.
Development tool (numbers under a profiler are not bench values)."""
import sys
from pathlib import Path

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2310_03294_b200.pipeline import HostAttention  # noqa: E402

h, n = 32, int(sys.argv[1]) if len(sys.argv) > 1 else 32768
host = [(torch.rand(h, n, 128) * 2 - 1).to(torch.bfloat16).pin_memory() for _ in range(4)]
outs = [torch.empty(h, n, 128, dtype=torch.bfloat16).pin_memory() for _ in range(3)]
ha = HostAttention(h, n, 128, heads_per_group=1)
for _ in range(3):
    ha(*host, *outs)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(4):
        ha(*host, *outs, sync=False)
    ha.join()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
kern = sorted((e.time_range.start, e.time_range.end, e.name) for e in ev
              if "Memcpy" not in e.name and "memcpy" not in e.name.lower())
cp = sorted((e.time_range.start, e.time_range.end, e.name) for e in ev if "emcpy" in e.name)
t0, t1 = min(k[0] for k in kern + cp), max(k[1] for k in kern + cp)
# union of kernel intervals (several streams)
busy, cur_s, cur_e = 0, None, None
gaps = []
for s, e, _ in kern:
    if cur_e is None or s > cur_e:
        if cur_e is not None:
            busy += cur_e - cur_s
            gaps.append((s - cur_e, cur_e - t0))
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
busy += cur_e - cur_s
print(f"window {(t1 - t0) / 1e3:.2f} ms, kernels busy {busy / 1e3:.2f} ms ({busy / (t1 - t0):.3f}); "
      f"first kernel at {(kern[0][0] - t0) / 1e3:.2f} ms, last ends {(t1 - kern[-1][1]) / 1e3:.2f} ms "
      f"before the window end")
for g, at in sorted(gaps, reverse=True)[:8]:
    print(f"  idle {g / 1e3:.3f} ms at {at / 1e3:.2f} ms")
