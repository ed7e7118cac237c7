"""Prints the forward kernel's per-iteration clock64 timeline (CTA 0, DA_TRACE build)."""
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2310_03294_b200 import _lib  # noqa: E402
from paper_2310_03294_b200.flashcore import MaskMode, block_attn_update_final  # noqa: E402

h, n = 32, int(sys.argv[1]) if len(sys.argv) > 1 else 16384
q, k, v = [(torch.rand(h, n, 128, device="cuda") * 2 - 1).to(torch.bfloat16) for _ in range(3)]
tr = torch.zeros(64 * 16 + 8 * h * ((n + 255) // 256), dtype=torch.int64, device="cuda")  # + per-CTA records
_lib.lib().da_debug_set_fwd_trace(C.c_void_p(tr.data_ptr()))
for _ in range(3):
    block_attn_update_final(q, k, v, None, MaskMode.Diagonal)
torch.cuda.synchronize()
t = tr[:1024].view(64, 16).cpu().tolist()
names = {0: "mma:loop", 1: "mma:p0_ok", 2: "mma:p1_ok"}
for tt in range(2):
    for k, nm in enumerate(("s_ok", "ld", "max", "bar", "exp", "p_done")):
        names[3 + 6 * tt + k] = f"sm{tt}:{nm}"
for j in range(4, 20):
    row = t[j]
    t0 = row[0]
    print(f"j {j:2d} period {t[j+1][0]-row[0]:6d}  " +
          " ".join(f"{names[s]}={row[s]-t0:+6d}" for s in (3, 4, 5, 6, 7, 8, 1, 9, 10, 11, 12, 13, 14, 2)))
