"""Prints the backward kernel's per-iteration clock64 timeline (CTA 0).
Needs a DA_TRACE build: DISTATTN_B200_LIB=paper_2310_03294_b200/variants/lib_trace.so"""
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2310_03294_b200 import _lib  # noqa: E402
from paper_2310_03294_b200.flashcore import (ChunkGrads, MaskMode, backward_aux,  # noqa: E402
                                             block_attn_backward, block_attn_update_final)

h, n = 32, int(sys.argv[1]) if len(sys.argv) > 1 else 16384
q, k, v, do = [(torch.rand(h, n, 128, device="cuda") * 2 - 1).to(torch.bfloat16) for _ in range(4)]
out = block_attn_update_final(q, k, v, None, MaskMode.Diagonal)
dvec = backward_aux(do, out.o)
g = ChunkGrads(torch.zeros(h, n, 128, device="cuda"), torch.empty(h, n, 128, device="cuda"),
               torch.empty(h, n, 128, device="cuda"))
tr = torch.zeros(64 * 16 + 8 * h * ((n + 127) // 128), dtype=torch.int64, device="cuda")  # + per-CTA records
_lib.lib().da_debug_set_bwd_trace(C.c_void_p(tr.data_ptr()))
for _ in range(3):
    block_attn_backward(q, k, v, out.o, out.lse, do, MaskMode.Diagonal, d_vec=dvec, grads=g)
torch.cuda.synchronize()
t = tr[:1024].view(64, 16).cpu().tolist()
names = ["mma:p_ok", "mma:ds_ok", "mma:drained", "P:s_ok", "P:done", "dS:dp_ok", "dS:p_read",
         "dS:done", "drn:dq_ok", "drn:drained", "drn:staged"]
for it in range(4, 20):
    row = t[it]
    t0 = row[0]
    print(f"it {it:2d} period {t[it + 1][0] - row[0]:6d}  " +
          " ".join(f"{names[s]}={row[s] - t0:+6d}" for s in range(1, 11)))
