"""Per-iteration timeline of the CTA-pair backward (pair 0, globaltimer ns).
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
tr = torch.zeros(64 * 16 + 8 * h * ((n + 127) // 128), dtype=torch.int64, device="cuda")
_lib.lib().da_debug_set_bwd_trace(C.c_void_p(tr.data_ptr()))
for _ in range(3):
    block_attn_backward(q, k, v, out.o, out.lse, do, MaskMode.Diagonal, d_vec=dvec, grads=g)
torch.cuda.synchronize()
t = tr[:1024].view(32, 32).cpu().tolist()
names = ["m:p_ok", "m:pread", "m:ds_ok", "m:kdq", "m:drnd", "m:doxz", "P0:s", "P0:done", "P1:s",
         "P1:done", "dS0:dp", "dS0:pld", "dS0:c2", "dS0:loop", "dS0:fnc", "dS0:done", "dS1:dp",
         "dS1:pld", "dS1:c2", "dS1:loop", "dS1:fnc", "dS1:done", "drn:dq", "drn:ld", "drn:stg",
         "m:dV_is", "m:S_is", "L:qxz", "L:doxz", "L:doy", "L:qy", "-"]
for it in range(2, 20):
    row = t[it]
    t0 = row[0]
    print(f"it {it:2d} period {t[it + 1][0] - row[0]:6d}")
    print("   " + " ".join(f"{names[s]}={row[s] - t0:+6d}" if row[s] else f"{names[s]}=  -"
                           for s in range(1, 31)))
