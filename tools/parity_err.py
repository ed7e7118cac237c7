"""Max relative errors of the chunk backward vs the fp32 reference (development tool).

    python tools/parity_err.py [heads] [rows]
Prints max|got-ref|/max|ref| for dq/dk/dv (causal Diagonal, MHA and GQA 4:1)
with the library at DISTATTN_B200_LIB (default: the in-tree build)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from paper_2310_03294_b200 import flashcore as F  # noqa: E402
from torch_ref import attention_grads_ref  # noqa: E402

h = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
for hkv, amp in ((h, 1.0), (max(1, h // 4), 1.0), (h, 8.0)):
    torch.manual_seed(0)
    q = ((torch.rand(h, n, 128, device="cuda") * 2 - 1) * amp).to(torch.bfloat16)
    k, v = [(torch.rand(hkv, n, 128, device="cuda") * 2 - 1).to(torch.bfloat16) for _ in range(2)]
    do = (torch.rand(h, n, 128, device="cuda") * 2 - 1).to(torch.bfloat16)
    out = F.block_attn_update_final(q, k, v, None, F.MaskMode.Diagonal)
    dvec = F.backward_aux(do, out.o)
    g = F.ChunkGrads(torch.zeros(h, n, 128, device="cuda"), torch.empty(hkv, n, 128, device="cuda"),
                     torch.empty(hkv, n, 128, device="cuda"))
    F.block_attn_backward(q, k, v, out.o, out.lse, do, F.MaskMode.Diagonal, d_vec=dvec, grads=g)
    ref = attention_grads_ref(q, k, v, do, True)
    errs = [((a - b).abs().max() / b.abs().max()).item() for a, b in zip((g.dq, g.dk, g.dv), ref)]
    print(f"h={h} hkv={hkv} n={n} amp={amp}: dq {errs[0]:.2e} dk {errs[1]:.2e} dv {errs[2]:.2e}")
