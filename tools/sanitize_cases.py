"""Small launches of every kernel for compute-sanitizer (tools/sanitize.sh):
forward (diagonal / full / ragged / chained accumulator / empty), merge,
finalize, backward preprocess, backward (diagonal / full ragged / GQA /
deterministic), bf16 conversion, the P-worker executor (incl. the split
backward), the host pipeline and the host-buffer entry points. With
DA_FWD_KERNEL=pair every forward runs on the CTA-pair kernel."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2310_03294_b200 import flashcore as F  # noqa: E402


def qkv(h, n, hkv=None, nk=None, seed=0):
    g = torch.Generator().manual_seed(seed)
    hkv, nk = hkv or h, nk or n
    mk = lambda hh, rr: ((torch.rand(hh, rr, 128, generator=g) * 2 - 1).to(torch.bfloat16).cuda())
    return mk(h, n), mk(hkv, nk), mk(hkv, nk)


def main():
    q, k, v = qkv(2, 384)
    out = F.block_attn_update_final(q, k, v, None, F.MaskMode.Diagonal)
    q2, k2, v2 = qkv(2, 300, 1, 130, seed=1)
    acc = F.block_attn_update(q2, k2, v2, None, F.MaskMode.Full)
    acc = F.block_attn_update(q2, k2, v2, acc, F.MaskMode.Full, out=acc)
    b = F.block_attn_update(q2, k2, v2, None, F.MaskMode.Full)
    m = F.rescale(acc, b)
    F.finalize(m)
    F.block_attn_update(q2, k2[:, :0].contiguous(), v2[:, :0].contiguous(), acc, F.MaskMode.Empty)
    do = qkv(2, 384, seed=2)[0]
    dvec = F.backward_aux(do, out.o)
    F.block_attn_backward(q, k, v, out.o, out.lse, do, F.MaskMode.Diagonal, d_vec=dvec)
    F.block_attn_backward(q, k, v, out.o, out.lse, do, F.MaskMode.Diagonal, d_vec=dvec,
                          deterministic=True)
    q3, k3, v3 = qkv(4, 256, 2, 384, seed=3)
    o3 = F.finalize(F.block_attn_update(q3, k3, v3, None, F.MaskMode.Full))
    do3 = qkv(4, 256, seed=4)[0]
    g3 = F.block_attn_backward(q3, k3, v3, o3.o, o3.lse, do3, F.MaskMode.Full)
    F.block_attn_backward(q3, k3, v3, o3.o, o3.lse, do3, F.MaskMode.Full, grads=g3,
                          accumulate_kv=True)
    # the native P-worker executor (schedules, message buffers, merges, split halves)
    from paper_2310_03294_b200.runtime import make_parity_shards, run_backward, run_forward
    for kind, bwd in (("balanced", "ring"), ("balanced_split", "balanced"), ("ring", "ring"),
                      ("balanced_split", "balanced_split")):
        shards = make_parity_shards(3, 4, 1024, 2, 128, heads_kv=1)
        run_forward(shards, kind)
        run_backward(shards, bwd)
    # the C++ host pipeline (pinned host in / out, per-group streams, GQA)
    from paper_2310_03294_b200.pipeline import HostAttention
    hq, hk, hv = (t.cpu().pin_memory() for t in qkv(4, 256, 2, seed=5))
    hdo = qkv(4, 256, seed=6)[0].cpu().pin_memory()
    outs = [torch.empty_like(t).pin_memory() for t in (hq, hk, hv)]
    ha = HostAttention(4, 256, heads_per_group=2, heads_kv=2)
    for _ in range(2):
        ha(hq, hk, hv, hdo, *outs, sync=False)
    ha.check()
    # the host-buffer (fp64) entry points behind the drop-in flashcore.hpp
    import ctypes as C
    import numpy as np
    from paper_2310_03294_b200 import _lib
    lib = _lib.lib()
    r = np.random.default_rng(0)
    qh, kh, vh, doh = (np.ascontiguousarray(r.uniform(-1, 1, (256, 128))) for _ in range(4))
    o, m, l = np.zeros((256, 128)), np.full(256, -np.inf), np.zeros(256)
    ptr = lambda a: C.c_void_p(a.ctypes.data)  # noqa: E731
    lib.da_host_attn_update(ptr(qh), 256, ptr(kh), ptr(vh), 256, 128, ptr(o), ptr(m), ptr(l), 0,
                            128 ** -0.5)
    out, lse = np.empty((256, 128)), np.empty(256)
    lib.da_host_attn_finalize(ptr(o), ptr(m), ptr(l), 256, 128, ptr(out), ptr(lse))
    g = [np.empty((256, 128)) for _ in range(3)]
    lib.da_host_attn_backward(ptr(qh), 256, ptr(kh), ptr(vh), 256, 128, ptr(out), ptr(lse),
                              ptr(doh), 0, 128 ** -0.5, *(ptr(x) for x in g))
    torch.cuda.synchronize()
    print("sanitize cases done")


if __name__ == "__main__":
    main()
