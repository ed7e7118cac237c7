"""Small launches of every kernel for compute-sanitizer (tools/sanitize.sh):
forward (diagonal / full / ragged / chained accumulator / empty), merge,
finalize, backward preprocess, backward (diagonal / full ragged / GQA /
deterministic), bf16 conversion."""
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
    for kind, bwd in (("balanced", "ring"), ("balanced_split", "balanced"), ("ring", "ring")):
        shards = make_parity_shards(3, 4, 1024, 2, 128, heads_kv=1)
        run_forward(shards, kind)
        run_backward(shards, bwd)
    torch.cuda.synchronize()
    print("sanitize cases done")


if __name__ == "__main__":
    main()
