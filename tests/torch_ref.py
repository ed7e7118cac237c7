"""Plain PyTorch fp32 references for the floating-point kernels (test infra)."""
import math

import torch


def attention_ref(q, k, v, causal_diag: bool, scale=None, kv_prefix=None):
    """q [H, n, d], k/v [Hkv, nk, d] (any float dtype) -> O fp32, lse fp32.

    causal_diag: query row i sees key rows <= i (n == nk, the Diagonal mask).
    GQA: q head h reads kv head h // (H / Hkv).
    """
    qf, kf, vf = q.float(), k.float(), v.float()
    H, Hkv = qf.shape[0], kf.shape[0]
    if Hkv != H:
        kf = kf.repeat_interleave(H // Hkv, dim=0)
        vf = vf.repeat_interleave(H // Hkv, dim=0)
    d = qf.shape[-1]
    scale = scale if scale is not None else 1.0 / math.sqrt(d)
    s = torch.einsum("hid,hjd->hij", qf, kf) * scale
    if causal_diag:
        n, nk = s.shape[1], s.shape[2]
        mask = torch.ones(n, nk, dtype=torch.bool, device=s.device).tril(nk - n)
        s = s.masked_fill(~mask, float("-inf"))
    lse = torch.logsumexp(s, dim=-1)
    p = torch.softmax(s, dim=-1)
    o = torch.einsum("hij,hjd->hid", p, vf)
    return o, lse


def attention_grads_ref(q, k, v, d_out, causal_diag: bool, scale=None):
    """fp32 autograd gradients of <d_out, O>."""
    qf = q.float().detach().requires_grad_(True)
    kf = k.float().detach().requires_grad_(True)
    vf = v.float().detach().requires_grad_(True)
    o, _ = attention_ref(qf, kf, vf, causal_diag, scale)
    o.backward(d_out.float())
    return qf.grad, kf.grad, vf.grad


def rel_err(x, ref):
    """max-abs error normalised by max |ref| (SURVEY §7 parity metric)."""
    x, ref = x.float(), ref.float()
    return ((x - ref).abs().max() / ref.abs().max().clamp_min(1e-30)).item()
