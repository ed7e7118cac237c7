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


def _kv_for(h, H, Hkv):
    return h // (H // Hkv)


@torch.no_grad()
def chunked_attention_fwd(q, k, v, causal: bool, scale=None, block=2048):
    """Exact fp32 (no TF32) forward over query blocks, for long sequences.

    q [H, n, d], k/v [Hkv, nk, d]; causal = the Diagonal mask (n == nk).
    Returns O fp32 [H, n, d], lse fp32 [H, n]. Each query block only reads the
    keys it can see, so memory is O(block * nk) per head."""
    H, n, d = q.shape
    Hkv, nk, _ = k.shape
    scale = scale if scale is not None else 1.0 / math.sqrt(d)
    o = torch.empty(H, n, d, dtype=torch.float32, device=q.device)
    lse = torch.empty(H, n, dtype=torch.float32, device=q.device)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        for h in range(H):
            kh, vh = k[_kv_for(h, H, Hkv)].float(), v[_kv_for(h, H, Hkv)].float()
            for i0 in range(0, n, block):
                i1 = min(n, i0 + block)
                kend = i1 if causal else nk
                s = (q[h, i0:i1].float() @ kh[:kend].T) * scale
                if causal:
                    r = torch.arange(i0, i1, device=q.device)[:, None]
                    c = torch.arange(kend, device=q.device)[None, :]
                    s.masked_fill_(c > r, float("-inf"))
                l_ = torch.logsumexp(s, -1)
                lse[h, i0:i1] = l_
                o[h, i0:i1] = torch.exp(s - l_[:, None]) @ vh[:kend]
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return o, lse


@torch.no_grad()
def chunked_attention_bwd(q, k, v, o, lse, d_out, causal: bool, scale=None, block=2048):
    """Exact fp32 gradients (no TF32) of <d_out, O> given the forward's O / lse,
    restating flashcore.hpp:269-337 blockwise: P = exp(scale qk^T - lse),
    dV += P^T dO, dS = P (dO V^T - D), dQ += scale dS K, dK += scale dS^T Q,
    D = rowsum(dO * O). GQA groups are summed into dK/dV."""
    H, n, d = q.shape
    Hkv, nk, _ = k.shape
    scale = scale if scale is not None else 1.0 / math.sqrt(d)
    dq = torch.zeros(H, n, d, dtype=torch.float32, device=q.device)
    dk = torch.zeros(Hkv, nk, d, dtype=torch.float32, device=q.device)
    dv = torch.zeros(Hkv, nk, d, dtype=torch.float32, device=q.device)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        for h in range(H):
            g = _kv_for(h, H, Hkv)
            kh, vh = k[g].float(), v[g].float()
            D = (d_out[h].float() * o[h].float()).sum(-1)
            for i0 in range(0, n, block):
                i1 = min(n, i0 + block)
                kend = i1 if causal else nk
                qb, dob = q[h, i0:i1].float(), d_out[h, i0:i1].float()
                s = (qb @ kh[:kend].T) * scale
                if causal:
                    r = torch.arange(i0, i1, device=q.device)[:, None]
                    c = torch.arange(kend, device=q.device)[None, :]
                    s.masked_fill_(c > r, float("-inf"))
                p = torch.exp(s - lse[h, i0:i1, None].float())
                dv[g, :kend] += p.T @ dob
                ds = p * (dob @ vh[:kend].T - D[i0:i1, None])
                dq[h, i0:i1] = (ds @ kh[:kend]) * scale
                dk[g, :kend] += (ds.T @ qb) * scale
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return dq, dk, dv


@torch.no_grad()
def sampled_attention_bwd(q, k, v, o, lse, d_out, causal: bool, q_rows, kv_rows, scale=None):
    """Exact fp32 dQ at query rows `q_rows` and dK/dV at key rows `kv_rows`
    (index tensors), single head pair q [n, d], k/v [nk, d] (GQA: call per
    query head and sum dK/dV). Used where a full fp32 backward is too slow."""
    n, d = q.shape
    nk = k.shape[0]
    scale = scale if scale is not None else 1.0 / math.sqrt(d)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        qf, kf, vf, dof = q.float(), k.float(), v.float(), d_out.float()
        D = (dof * o.float()).sum(-1)
        # dq rows: scores of the sampled query rows against every key
        s = (qf[q_rows] @ kf.T) * scale
        if causal:
            s.masked_fill_(torch.arange(nk, device=q.device)[None, :] > q_rows[:, None], float("-inf"))
        p = torch.exp(s - lse[q_rows, None].float())
        ds = p * (dof[q_rows] @ vf.T - D[q_rows, None])
        dq = (ds @ kf) * scale
        # dk / dv rows: every query row against the sampled keys
        s = (qf @ kf[kv_rows].T) * scale
        if causal:
            s.masked_fill_(kv_rows[None, :] > torch.arange(n, device=q.device)[:, None], float("-inf"))
        p = torch.exp(s - lse[:, None].float())
        dv = p.T @ dof
        ds = p * (dof @ vf[kv_rows].T - D[:, None])
        dk = (ds.T @ qf) * scale
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return dq, dk, dv
