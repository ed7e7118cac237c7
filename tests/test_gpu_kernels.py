"""GPU parity of the sm_100a chunk kernels against plain PyTorch fp32 references.

Tolerances (north_star): O/dQ/dK/dV max-abs error / max|ref| <= 2e-2,
logsumexp max-abs <= 1e-3, for bf16 inputs with fp32 accumulation.
"""
import math

import pytest
import torch

from torch_ref import attention_grads_ref, attention_ref, rel_err

pytestmark = pytest.mark.gpu

TOL = 2e-2
LSE_TOL = 1e-3


def _qkv(h, n, hkv=None, nk=None, seed=0, dev="cuda", amp=1.0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    hkv = hkv or h
    nk = nk or n
    q = (torch.rand(h, n, 128, generator=g) * 2 - 1) * amp
    k = torch.rand(hkv, nk, 128, generator=g) * 2 - 1
    v = torch.rand(hkv, nk, 128, generator=g) * 2 - 1
    return [x.to(torch.bfloat16).to(dev) for x in (q, k, v)]


def test_debug_scores_layout(cuda):
    from paper_2310_03294_b200 import _lib
    import ctypes as C
    q, k, _ = _qkv(1, 128)
    s = torch.zeros(128, 128, dtype=torch.float32, device=cuda)
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    rc = _lib.lib().da_debug_scores(C.c_void_p(q.data_ptr()), C.c_void_p(k.data_ptr()), 128,
                                    C.c_void_p(s.data_ptr()), st)
    assert rc == 0, _lib.lib().da_last_error()
    ref = q[0].float() @ k[0].float().T
    assert rel_err(s, ref) < 1e-3


@pytest.mark.parametrize("h,n", [(1, 128), (2, 256), (2, 384), (3, 200), (2, 1024)])
def test_fwd_diagonal_finalize(cuda, h, n):
    from paper_2310_03294_b200.flashcore import MaskMode, block_attn_update_final
    q, k, v = _qkv(h, n, seed=n)
    out = block_attn_update_final(q, k, v, None, MaskMode.Diagonal)
    torch.cuda.synchronize()
    o_ref, lse_ref = attention_ref(q, k, v, True)
    assert rel_err(out.o, o_ref) < TOL
    assert (out.lse - lse_ref).abs().max().item() < LSE_TOL


@pytest.mark.parametrize("h,hkv,n,nk", [(2, 2, 256, 256), (4, 1, 128, 384), (2, 2, 300, 130)])
def test_fwd_full_accumulator(cuda, h, hkv, n, nk):
    from paper_2310_03294_b200.flashcore import MaskMode, block_attn_update, finalize
    q, k, v = _qkv(h, n, hkv, nk, seed=7)
    acc = block_attn_update(q, k, v, None, MaskMode.Full)
    out = finalize(acc)
    o_ref, lse_ref = attention_ref(q, k, v, False)
    assert rel_err(out.o, o_ref) < TOL
    assert (out.lse - lse_ref).abs().max().item() < LSE_TOL


def test_fwd_chunk_chain_matches_full_causal(cuda):
    """Owner of chunk 3 absorbs kv 3 (diagonal), then kv 1, kv 2 (full), merging in-kernel."""
    from paper_2310_03294_b200.flashcore import MaskMode, block_attn_update, block_attn_update_final
    h, c = 2, 256
    q, k, v = _qkv(h, 3 * c, seed=3)
    qs, ks, vs = (x.split(c, dim=1) for x in (q, k, v))
    qs, ks, vs = [t.contiguous() for t in qs], [t.contiguous() for t in ks], [t.contiguous() for t in vs]
    acc = block_attn_update(qs[2], ks[2], vs[2], None, MaskMode.Diagonal)
    acc = block_attn_update(qs[2], ks[0], vs[0], acc, MaskMode.Full, out=acc)
    out = block_attn_update_final(qs[2], ks[1], vs[1], acc, MaskMode.Full)
    o_ref, lse_ref = attention_ref(q, k, v, True)
    assert rel_err(out.o, o_ref[:, 2 * c:]) < TOL
    assert (out.lse - lse_ref[:, 2 * c:]).abs().max().item() < LSE_TOL


def test_rescale_merge_and_identity(cuda):
    from paper_2310_03294_b200.flashcore import (AttnAccumulator, MaskMode, block_attn_update,
                                                 finalize, rescale)
    h, c = 2, 128
    q, k, v = _qkv(h, 2 * c, seed=11)
    ks, vs = k.split(c, dim=1), v.split(c, dim=1)
    a = block_attn_update(q, ks[0].contiguous(), vs[0].contiguous(), None, MaskMode.Full)
    b = block_attn_update(q, ks[1].contiguous(), vs[1].contiguous(), None, MaskMode.Full)
    m = rescale(a, b)
    out = finalize(m)
    o_ref, lse_ref = attention_ref(q, k, v, False)
    assert rel_err(out.o, o_ref) < TOL
    # a fresh accumulator is the identity (flashcore.hpp:214-217)
    fresh = AttnAccumulator.fresh(h, 2 * c)
    same = rescale(fresh, m)
    assert torch.equal(same.o, m.o) and torch.equal(same.l, m.l) and torch.equal(same.m, m.m)


@pytest.mark.parametrize("h,hkv,n,diag", [(1, 1, 128, True), (2, 2, 256, True), (2, 2, 384, True),
                                          (4, 2, 256, True), (2, 2, 256, False), (3, 3, 200, True)])
def test_bwd_chunk(cuda, h, hkv, n, diag):
    from paper_2310_03294_b200.flashcore import MaskMode, block_attn_backward
    q, k, v = _qkv(h, n, hkv, seed=100 + n)
    g = torch.Generator().manual_seed(5)
    d_out = (torch.rand(h, n, 128, generator=g) * 2 - 1).to(torch.bfloat16).to(cuda)
    o_ref, lse_ref = attention_ref(q, k, v, diag)
    out_bf = o_ref.to(torch.bfloat16)
    mask = MaskMode.Diagonal if diag else MaskMode.Full
    grads = block_attn_backward(q, k, v, out_bf, lse_ref.contiguous(), d_out, mask)
    torch.cuda.synchronize()
    dq, dk, dv = attention_grads_ref(q, k, v, d_out, diag)
    assert rel_err(grads.dv, dv) < TOL, "dv"
    assert rel_err(grads.dk, dk) < TOL, "dk"
    assert rel_err(grads.dq, dq) < TOL, "dq"


@pytest.mark.parametrize("h,hkv,n,nk", [(2, 2, 300, 130), (4, 1, 128, 384), (2, 1, 1000, 260)])
def test_bwd_full_ragged(cuda, h, hkv, n, nk):
    """Full-mask chunk pair with rows_q != rows_kv and partial tiles on both sides
    (the helper/direct tasks of uneven shards), GQA groups summed into dK/dV."""
    from paper_2310_03294_b200.flashcore import MaskMode, block_attn_backward
    q, k, v = _qkv(h, n, hkv, nk, seed=n + nk)
    d_out = _qkv(h, n, seed=n * 3)[0]
    o_ref, lse_ref = attention_ref(q, k, v, False)
    grads = block_attn_backward(q, k, v, o_ref.to(torch.bfloat16), lse_ref.contiguous(), d_out,
                                MaskMode.Full)
    torch.cuda.synchronize()
    dq, dk, dv = attention_grads_ref(q, k, v, d_out, False)
    assert rel_err(grads.dv, dv) < TOL, "dv"
    assert rel_err(grads.dk, dk) < TOL, "dk"
    assert rel_err(grads.dq, dq) < TOL, "dq"


@pytest.mark.parametrize("amp", [8.0, 24.0])
def test_peaky_fwd_bwd_chunk_chain(cuda, amp):
    """SURVEY §8(d) "peaky" set: q scaled so single keys dominate rows and the
    running max moves between chunks; the chain diag(kv2) -> full(kv0) ->
    full(kv1) + finalize and the backward over all three pairs match fp32."""
    from paper_2310_03294_b200.flashcore import (MaskMode, block_attn_backward, block_attn_update,
                                                 block_attn_update_final)
    h, c = 2, 256
    q, k, v = _qkv(h, 3 * c, seed=int(amp), amp=amp)
    d_out = _qkv(h, 3 * c, seed=99)[0]
    sl = [slice(i * c, (i + 1) * c) for i in range(3)]
    qs, ks, vs = ([x[:, s_].contiguous() for s_ in sl] for x in (q, k, v))
    acc = block_attn_update(qs[2], ks[2], vs[2], None, MaskMode.Diagonal)
    acc = block_attn_update(qs[2], ks[0], vs[0], acc, MaskMode.Full, out=acc)
    out = block_attn_update_final(qs[2], ks[1], vs[1], acc, MaskMode.Full)
    o_ref, lse_ref = attention_ref(q, k, v, True)
    assert rel_err(out.o, o_ref[:, sl[2]]) < TOL
    assert (out.lse - lse_ref[:, sl[2]]).abs().max().item() < LSE_TOL
    # backward of the last query chunk: dq summed over its three kv chunks
    do2 = d_out[:, sl[2]].contiguous()
    lse2 = lse_ref[:, sl[2]].contiguous()
    o2 = o_ref[:, sl[2]].to(torch.bfloat16)
    g = block_attn_backward(qs[2], ks[2], vs[2], o2, lse2, do2, MaskMode.Diagonal)
    dks, dvs = [g.dk], [g.dv]
    for j in (0, 1):
        gj = block_attn_backward(qs[2], ks[j], vs[j], o2, lse2, do2, MaskMode.Full)
        g.dq += gj.dq
        dks.append(gj.dk)
        dvs.append(gj.dv)
    torch.cuda.synchronize()
    d_full = torch.zeros_like(d_out)
    d_full[:, sl[2]] = do2
    dq, dk, dv = attention_grads_ref(q, k, v, d_full, True)
    assert rel_err(g.dq, dq[:, sl[2]]) < TOL, "dq"
    assert rel_err(dks[0], dk[:, sl[2]]) < TOL and rel_err(dvs[0], dv[:, sl[2]]) < TOL
    assert rel_err(dks[1], dk[:, sl[0]]) < TOL and rel_err(dvs[1], dv[:, sl[0]]) < TOL
    assert rel_err(dks[2], dk[:, sl[1]]) < TOL and rel_err(dvs[2], dv[:, sl[1]]) < TOL


@pytest.mark.parametrize("h,n,hpg", [(4, 1024, 2), (6, 700, 3), (2, 256, 2)])
def test_host_pipeline_matches_direct_calls(cuda, h, n, hpg):
    """pipeline.HostAttention (the C++ host pipeline, da_pipeline_*: pinned host
    in/out, per-head-group overlap) computes
    the same step as the ungrouped device calls: dK/dV bit-exact (deterministic
    in-CTA reductions), dQ within one bf16 ulp (fp32 reduction order differs)."""
    from paper_2310_03294_b200 import flashcore as F
    from paper_2310_03294_b200.pipeline import HostAttention
    q, k, v = _qkv(h, n, seed=h * n)
    do = _qkv(h, n, seed=h * n + 1)[0]
    out = F.block_attn_update_final(q, k, v, None, F.MaskMode.Diagonal)
    g = F.block_attn_backward(q, k, v, out.o, out.lse, do, F.MaskMode.Diagonal)
    ref = [x.to(torch.bfloat16).cpu() for x in (g.dq, g.dk, g.dv)]
    host_in = [x.cpu().pin_memory() for x in (q, k, v, do)]
    host_out = [torch.empty(h, n, 128, dtype=torch.bfloat16).pin_memory() for _ in range(3)]
    ha = HostAttention(h, n, heads_per_group=hpg)
    for _ in range(2):  # second call reuses the device buffers
        ha(*host_in, *host_out)
    assert torch.equal(host_out[1], ref[1]) and torch.equal(host_out[2], ref[2])
    assert rel_err(host_out[0].float(), ref[0].float()) < 1e-2
    o_ref, _ = attention_ref(q, k, v, True)
    assert rel_err(ha.outputs()[0], o_ref) < TOL


def test_host_pipeline_back_to_back_async_calls(cuda):
    """Consecutive sync=False calls overlap (call i+1's copies of group g wait
    only for call i's group g); each call's outputs are its own inputs' grads."""
    from paper_2310_03294_b200 import flashcore as F
    from paper_2310_03294_b200.pipeline import HostAttention
    h, n = 4, 512
    ha = HostAttention(h, n, heads_per_group=1)
    steps = []
    for s_ in range(3):
        q, k, v = _qkv(h, n, seed=50 + s_)
        do = _qkv(h, n, seed=60 + s_)[0]
        host_in = [x.cpu().pin_memory() for x in (q, k, v, do)]
        host_out = [torch.empty(h, n, 128, dtype=torch.bfloat16).pin_memory() for _ in range(3)]
        ha(*host_in, *host_out, sync=False)
        steps.append(((q, k, v, do), host_out, host_in))
    ha.join()
    torch.cuda.synchronize()
    ha.check()
    for (q, k, v, do), host_out, _ in steps:
        out = F.block_attn_update_final(q, k, v, None, F.MaskMode.Diagonal)
        g = F.block_attn_backward(q, k, v, out.o, out.lse, do, F.MaskMode.Diagonal)
        assert torch.equal(host_out[1], g.dk.to(torch.bfloat16).cpu())
        assert torch.equal(host_out[2], g.dv.to(torch.bfloat16).cpu())
        assert rel_err(host_out[0].float(), g.dq.to(torch.bfloat16).cpu().float()) < 1e-2


def test_host_pipeline_degenerate_rows_raise(cuda):
    """A finalize over a row that attended to no key raises DegenerateRowError
    (flashcore.hpp:233-235) even with the deferred (sync-free) flag."""
    from paper_2310_03294_b200 import flashcore as F
    from paper_2310_03294_b200.errors import DegenerateRowError
    q, k, v = _qkv(2, 128, nk=128)
    flag = torch.zeros(1, dtype=torch.int32, device=cuda)
    F.block_attn_update_final(q, k[:, :0].contiguous(), v[:, :0].contiguous(), None,
                              F.MaskMode.Full, degenerate_flag=flag)
    with pytest.raises(DegenerateRowError):
        F.check_degenerate(flag)


@pytest.mark.parametrize("h,hkv,n,diag", [(2, 2, 1024, True), (4, 2, 640, True), (2, 2, 384, False),
                                          (1, 1, 40000, True)])
def test_bwd_deterministic_dq_is_bitwise_reproducible(cuda, h, hkv, n, diag):
    """deterministic=True orders the fp32 dq partials (descending kv tile), so
    repeated launches give identical bits; the values match the default
    (unordered) reduction to fp32 rounding and the fp32 reference."""
    from paper_2310_03294_b200.flashcore import MaskMode, block_attn_backward
    q, k, v = _qkv(h, n, hkv, seed=7 + n)
    d_out = _qkv(h, n, hkv, seed=8 + n)[0]
    mask = MaskMode.Diagonal if diag else MaskMode.Full
    if n <= 2048:
        o_ref, lse_ref = attention_ref(q, k, v, diag)
    else:  # long single head: the kernel's own forward supplies O / LSE
        from paper_2310_03294_b200.flashcore import block_attn_update_final
        fo = block_attn_update_final(q, k, v, None, mask)
        o_ref, lse_ref = fo.o.float(), fo.lse
    out_bf = o_ref.to(torch.bfloat16)
    runs = [block_attn_backward(q, k, v, out_bf, lse_ref.contiguous(), d_out, mask,
                                deterministic=True) for _ in range(3)]
    fast = block_attn_backward(q, k, v, out_bf, lse_ref.contiguous(), d_out, mask)
    torch.cuda.synchronize()
    for g in runs[1:]:
        assert torch.equal(g.dq, runs[0].dq) and torch.equal(g.dk, runs[0].dk) and \
            torch.equal(g.dv, runs[0].dv)
    assert rel_err(runs[0].dq, fast.dq) < 1e-5
    assert torch.equal(runs[0].dk, fast.dk) and torch.equal(runs[0].dv, fast.dv)
    if n <= 2048:
        dq, dk, dv = attention_grads_ref(q, k, v, d_out, diag)
        assert rel_err(runs[0].dq, dq) < TOL


def test_shape_errors_before_the_c_abi(cuda):
    """The reference's operand checks (flashcore.hpp:143-147, 284-293) raise
    ShapeError before any pointer reaches a kernel."""
    from paper_2310_03294_b200 import flashcore as F
    from paper_2310_03294_b200.errors import ShapeError
    q, k, v = _qkv(2, 256)
    with pytest.raises(ShapeError, match="k/v row mismatch"):
        F.block_attn_update(q, k, v[:, :128].contiguous(), None, F.MaskMode.Full)
    with pytest.raises(ShapeError, match="hidden dims disagree"):
        F.block_attn_update(q, k[..., :64].contiguous(), v[..., :64].contiguous(), None,
                            F.MaskMode.Full)
    acc = F.AttnAccumulator.fresh(2, 128)
    with pytest.raises(ShapeError, match="accumulator shape mismatch"):
        F.block_attn_update(q, k, v, acc, F.MaskMode.Full)
    out = F.block_attn_update_final(q, k, v, None, F.MaskMode.Diagonal)
    do = _qkv(2, 256, seed=3)[0]
    with pytest.raises(ShapeError, match="logsumexp length mismatch"):
        F.block_attn_backward(q, k, v, out.o, out.lse[:, :100].contiguous(), do, F.MaskMode.Diagonal)
    with pytest.raises(ShapeError, match="upstream grad shape mismatch"):
        F.block_attn_backward(q, k, v, out.o, out.lse, do[:1].contiguous(), F.MaskMode.Diagonal)
    with pytest.raises(ShapeError, match="output shape mismatch"):
        F.block_attn_backward(q, k, v, out.o[:, :128].contiguous(), out.lse, do, F.MaskMode.Diagonal)
    bad = F.ChunkGrads(torch.zeros(2, 256, 128, device=cuda), torch.zeros(2, 128, 128, device=cuda),
                       torch.zeros(2, 256, 128, device=cuda))
    with pytest.raises(ShapeError, match="dk accumulator shape mismatch"):
        F.block_attn_backward(q, k, v, out.o, out.lse, do, F.MaskMode.Diagonal, grads=bad)


def test_deterministic_backward_on_two_streams(cuda):
    """Deterministic launches in flight on two streams use separate semaphore
    workspaces (one per stream): both finish and agree bitwise."""
    from paper_2310_03294_b200 import flashcore as F
    q, k, v = _qkv(2, 2048, seed=5)
    do = _qkv(2, 2048, seed=6)[0]
    out = F.block_attn_update_final(q, k, v, None, F.MaskMode.Diagonal)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = []
    for s in (s1, s2, s1, s2):
        with torch.cuda.stream(s):
            res.append(F.block_attn_backward(q, k, v, out.o, out.lse, do, F.MaskMode.Diagonal,
                                             deterministic=True, stream=s))
    torch.cuda.synchronize()
    for g in res[1:]:
        assert torch.equal(g.dq, res[0].dq) and torch.equal(g.dk, res[0].dk)


def test_host_pipeline_gqa(cuda):
    """The C++ host pipeline with GQA (8 q heads / 2 kv heads, groups of one kv
    group): dK/dV summed over each group, equal to the device calls."""
    from paper_2310_03294_b200 import flashcore as F
    from paper_2310_03294_b200.pipeline import HostAttention
    h, hk, n = 8, 2, 640
    q, k, v = _qkv(h, n, hk, seed=77)
    do = _qkv(h, n, seed=78)[0]
    out = F.block_attn_update_final(q, k, v, None, F.MaskMode.Diagonal)
    g = F.block_attn_backward(q, k, v, out.o, out.lse, do, F.MaskMode.Diagonal)
    host_in = [x.cpu().pin_memory() for x in (q, k, v, do)]
    host_out = [torch.empty(*x.shape, dtype=torch.bfloat16).pin_memory() for x in (q, k, v)]
    ha = HostAttention(h, n, heads_per_group=4, heads_kv=hk)
    ha(*host_in, *host_out)
    assert torch.equal(host_out[1], g.dk.to(torch.bfloat16).cpu())
    assert torch.equal(host_out[2], g.dv.to(torch.bfloat16).cpu())
    assert rel_err(host_out[0].float(), g.dq.to(torch.bfloat16).cpu().float()) < 1e-2
    with pytest.raises(Exception):
        HostAttention(h, n, heads_per_group=2, heads_kv=hk)  # splits a kv group
