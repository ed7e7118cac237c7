"""Per-CTA timeline of one backward (or forward: 3rd arg "fwd") launch (DA_TRACE
build): SM occupancy, clocks per iteration including CTA prologue/epilogue, tail.
DISTATTN_B200_LIB=paper_2310_03294_b200/variants/lib_trace.so python tools/trace_ctas.py [n] [h] [fwd|bwd] [h_kv]"""
import ctypes as C
import sys
from collections import defaultdict
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2310_03294_b200 import _lib  # noqa: E402
from paper_2310_03294_b200.flashcore import (ChunkGrads, MaskMode, backward_aux,  # noqa: E402
                                             block_attn_backward, block_attn_update_final)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
h = int(sys.argv[2]) if len(sys.argv) > 2 else 32
hkv = int(sys.argv[4]) if len(sys.argv) > 4 else h
det = len(sys.argv) > 5 and sys.argv[5] == "det"  # deterministic dQ order
q, do = [(torch.rand(h, n, 128, device="cuda") * 2 - 1).to(torch.bfloat16) for _ in range(2)]
k, v = [(torch.rand(hkv, n, 128, device="cuda") * 2 - 1).to(torch.bfloat16) for _ in range(2)]
out = block_attn_update_final(q, k, v, None, MaskMode.Diagonal)
dvec = backward_aux(do, out.o)
g = ChunkGrads(torch.zeros(h, n, 128, device="cuda"), torch.empty(hkv, n, 128, device="cuda"),
               torch.empty(hkv, n, 128, device="cuda"))
fwd = len(sys.argv) > 3 and sys.argv[3] == "fwd"
n_cta = h * ((n + 127) // 128) // 2 if fwd else hkv * ((n + 127) // 128)
tr = torch.zeros(1024 + 8 * n_cta, dtype=torch.int64, device="cuda")
if fwd:
    _lib.lib().da_debug_set_fwd_trace(C.c_void_p(tr.data_ptr()))
    for _ in range(3):
        block_attn_update_final(q, k, v, None, MaskMode.Diagonal)
else:
    _lib.lib().da_debug_set_bwd_trace(C.c_void_p(tr.data_ptr()))
    for _ in range(3):
        block_attn_backward(q, k, v, out.o, out.lse, do, MaskMode.Diagonal, d_vec=dvec, grads=g,
                            deterministic=det)
torch.cuda.synchronize()
rec = tr[1024:].view(n_cta, 8).cpu().tolist()
t0 = min(r[0] for r in rec)
t1 = max(r[1] for r in rec)
span_ns = t1 - t0
per_sm = defaultdict(list)
for r in rec:
    per_sm[r[4]].append(r)
busy = [sum(x[1] - x[0] for x in v_) for v_ in per_sm.values()]
ends = sorted(max(x[1] for x in v_) - t0 for v_ in per_sm.values())
clk = sum(r[3] - r[2] for r in rec)
its = sum(r[5] for r in rec)
ns_total = sum(r[1] - r[0] for r in rec)
print(f"ctas {n_cta} sms {len(per_sm)} span {span_ns / 1e6:.3f} ms")
print(f"mean SM busy {sum(busy) / len(busy) / span_ns:.4f} of span; first SM idle at "
      f"{ends[0] / 1e6:.3f} ms, median {ends[len(ends) // 2] / 1e6:.3f}")
print(f"clk per iteration (incl. CTA overheads) {clk / its:.0f}; effective clock "
      f"{clk / ns_total * 1e3:.0f} MHz")
short = sorted(rec, key=lambda r: r[5])[:3]
for r in short:
    print(f"  smallest CTA: {r[5]} it, {r[3] - r[2]} clk -> {(r[3] - r[2]) / max(r[5], 1):.0f} clk/it")
big = sorted(rec, key=lambda r: -r[5])[:3]
for r in big:
    print(f"  largest CTA: {r[5]} it, {r[3] - r[2]} clk -> {(r[3] - r[2]) / max(r[5], 1):.0f} clk/it")
# per-SM body rate (clk per iteration over the SM's CTAs, first-MMA to last
# commit): is the spread between CTAs a property of the SM (die, TPC) or of
# the CTA's position in the grid?
rate = {}
for sm, v_ in per_sm.items():
    it_ = sum(x[5] for x in v_)
    if it_:
        # backward: first MMA -> last commit; forward: whole CTA (no MMA stamps)
        rate[sm] = sum((x[3] - x[2]) if fwd else (x[7] - x[6]) for x in v_) / it_
sms = sorted(rate)
half = len(sms) // 2
lo = [rate[s] for s in sms[:half]]
hi = [rate[s] for s in sms[half:]]
print(f"per-SM body clk/it: min {min(rate.values()):.0f} median {sorted(rate.values())[len(rate) // 2]:.0f} "
      f"max {max(rate.values()):.0f}; SM ids < {sms[half]}: mean {sum(lo) / len(lo):.0f}, "
      f">= : mean {sum(hi) / len(hi):.0f}")
tpc = defaultdict(list)
for s in sms:
    tpc[s // 2].append(rate[s])
pair_gap = sorted(abs(v_[0] - v_[1]) for v_ in tpc.values() if len(v_) == 2)
print(f"|rate(SM 2t) - rate(SM 2t+1)| median {pair_gap[len(pair_gap) // 2]:.0f} clk/it")
slow = sorted(rate, key=lambda s: -rate[s])[:12]
print("slowest SMs:", [(s, round(rate[s])) for s in slow])
mhz = {sm: sum(x[3] - x[2] for x in v_) / sum(x[1] - x[0] for x in v_) * 1e3
       for sm, v_ in per_sm.items()}
nsit = {sm: sum(x[1] - x[0] for x in v_) / max(1, sum(x[5] for x in v_)) for sm, v_ in per_sm.items()}
fast = [s for s in sms if rate[s] < sorted(rate.values())[len(rate) // 4]]
slow_ = [s for s in sms if rate[s] >= sorted(rate.values())[len(rate) // 2]]
print(f"SM clock (clk64 / globaltimer): fast-quartile SMs {sum(mhz[s] for s in fast) / len(fast):.0f} MHz, "
      f"upper-half SMs {sum(mhz[s] for s in slow_) / len(slow_):.0f} MHz; ns per iteration: "
      f"{sum(nsit[s] for s in fast) / len(fast):.0f} vs {sum(nsit[s] for s in slow_) / len(slow_):.0f}")
print("per-SM body clk/it by SM id:")
print(" ".join(f"{s}:{round(rate[s])}" for s in sms))
if fwd:
    sys.exit(0)
pro = sorted(r[6] - r[2] for r in rec)
epi = sorted(r[3] - r[7] for r in rec)
body = sum(r[7] - r[6] for r in rec)
print(f"prologue (start -> first MMA) median {pro[len(pro) // 2]} clk, epilogue (last commit -> end) "
      f"median {epi[len(epi) // 2]} clk; body {body / its:.0f} clk/it; overhead share "
      f"{(sum(pro) + sum(epi)) / clk:.3f}")
one = [r for r in rec if r[5] == 1]
if one:
    print(f"1-iteration CTAs: body {sum(r[7] - r[6] for r in one) / len(one):.0f} clk")
# gaps between consecutive CTAs on one SM (launch latency)
gaps = []
for v_ in per_sm.values():
    v_ = sorted(v_)
    gaps += [b[0] - a[1] for a, b in zip(v_, v_[1:])]
gaps.sort()
print(f"CTA-to-CTA gap on an SM: median {gaps[len(gaps) // 2]} ns, p90 {gaps[int(len(gaps) * .9)]} ns, "
      f"total {sum(gaps) / len(per_sm) / 1e6:.3f} ms per SM")
