"""Quick device timing of the chunk kernels (development probe, not the bench)."""
import math
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2310_03294_b200.flashcore import MaskMode, block_attn_backward, block_attn_update_final, backward_aux  # noqa


def timeit(fn, iters=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    h = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
    hkv = int(sys.argv[3]) if len(sys.argv) > 3 else h
    mask = MaskMode.Full if len(sys.argv) > 4 and sys.argv[4] == "full" else MaskMode.Diagonal
    causal = 1 if mask == MaskMode.Diagonal else 2  # a full chunk pair does twice the causal work
    torch.manual_seed(0)
    q = (torch.rand(h, n, 128, device="cuda") * 2 - 1).to(torch.bfloat16)
    k, v = [(torch.rand(hkv, n, 128, device="cuda") * 2 - 1).to(torch.bfloat16) for _ in range(2)]
    fl_fwd = 2 * n * n * 128 * h * causal  # causal: 4*n^2*d*h/2
    fl_bwd = 5 * n * n * 128 * h * causal
    out = block_attn_update_final(q, k, v, None, mask)
    t_fwd = timeit(lambda: block_attn_update_final(q, k, v, None, mask))
    print(f"fwd  H={h}/{hkv} N={n}: {t_fwd:.3f} ms  {fl_fwd / t_fwd / 1e9:.1f} TFLOP/s", flush=True)
    d_out = (torch.rand_like(out.o, dtype=torch.float32) * 2 - 1).to(torch.bfloat16)
    dvec = backward_aux(d_out, out.o)
    from paper_2310_03294_b200.flashcore import ChunkGrads
    grads = ChunkGrads(torch.zeros(h, n, 128, device="cuda"), torch.empty(hkv, n, 128, device="cuda"),
                       torch.empty(hkv, n, 128, device="cuda"))
    def bwd():
        block_attn_backward(q, k, v, out.o, out.lse, d_out, mask, d_vec=dvec, grads=grads)
    t_bwd = timeit(bwd)
    print(f"bwd  H={h} N={n}: {t_bwd:.3f} ms  {fl_bwd / t_bwd / 1e9:.1f} TFLOP/s", flush=True)

    def bwd_det():
        block_attn_backward(q, k, v, out.o, out.lse, d_out, mask, d_vec=dvec, grads=grads,
                            deterministic=True)
    t_det = timeit(bwd_det)
    print(f"bwd (deterministic dq) H={h} N={n}: {t_det:.3f} ms  {fl_bwd / t_det / 1e9:.1f} TFLOP/s",
          flush=True)
    print(f"fwd+bwd: {t_fwd + t_bwd:.3f} ms  {(fl_fwd + fl_bwd) / (t_fwd + t_bwd) / 1e9:.1f} TFLOP/s")


if __name__ == "__main__":
    main()
