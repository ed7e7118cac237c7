"""The CTA-pair backward kernel (attn_bwd_pair_sm100.cu, tcgen05 cta_group::2).

It is an opt-in experiment (DA_BWD_KERNEL=pair, read once per process): it is
correct but measured slower than the single-CTA kernel, so the
product path does not use it. These tests keep its correctness claim honest by
re-running the backward parity suites in a child process that selects it:
the kernel-level fp32 comparisons (diagonal, full, ragged, GQA, peaky) and the
cfg2 32K every-element comparison.
"""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
TESTS = Path(__file__).resolve().parent


def _run(args, timeout):
    env = dict(os.environ, DA_BWD_KERNEL="pair")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", *args],
                       cwd=TESTS.parent, env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    return r.stdout


def test_pair_kernel_backward_parity_small(cuda):
    out = _run([str(TESTS / "test_gpu_kernels.py"), "-k", "bwd_chunk or bwd_full_ragged or peaky"],
               600)
    assert " passed" in out


def test_pair_kernel_cfg2_32k_all_outputs(cuda):
    out = _run([str(TESTS / "test_gpu_parity_scale.py"), "-k", "cfg2_32k_all_outputs or gqa_4to1"],
               900)
    assert " passed" in out
