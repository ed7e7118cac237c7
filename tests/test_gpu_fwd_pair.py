"""The CTA-pair forward kernel (attn_fwd_pair_sm100.cu, tcgen05 cta_group::2).

Selected with DA_FWD_KERNEL=pair (read once per process), so these tests re-run
the forward parity suites in a child process that selects it: the kernel-level
fp32 comparisons (diagonal + finalize, full with an incoming accumulator,
ragged and GQA shapes, the chunk chain, peaky logits) and the cfg2 32K
every-element comparison, GQA 4:1 at 32K and the 64K Full chunk pair.
"""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
TESTS = Path(__file__).resolve().parent


def _run(args, timeout):
    env = dict(os.environ, DA_FWD_KERNEL="pair")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", *args],
                       cwd=TESTS.parent, env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    return r.stdout


def test_pair_forward_parity_small(cuda):
    out = _run([str(TESTS / "test_gpu_kernels.py"), "-k", "fwd or chain or peaky or host_pipeline"],
               600)
    assert " passed" in out


def test_pair_forward_parity_scale(cuda):
    out = _run([str(TESTS / "test_gpu_parity_scale.py"), "-k",
                "cfg2_32k_all_outputs or gqa_4to1 or full_mask_64k or oracle_fp64"], 900)
    assert " passed" in out
