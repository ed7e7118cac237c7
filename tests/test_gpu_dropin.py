"""The signature-level drop-in (include/distattn/flashcore.hpp) under the
reference's OWN call sites.

oracle/_ref/dropin_driver is oracle/ref_driver.cpp plus the unmodified
reference runtime.cpp / schedule.cpp / ckptplan.cpp / analyzer.cpp, compiled
with this repository's include/ first on the path (oracle/Makefile), so every
block_attn_update / rescale / finalize / block_attn_backward the reference
runtime issues (runtime.cpp:286-328, 605-716; ckptplan.cpp:146-155, 198-206)
runs on the sm_100a kernels through the C ABI host entry points. Its outputs
are compared with oracle/_ref/ref_driver — the same driver on the reference's
own fp64 flashcore.hpp — on identical bf16-rounded inputs.
"""
import json
import subprocess
import tempfile
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

TOL = 2e-2
LSE_TOL = 1e-3


def _need_drivers():
    if not (O.DROPIN_DRIVER.exists() and O.REF_DRIVER.exists()):
        pytest.fail("oracle/_ref/{ref,dropin}_driver missing: build them with `make -C oracle ref` "
                    "where /root/reference exists (they travel prebuilt)")


def _rel(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


@pytest.mark.parametrize("schedule", ["balanced", "ring"])
def test_reference_runtime_on_b200_kernels_cfg1(cuda, schedule):
    """BASELINE configs[0] (seq 4096, d=128, P=4, one head) through the
    reference's run_forward / run_backward with our kernels underneath: the
    outputs match the unmodified reference; the stepper and the concurrent
    executor (one thread + stream per worker, overlap on) give identical bits,
    as the reference guarantees (runtime.hpp:7-9); counters are the reference's."""
    _need_drivers()
    got, gmeta = O.ref_run(4096, 4, 1, 128, 0, schedule, True, driver=O.DROPIN_DRIVER,
                           executor="both")
    ref, rmeta = O.ref_run(4096, 4, 1, 128, 0, schedule, True)
    for name in ("q", "k", "v", "d_out"):
        assert np.array_equal(got[name], ref[name]), f"inputs differ: {name}"
    assert gmeta["heads"][0]["executors_bitwise_equal"] is True
    for key in ("fwd_counters", "bwd_counters", "fwd_kernel_calls", "bwd_kernel_calls"):
        assert gmeta["heads"][0][key] == rmeta["heads"][0][key], key
    assert _rel(got["out"], ref["out"]) < TOL
    assert np.abs(got["lse"] - ref["lse"]).max() < LSE_TOL
    for name in ("dq", "dk", "dv"):
        assert _rel(got[name], ref[name]) < TOL, name


def test_reference_checkpoint_plans_on_b200_kernels(cuda):
    """The reference's checkpointed layer pipeline (ckptplan.cpp) at d = 128:
    recompute counts equal the reference's, the three plans' input gradients
    are bit-identical (ckptplan.hpp:8-9, deterministic kernels), and match
    the fp64 reference."""
    _need_drivers()
    with tempfile.TemporaryDirectory() as td:
        outs = {}
        for name, drv in (("dropin", O.DROPIN_DRIVER), ("ref", O.REF_DRIVER)):
            r = subprocess.run([str(drv), "ckpt128", str(Path(td, name + ".bin"))], check=True,
                               capture_output=True, text=True, timeout=300)
            outs[name] = (json.loads(r.stdout), np.fromfile(Path(td, name + ".bin")))
    (gm, gx), (rm, rx) = outs["dropin"], outs["ref"]
    assert gm["bitwise_equal"] is True and rm["bitwise_equal"] is True
    assert gm["counts"] == rm["counts"]
    assert _rel(gx, rx) < TOL
