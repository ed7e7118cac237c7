"""Runs the C++ drop-in API tests (tests/cpp/test_b200_api.cpp over
include/distattn/b200.hpp): schedule parity on CPU; kernels and the runtime
on a B200. The binary is built by __graft_entry__.build()."""
import subprocess
from pathlib import Path

import pytest

EXE = Path(__file__).resolve().parent / "cpp" / "_build" / "test_b200_api"


def _run(*args):
    if not EXE.exists():
        from paper_2310_03294_b200 import build as B
        B.build_cpp_tests()
    r = subprocess.run([str(EXE), *args], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout, r.stdout
    return r.stdout


def test_cpp_api_schedules_cpu():
    out = _run("--cpu-only")
    assert "4 passed" in out


@pytest.mark.gpu
def test_cpp_api_kernels_and_runtime(cuda):
    out = _run()
    assert "FAIL" not in out


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_cpp_rank_runtime_multiprocess(cuda, world):
    """tests/cpp/test_rank_cpp.cpp: W forked processes drive
    distattn::b200::RankRuntime from C++ only (shared-memory allgather
    bootstrap, IPC transport, split forward + split backward, deterministic);
    each rank's chunk matches the C oracle and a second pass repeats its bits."""
    exe = EXE.parent / "test_rank_cpp"
    if not exe.exists():
        from paper_2310_03294_b200 import build as B
        B.build_cpp_tests()
    r = subprocess.run([str(exe), str(world), str(512 * world), "2"], capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
