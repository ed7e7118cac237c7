"""bench.py's N>1 path end to end on one GPU (--share-gpu: both ranks on
cuda:0, CUDA-IPC transport): self-spawned ranks, one JSON line with the
contract keys, the schedule legs, the no-comm arm and the roofline fields."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


def _line(out: str) -> dict:
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out
    return json.loads(lines[0])


def test_bench_two_ranks_self_spawned(cuda):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--seq", "4096",
                        "--heads", "2", "--share-gpu", "--steps", "2", "--warmup", "3",
                        "--leg-steps", "2"], capture_output=True, text=True, timeout=600,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-4000:]
    j = _line(r.stdout)
    assert j["n_gpus"] == 2 and j["steps"] == 2 and j["warmup"] == 3
    assert j["metric"] == "attn fwd+bwd TFLOP/s" and j["value"] > 0 and j["scaling"] == "strong"
    assert j["config"]["transport"] == "ipc" and j["config"]["seq_len"] == 4096
    assert {"balanced_split+balanced_split", "ring+ring", "balanced+balanced", "nocomm"} <= set(j["legs"])
    assert j["balanced_speedup_vs_ring"] > 0 and j["exposed_comm_pct"] is not None
    roof = j["roofline"]
    assert roof["bound"] in ("tensor", "nvlink") and roof["nvlink_bytes_per_gpu"] > 0
    assert roof["t_roof_ms"] == max(roof["t_tensor_ms"], roof["t_nvlink_ms"])
    assert j["e2e"]["h2d_bytes_per_step"] == 4 * 2 * 4096 * 128 * 2
    assert j["gpu_launches"] > 0 and "clocks" in j


def test_bench_gqa_config_single_gpu(cuda):
    """--config cfg2gqa (32 q / 8 kv heads, cfg5's ratio) at a reduced length."""
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--config", "cfg2gqa", "--seq",
                        "4096", "--steps", "2", "--warmup", "3", "--no-cpu-baseline"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-4000:]
    j = _line(r.stdout)
    assert j["config"]["heads_kv"] == 8 and j["config"]["heads"] == 32
    assert j["e2e"]["h2d_bytes_per_step"] == (2 * 32 + 2 * 8) * 4096 * 128 * 2


def test_bench_eight_ranks_self_spawned(cuda):
    """The SCALE run's largest N: eight self-spawned ranks (sharing cuda:0)
    through every leg of the N>1 line."""
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "8", "--seq", "8192",
                        "--heads", "2", "--share-gpu", "--steps", "2", "--warmup", "3",
                        "--leg-steps", "2"], capture_output=True, text=True, timeout=900,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-4000:]
    j = _line(r.stdout)
    assert j["n_gpus"] == 8 and j["config"]["tokens_per_gpu"] == 1024
    assert {"balanced_split+balanced_split", "ring+ring", "balanced+balanced", "nocomm"} <= set(j["legs"])


def test_bench_nccl_failure_falls_back_to_ipc(cuda):
    """--transport nccl with both ranks on one GPU: NCCL's communicator init
    fails on every rank (duplicate GPU); the ranks agree and run the IPC
    transport instead, and the line records why."""
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--seq", "4096",
                        "--heads", "2", "--share-gpu", "--transport", "nccl", "--steps", "2",
                        "--warmup", "3", "--no-legs"], capture_output=True, text=True, timeout=600,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-4000:]
    j = _line(r.stdout)
    assert j["config"]["transport"] == "ipc" and "NCCL" in j["config"]["transport_fallback"]
