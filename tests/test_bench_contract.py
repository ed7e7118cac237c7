"""bench.py's reference arm (no GPU): one JSON line with the contract's keys,
measured by the unmodified reference build (oracle/_ref/ref_driver)."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.skipif(not (ROOT / "oracle" / "_ref" / "ref_driver").exists(),
                    reason="reference build absent (make -C oracle ref)")
def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    j = json.loads(lines[0])
    assert j["impl"] == "reference" and j["metric"] == "attn fwd+bwd TFLOP/s"
    assert j["unit"] == "TFLOP/s" and j["higher_is_better"] is True and j["value"] > 0
    assert j["cpu_baseline"]["kind"] == "reference" and j["cpu_baseline"]["cores"] >= 1
    assert j["e2e"] == {"value": j["value"], "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert j["steps"] == 1 and j["warmup"] == 3


@pytest.mark.skipif(not (ROOT / "oracle" / "_ref" / "ref_driver").exists(),
                    reason="reference build absent (make -C oracle ref)")
def test_reference_arm_multi_gpu_line_names_cfg3():
    """--impl reference --gpus 2 (the driver's N>1 reference arm): rank 0 prints
    one line on the N>1 default config (cfg3, strong scaling); other ranks exit 0."""
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "3"], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    j = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][0])
    assert j["n_gpus"] == 2 and j["scaling"] == "strong" and j["config"]["seq_len"] == 131072
    env = dict(__import__("os").environ, RANK="1", WORLD_SIZE="2")
    r1 = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2",
                         "--steps", "1", "--warmup", "3"], capture_output=True, text=True,
                        timeout=600, cwd=ROOT, env=env)
    assert r1.returncode == 0 and not r1.stdout.strip()


def test_bench_rejects_missing_gpus_without_share_flag(tmp_path):
    """A rank of `--gpus 2` on a host with fewer visible GPUs fails fast with a
    clear message instead of silently sharing a device."""
    import os
    env = dict(os.environ, RANK="0", WORLD_SIZE="2", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
               MASTER_PORT="29555", CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode != 0 and "visible GPUs" in (r.stderr + r.stdout)
