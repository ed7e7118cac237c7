"""Regenerates tests/golden/ from the UNMODIFIED reference build (oracle/_ref/ref_driver).

    make -C oracle ref && python oracle/make_golden.py

Fixtures (all produced by the reference's own code, run here):
  rng.json            splitmix64 KAT (numerics.hpp:140-174)
  schedules.json      ring + balanced flat tables, P = 1..16 (schedule.cpp:60-108)
  numerics_small.npz  float64 run_forward/run_backward outputs + counters on the
                      reference acceptance grid shapes (P x N x d, seed 0)
  numerics_d128.npz   bf16-rounded inputs, N=512, P=4, d=128, balanced, float32
                      outputs (the GPU-shape fixture)
  ckpt.json           checkpoint plans (ckptplan.cpp): positions, recompute counts,
                      cost-model times, saved scalars for L = 1..3
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
from oracle import oracle as O  # noqa: E402

OUT = HERE.parent / "tests" / "golden"

SMALL_GRID = [(P, N, d, sched) for P in (1, 2, 4, 8) for N in (32, 64) for d in (4, 16)
              for sched in ("ring", "balanced")]


def main():
    if not O.ref_available():
        raise SystemExit("oracle/_ref/ref_driver missing: run `make -C oracle ref` first")
    OUT.mkdir(parents=True, exist_ok=True)
    (OUT / "rng.json").write_text(json.dumps(O.ref_json("rng"), indent=1) + "\n")
    (OUT / "schedules.json").write_text(json.dumps(O.ref_json("schedules")) + "\n")
    (OUT / "ckpt.json").write_text(json.dumps(O.ref_json("ckpt"), indent=0) + "\n")

    arrays, meta = {}, {}
    for P, N, d, sched in SMALL_GRID:
        key = f"P{P}_N{N}_d{d}_{sched}"
        ref, m = O.ref_run(N, P, 1, d, 0, sched, bf16=False)
        for name in ("out", "lse", "dq", "dk", "dv"):
            arrays[f"{key}/{name}"] = ref[name][0]
        meta[key] = m["heads"][0]
    np.savez_compressed(OUT / "numerics_small.npz", **arrays)
    (OUT / "numerics_small.json").write_text(json.dumps(meta, indent=0) + "\n")

    ref, m = O.ref_run(512, 4, 1, 128, 0, "balanced", bf16=True)
    np.savez_compressed(OUT / "numerics_d128.npz",
                        **{n: ref[n][0].astype(np.float32) for n in ("out", "lse", "dq", "dk", "dv")})
    (OUT / "numerics_d128.json").write_text(json.dumps(m, indent=0) + "\n")
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
