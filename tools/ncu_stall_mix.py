"""Kernel-wide warp-stall reason mix from an ncu --set full capture (source page).

    python tools/ncu_stall_mix.py gpurun_out/prof_bwd_r2j.ncu-rep
"""
import csv
import io
import subprocess
import sys


def main(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    cols = {h: i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h}
    tot = {}
    for r in rows:
        if len(r) >= 6 and r[0].isdigit() and r[2] == "-":
            for h, i in cols.items():
                if r[i].isdigit():
                    tot[h] = tot.get(h, 0) + int(r[i])
    s = sum(tot.values()) or 1
    print(rep)
    for h, v in sorted(tot.items(), key=lambda x: -x[1])[:12]:
        print(f"  {h[6:]:20s} {100 * v / s:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
