"""Top source lines by warp-stall samples from an ncu --set full capture
(--import-source, -lineinfo builds), with each line's dominant stall reasons.

    python tools/ncu_stalls.py gpurun_out/prof_bwd_r1l.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys


def main(rep, top=25):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    cols = {h: i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h}
    lines = []
    for r in rows:
        if len(r) >= 6 and r[0].isdigit() and r[2] == "-":
            try:
                lines.append((int(r[4]), int(r[0]), r[1].strip()[:80],
                              sorted(((int(r[i]) if r[i].isdigit() else 0, h[6:]) for h, i in cols.items()),
                                     reverse=True)[:3]))
            except ValueError:
                pass
    tot = sum(x[0] for x in lines) or 1
    print(f"{rep}: {tot} warp-stall samples")
    for n, ln, src, st in sorted(lines, reverse=True)[:top]:
        print(f"{100 * n / tot:5.1f}%  L{ln:<4d} {src:80s} " + ", ".join(f"{h} {c}" for c, h in st))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
