"""Aggregate an ncu source page (cuda,sass correlated) per CUDA source line.

    python tools/ncu_lines.py gpurun_out/prof.ncu-rep [top_n]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, hdr = "?", None
    agg = defaultdict(lambda: [0.0, 0.0, ""])
    stall = defaultdict(lambda: defaultdict(float))
    cur = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = {h: k for k, h in enumerate(r)}
            continue
        if hdr is None or r[0] == "Function Name":
            continue
        if r[0] and r[0].isdigit():
            cur = (fname, int(r[0]))
            agg[cur][2] = r[1]
        if cur is None or len(r) < 6:
            continue
        def f(k):
            try:
                return float(r[hdr[k]])
            except (KeyError, ValueError):
                return 0.0
        agg[cur][0] += f("Warp Stall Sampling (All Samples)")
        agg[cur][1] += f("Instructions Executed")
        for h, k in hdr.items():
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    stall[cur][h[6:]] += float(r[k])
                except ValueError:
                    pass
    ts = sum(v[0] for v in agg.values()) or 1
    ti = sum(v[1] for v in agg.values()) or 1
    print(f"total samples {ts:.0f}  total warp-instructions {ti:.0f}")
    for key, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        st = sorted(stall[key].items(), key=lambda kv: -kv[1])[:3]
        sts = " ".join(f"{n}={100 * x / max(v[0], 1):.0f}%" for n, x in st if x > 0)
        print(f"{key[0]}:{key[1]:<4} samp {100 * v[0] / ts:5.1f}%  inst {100 * v[1] / ti:5.1f}%  [{sts}]  {v[2].strip()[:70]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
