"""Instruction / stall-sample split of an ncu report by source-line category (kernel v5).

    python tools/ncu_cats.py gpurun_out/prof.ncu-rep
"""
import collections
import csv
import io
import subprocess
import sys


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    src = {}
    for f in ("fea_kernels5.cu", "fea_device.cuh"):
        src[f] = open(f"paper_2204_03893_b200/csrc/{f}").read().split("\n")
    fname = hdr = cur = None
    agg, samp = collections.Counter(), collections.Counter()
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
        if r[0].isdigit():
            cur = (fname, int(r[0]))
        if cur is None or len(r) < 6:
            continue
        try:
            ins = float(r[hdr["Instructions Executed"]])
            sm = float(r[hdr["Warp Stall Sampling (All Samples)"]])
        except (KeyError, ValueError):
            continue
        f, line = cur
        text = src[f][line - 1] if f in src and line - 1 < len(src[f]) else ""
        if f == "fea_device.cuh" and ("items5" in text or "vm[" in text or "vc[" in text or "am" in text or
                                      "u16_of" in text or "word_of" in text or "it[" in text or "cls[" in text or
                                      "switch (c.x)" in text or "case " in text or "slot" in text):
            cat = "phaseB"
        elif f == "fea_device.cuh" and ("mbar" in text or "try_wait" in text or "WAIT_" in text or "smem_u32" in text):
            cat = "mbarrier"
        elif f == "fea_kernels5.cu" and any(k in text for k in ("fma(", "y[q]", "z0[q]", "z1[q]", "sVm[t", "sVc[t", "jset", "J(0", "uq[q]", "lm[q]", "B0", "A00", "A11", "A01", "det", "keval")):
            cat = "compute"
        elif f == "fea_kernels5.cu" and any(k in text for k in ("settle", "advance", "nunits", "blk_of", "cu ", "cs ", "ls", "lu")):
            cat = "cursor"
        elif f == "fea_kernels5.cu" and any(k in text for k in ("ldg", "dof", "g.u", "g.x", "ga = gb", "refill")):
            cat = "gather"
        elif "sm_20_intrinsics" in f:
            cat = "mbarrier"
        elif f == "fea_device.cuh" and ("horner" in text or "k[q]" in text or "par[" in text):
            cat = "compute"
        else:
            cat = f"other:{f}"
        agg[cat] += ins
        samp[cat] += sm
    ti, ts = sum(agg.values()) or 1, sum(samp.values()) or 1
    for k, v in agg.most_common():
        print(f"{k:28s} inst {100 * v / ti:5.1f}%  samples {100 * samp[k] / ts:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
