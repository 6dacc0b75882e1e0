#!/usr/bin/env python
"""SASS evidence for DESIGN.md: per-kernel counts of the instruction classes the design relies on
(DMMA = FP64 tensor-core mma.sync m8n8k4, UBLKCP = cp.async.bulk (TMA bulk copy), UBLKPF = bulk L2
prefetch, LDGSTS = cp.async, SYNCS = mbarrier ops, REDG = global reductions (diagnostics only),
LDL/STL = local-memory spills) in libfea.so.   usage: python tools/sass_summary.py [libfea.so]"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2204_03893_b200", "libfea.so")
KEYS = ["DMMA", "DFMA", "UBLKCP", "UBLKPF", "LDGSTS", "SYNCS", "BAR.SYNC", "LDS.64", "LDS.128", "STS.128",
        "STG.E.64", "REDG", "LDL", "STL"]
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
arch = sorted(set(re.findall(r"arch = (sm_\w+)", sass)))
cnt = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        cur = cur.replace("(anonymous namespace)::", "")
        cnt[cur] = collections.Counter()
        continue
    if cur and re.match(r"\s+/\*[0-9a-f]{4}\*/", line):
        op = line.split("*/", 1)[1].strip().split()
        if not op:
            continue
        if op[0].startswith("@"):
            op = op[1:]
        for k in KEYS:
            if op and (op[0] == k or op[0].startswith(k + ".")):
                cnt[cur][k] += 1
print(f"# cuobjdump -sass {os.path.basename(lib)}: {len(cnt)} kernels, arch {', '.join(arch)}")
print("# kernel | " + " ".join(KEYS))
for f, c in cnt.items():
    print(f"{f.split('(')[0]:48s} " + " ".join(f"{k}={c[k]}" for k in KEYS if c[k]))
