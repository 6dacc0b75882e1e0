"""Diagnostics: event trace of CTA 0 / thread 0 of k_reassemble5 (FEA_DEBUG_MODE=8 + FEA_DEBUG_TIMING=1).

    FEA_DEBUG_TIMING=1 FEA_DEBUG_MODE=8 python tools/diag_trace.py C2
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fea_inputs import CONFIGS, make_workload  # noqa: E402
from paper_2204_03893_b200 import Assembler  # noqa: E402

NAMES = {9: "entry", 6: "prologue done", 0: "compute", 1: "move+refill", 2: "bar1", 3: "rec wait", 4: "phase B",
         5: "bar2"}
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
wl = make_workload(cfg)
m = wl.mesh
coef = (cfg.k_kind, tuple(cfg.k_par))
asm = Assembler(cfg.p, wl.q_xy, wl.q_w, m.vert_xy, m.elem_vert, m.n_dof, m.elem_dof, device=0,
                reorder=cfg.reorder, which=cfg.which, coef_m=coef, coef_c=coef)
u = torch.tensor(asm.to_library(wl.u0), dtype=torch.float64, device="cuda:0")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda:0")
for it in range(3):
    flush.fill_(float(it))
    torch.cuda.synchronize()
    asm.reassemble(u)
    torch.cuda.synchronize()
ev = []
for k in range(56):
    slot, t = asm.ctx.stat(40 + 2 * k), asm.ctx.stat(41 + 2 * k)
    if t == 0:
        break
    ev.append((slot, t))
t0 = ev[0][1] if ev else 0
prev = t0
for slot, t in ev:
    name = NAMES.get(slot, slot) if slot < 100 else f"  class C={(slot - 100) // 100} n~{10 * ((slot - 100) % 100)}"
    print(f"{(t - t0) / 1000:8.2f} us  (+{(t - prev) / 1000:6.2f})  {name}")
    prev = t

if os.environ.get("FEA_DEBUG_MODE", "0").isdigit() and int(os.environ.get("FEA_DEBUG_MODE", "0")) & 32:
    import numpy as np
    g = asm.ctx.stat(8)
    raw = np.array([asm.ctx.stat(40 + 184 + k) for k in range(3 * min(g, 400))], dtype=np.int64).reshape(-1, 3)
    t0 = raw[:, 0].min()
    st, en = (raw[:, 0] - t0) / 1000, (raw[:, 1] - t0) / 1000
    nb = [(asm.ctx.stat(1) - 1 - b) // g + 1 for b in range(len(st))]
    print(f"CTAs {len(st)}: start min/med/max {st.min():.2f}/{np.median(st):.2f}/{st.max():.2f} us, "
          f"end min/med/max {en.min():.2f}/{np.median(en):.2f}/{en.max():.2f} us")
    for k in sorted(set(nb)):
        sel = np.array(nb) == k
        print(f"  CTAs with {k} blocks: {sel.sum()}, end median {np.median(en[sel]):.2f} max {en[sel].max():.2f}")
    sm = raw[:, 2]
    order = np.argsort(-en)[:6]
    print("  slowest CTAs:", [(int(b), round(float(en[b]), 2), int(sm[b]), nb[b]) for b in order])
