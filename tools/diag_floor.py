"""Diagnostics: fixed per-launch cost as the bench times it (after a 256 MB flush)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fea_inputs import CONFIGS, make_workload  # noqa: E402
from paper_2204_03893_b200 import Assembler  # noqa: E402

cfg = CONFIGS["C2"]
wl = make_workload(cfg)
m = wl.mesh
coef = (cfg.k_kind, tuple(cfg.k_par))
asm = Assembler(cfg.p, wl.q_xy, wl.q_w, m.vert_xy, m.elem_vert, m.n_dof, m.elem_dof, device=0,
                reorder=cfg.reorder, which=cfg.which, coef_m=coef, coef_c=coef)
u = torch.tensor(asm.to_library(wl.u0), dtype=torch.float64, device="cuda:0")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda:0")
tiny = torch.empty(1, dtype=torch.float32, device="cuda:0")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fn, n=20):
    ts = []
    for i in range(n):
        flush.fill_(float(i))
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


print(f"empty-ish torch op (tiny fill) after flush: {timed(lambda: tiny.fill_(2.0)):.1f} us")
print(f"events only: {timed(lambda: None):.1f} us")
print(f"reassemble (FEA_DEBUG_MODE={os.environ.get('FEA_DEBUG_MODE', '0')}): {timed(lambda: asm.reassemble(u)):.1f} us")
