#!/usr/bin/env python
"""Planning-only (no GPU) statistics of a config's plan: blocks, e_max, element visits, v6 A2
row-tile work with skipping (per mille of full) and the A-warp imbalance (per mille: NA x the
busiest warp's work / total work).   usage: python tools/plan_stats.py C5 [N] [key=value ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fea_inputs import CONFIGS, make_workload, scaled  # noqa: E402
from paper_2204_03893_b200 import fea  # noqa: E402

cfg = CONFIGS[sys.argv[1]]
if len(sys.argv) > 2 and sys.argv[2].isdigit():
    cfg = scaled(cfg, int(sys.argv[2]))
tun = [a.split("=") for a in sys.argv[2:] if "=" in a]
wl = make_workload(cfg)
m = wl.mesh
ctx = fea.Context(device=-1)
ctx.set_element(cfg.p, wl.q_xy, wl.q_w)
ctx.mesh_upload(m.vert_xy, m.elem_vert, m.n_dof, m.elem_dof, reorder=cfg.reorder)
for k, v in tun:
    ctx.set_tuning(int(k), int(v))
t = time.time()
ctx.build_pattern()
print(f"{sys.argv[1]} N={cfg.N}: plan {time.time() - t:.1f} s, kver {ctx.stat(11)}, blocks {ctx.stat(1)}, "
      f"e_max {ctx.stat(7)}, visits {ctx.stat(2) / max(1, ctx.stat(3)):.3f}, smem {ctx.stat(6)}, "
      f"A2 work {ctx.stat(38)}/1000, A-warp imbalance {ctx.stat(39)}/1000")
