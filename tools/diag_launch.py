"""Diagnostics: host submission cost vs device time of fea_reassemble (not a bench).

    python tools/diag_launch.py C2 [n]
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fea_inputs import CONFIGS, make_workload  # noqa: E402
from paper_2204_03893_b200 import Assembler  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200
wl = make_workload(cfg)
m = wl.mesh
coef = (cfg.k_kind, tuple(cfg.k_par))
asm = Assembler(cfg.p, wl.q_xy, wl.q_w, m.vert_xy, m.elem_vert, m.n_dof, m.elem_dof, device=0,
                reorder=cfg.reorder, which=cfg.which, coef_m=coef, coef_c=coef)
u = torch.tensor(asm.to_library(wl.u0), dtype=torch.float64, device="cuda:0")
for _ in range(5):
    asm.reassemble(u)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(n):
    asm.reassemble(u)
t_host = (time.perf_counter() - t0) / n
torch.cuda.synchronize()
t_all = (time.perf_counter() - t0) / n
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(n):
    asm.reassemble(u)
b.record()
torch.cuda.synchronize()
print(f"{cfg.name}: host submit {t_host * 1e6:.1f} us/call, wall {t_all * 1e6:.1f} us/call, "
      f"device back-to-back {a.elapsed_time(b) * 1e3 / n:.1f} us/call (L2 warm)")
# single call with an idle GPU (as timed in bench.py, without the flush)
ts = []
for _ in range(20):
    torch.cuda.synchronize()
    a.record()
    asm.reassemble(u)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
ts.sort()
print(f"{cfg.name}: isolated call (idle GPU) median {ts[len(ts) // 2]:.1f} us")
# GPU busy ahead of the call (a long fill first, so host submission overlaps)
big = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda:0")
ts = []
for _ in range(20):
    torch.cuda.synchronize()
    big.fill_(1.0)
    a.record()
    asm.reassemble(u)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
ts.sort()
print(f"{cfg.name}: call after a 256 MB fill median {ts[len(ts) // 2]:.1f} us")
