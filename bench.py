#!/usr/bin/env python
"""Benchmark of the per-Newton-iteration reassembly (BASELINE.json metric:
"element-matrix entries assembled/s (FP64, into CSR) and % of HBM roofline").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

A step = one reassembly (fea_reassemble: [allgather u] + the fused kernel) of every matrix the
config names, with a fresh u (u_r = u_{r-1} + 0.01 xi_r, reading 14), inputs resident in HBM.
Entries per step = n_e * n_p^2 * (#matrices).  L2 is flushed (256 MiB write)
before every timed step, outside the timed region.  Per-step device time from CUDA events on
the launching stream; the K steps are bracketed by barrier + synchronize; max over ranks.
Rank 0 prints one JSON line.  --impl reference times the CPU oracle (the reference arm of this
tier) on the host cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from fea_inputs import CONFIGS, MASS, STIFF, make_workload  # noqa: E402

METRIC = "element-matrix entries assembled/s (FP64, into CSR) and % of HBM roofline"
UNIT = "entries/s"
# The largest single-GPU config: C5, P4 M+K, 33.9 GB of algorithmic traffic per
# reassembly (HBM-resident; C2's 73.5 MB fits in L2).  The other configs are parity cases.
DEFAULT_CONFIG = "C5"


def canonical_bytes(n_v, n_e, n_p, n_dof, nnz, nmat):
    """Algorithmic bytes per reassembly (exactly the north_star list):
    coords 16 n_v + DOF map 4 n_p n_e + u 8 n_dof + scatter map 4 n_p^2 n_e + CSR 8 nnz #mat."""
    return 16 * n_v + 4 * n_p * n_e + 8 * n_dof + 4 * n_p * n_p * n_e + 8 * nnz * nmat


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling through NVML during the timed region."""

    def __init__(self, device_index: int, period_s: float = 0.005):
        self.ok = False
        self.samples = []
        self.reasons = set()
        self.period = period_s
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)
        self._stop = threading.Event()

    def _reason_names(self, mask):
        nv = self.nv
        names = {
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        return [k for k, v in names.items() if mask & v]

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                try:
                    mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:
                    mask = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.reasons.update(self._reason_names(mask))
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": getattr(self, "max_mhz", None), "reasons": sorted(self.reasons),
                    "samples": len(self.samples)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def env_dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_desc(cfg, wl):
    m = wl.mesh
    return {"workload": f"{cfg.name}: {cfg.description}", "config_index": cfg.index, "p": cfg.p, "N": cfg.N,
            "n_e": m.n_e, "n_dof": m.n_dof, "n_q": int(wl.q_w.shape[0]),
            "matrices": ("M+K" if cfg.which == 3 else "M" if cfg.which == 1 else "K"),
            "k": {0: "poly", 1: "exp", 2: "pwl"}[cfg.k_kind] + str(list(cfg.k_par)),
            "reorder": "morton" if cfg.reorder else "none"}


def cpu_oracle_run(wl, cfg, target_s: float, nthreads: int, lib_to_user=None, tensor: bool = False):
    """Time the oracle (Algorithm 1, as it stands) on a bounded sample: whole reassemblies of the
    workload if one takes < target_s, else a leading block of rows.  Returns (entries/s, desc,
    seconds per sample, pattern-build seconds of the sample) -- formation (values) and the
    structural pattern are timed separately, mirroring the paper's split."""
    import oracle
    m = wl.mesh
    if lib_to_user is not None:  # same numbering as the GPU run
        import copy
        inv = np.empty_like(lib_to_user)
        inv[lib_to_user] = np.arange(lib_to_user.shape[0])
        m = copy.copy(m)
        m.elem_dof = inv[m.elem_dof].astype(np.int32)
        u = np.ascontiguousarray(wl.u0[lib_to_user])
    else:
        u = wl.u0
    coef, mcoef = cfg.coef_c, cfg.coef_m
    if tensor:  # the oracle's tensor contraction (single-threaded: it has no OpenMP path)
        v = np.full_like(u, 0.01)
        nthreads = 1

        def run(r1, pat):
            oracle.assemble_tensor_contraction(m, wl.q_xy, wl.q_w, u, v, m_coef=mcoef if cfg.which & MASS else None,
                                               c_coef=coef if cfg.which & STIFF else None, r0=0, r1=r1, pat=pat)
    else:
        def run(r1, pat):
            oracle.assemble(m, wl.q_xy, wl.q_w, u, m_coef=mcoef, c_coef=coef, which=cfg.which, r0=0, r1=r1,
                            nthreads=nthreads, pat=pat)
    n_p = cfg.n_p
    nmat = cfg.n_matrices
    # sample rows [0, r1): grow until the estimated time reaches target_s
    r1 = min(m.n_dof, max(1000, m.n_dof // 64))
    while True:
        tp = time.perf_counter()
        pat = oracle.pattern(m.n_dof, m.elem_dof, 0, r1)
        t_pat = time.perf_counter() - tp
        t0 = time.perf_counter()
        run(r1, pat)
        dt = time.perf_counter() - t0
        if r1 >= m.n_dof or dt >= 0.25 * target_s:
            break
        r1 = min(m.n_dof, int(r1 * max(2.0, 0.5 * target_s / max(dt, 1e-3))))
    reps = max(1, int(target_s / max(dt, 1e-6)))
    t0 = time.perf_counter()
    for _ in range(reps):
        run(r1, pat)
    dt = (time.perf_counter() - t0) / reps
    # entries attributable to the sampled rows: local entries whose row lies in [0, r1)
    ed = m.elem_dof
    rows_in = (ed < r1).sum(axis=1)  # per element: local rows in the sample
    entries = int(rows_in.sum()) * n_p * nmat
    desc = (f"oracle rows [0,{r1}) of {m.n_dof} ({100.0 * r1 / m.n_dof:.1f}%), {reps} rep(s), "
            f"pattern build timed separately, {nthreads} thread(s)")
    return entries / dt, desc, dt, t_pat


def run_reference(args):
    """--impl reference: the CPU oracle (this tier's reference arm) on the host cores."""
    rank, world, _ = env_dist()
    if rank != 0:
        return 0
    cfg = CONFIGS[args.config]
    wl = make_workload(cfg)
    cores = len(os.sched_getaffinity(0))
    step_target = float(os.environ.get("FEA_REF_STEP_S", "1.0"))
    times = []
    desc = ""
    for i in range(args.warmup + args.steps):
        rate, desc, dt, _ = cpu_oracle_run(wl, cfg, step_target, cores)
        if i >= args.warmup:
            times.append(rate)
    value = statistics.median(times)
    ent_step = wl.mesh.n_e * cfg.n_p ** 2 * cfg.n_matrices
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": max(world, args.gpus), "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * ent_step / value, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference", "config": workload_desc(cfg, wl),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    rank, world, local = env_dist()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    from paper_2204_03893_b200 import Assembler
    cfg = CONFIGS[args.config]
    if args.scale:  # diagnostics only: the config's recipe on an N x N grid (not a bench value)
        from fea_inputs import scaled
        cfg = scaled(cfg, args.scale)
    t_setup = time.perf_counter()
    wl = make_workload(cfg)
    m = wl.mesh
    coef, mcoef = cfg.coef_c, cfg.coef_m
    tuning = {int(kv.split("=")[0]): int(kv.split("=")[1]) for kv in args.tune}
    if world > 1:
        tuning.setdefault(11, 1)  # FEA_TUNE_TIMING: exchange / assembly events per call (split below)
    asm = Assembler(cfg.p, wl.q_xy, wl.q_w, m.vert_xy, m.elem_vert, m.n_dof, m.elem_dof, device=local,
                    reorder=cfg.reorder, which=cfg.which, coef_m=mcoef, coef_c=coef, rank=rank, world=world,
                    tuning=tuning)
    t_setup = time.perf_counter() - t_setup
    nmat = cfg.n_matrices
    # distinct u per step (library numbering, owned rows), resident in HBM
    R = max(2, min(cfg.reassemblies, 10))
    us = []
    for u in wl.u_sequence(R):
        ul = asm.to_library(u)
        us.append(torch.tensor(asm.owned_slice(ul) if world > 1 else ul, dtype=torch.float64, device=dev))
    flush_mb = int(os.environ.get("FEA_FLUSH_MB", "256"))  # diagnostics only; the bench default flushes
    flush = torch.empty(max(1, flush_mb * 1024 * 1024 // 4), dtype=torch.float32, device=dev)
    # diagnostics: FEA_FLUSH_CLEAN=1 follows the write with a read of another buffer larger than
    # L2, so the kernel starts with a cold but CLEAN L2 (no dirty write-back of the flush data)
    clean = torch.empty_like(flush) if os.environ.get("FEA_FLUSH_CLEAN") else None
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    tensor = args.op == "tensor"
    if tensor:  # NEXT-1/2: (M o2 v), (C o2 v) at u = u_r, v = u_{r+1} - u_r (a Newton direction)
        if world > 1:
            raise SystemExit("--op tensor is single-GPU")
        vs = [us[(i + 1) % R] - us[i % R] for i in range(R)]
        mt = torch.empty(max(asm.nnz, 1), dtype=torch.float64, device=dev) if cfg.which & MASS else None
        ct = torch.empty(max(asm.nnz, 1), dtype=torch.float64, device=dev) if cfg.which & STIFF else None

        def step(i):
            asm.ctx.assemble_tensor(us[i % R], vs[i % R], mt, ct)
    else:
        def step(i):
            asm.reassemble(us[i % R])
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    sampler = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    split = []  # world > 1: (exchange us, assembly us) of every timed step (library events)
    with sampler:
        for i in range(args.steps):
            if flush_mb:
                flush.fill_(float(i))  # evict L2 (126 MB) before every timed step, outside the events
                if clean is not None:
                    clean.sum()
            ev[i][0].record(stream)
            step(i)
            ev[i][1].record(stream)
            if world > 1 and not tensor:
                split.append((asm.ctx.stat(36), asm.ctx.stat(37)))
        torch.cuda.synchronize()
    barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    tot = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(tot, op=torch.distributed.ReduceOp.MAX)
    total_ms = float(tot.item())
    ms_per_step = total_ms / args.steps
    entries_step = m.n_e * cfg.n_p ** 2 * nmat
    value = entries_step / (ms_per_step * 1e-3)

    # roofline of the dominant (only) kernel: canonical bytes of this rank's share / kernel time
    peak, peak_src = load_peaks()
    rp, _ = asm.pattern()
    nnz_local = asm.nnz
    if world == 1:
        B = canonical_bytes(m.n_v, m.n_e, cfg.n_p, m.n_dof, nnz_local, nmat) + (8 * m.n_dof if tensor else 0)
    else:  # per-rank share of the canonical bytes (rows owned)
        frac_rows = asm.n_rows / m.n_dof
        B = canonical_bytes(m.n_v, m.n_e, cfg.n_p, m.n_dof, 0, nmat) * frac_rows + 8 * nnz_local * nmat
    kern_ms = statistics.median(step_ms)
    xsplit = None
    if split:  # median per rank, then the max over ranks (allgather and kernels reported apart)
        med = torch.tensor([statistics.median(x for x, _ in split), statistics.median(k for _, k in split)],
                           dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(med, op=torch.distributed.ReduceOp.MAX)
        xsplit = {"exchange_ms_max_over_ranks": float(med[0]) / 1e3,
                  "assembly_ms_max_over_ranks": float(med[1]) / 1e3,
                  "note": "per-rank medians over the timed steps (CUDA events on the library's streams); the "
                          "assembly span includes any wait of the boundary blocks for the halo"}
        kern_ms = float(med[1]) / 1e3
    achieved = B / (kern_ms * 1e-3) / 1e9
    traffic = None
    if tensor:
        kname = {4: "k_tensor4", 5: "k_tensor5"}.get(asm.ctx.stat(12), "k_tensor")
    else:
        kname = {5: "k_reassemble5", 6: "k_reassemble6"}.get(asm.ctx.stat(11), "k_reassemble")
    prof = os.path.join(ROOT, "profiles", f"ncu_traffic_{cfg.name}_{kname}.json")
    if os.path.exists(prof):  # an ncu --set full capture of this kernel on this config
        with open(prof) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")

    # e2e: public API with host buffers (pinned), H2D of u and D2H of the values inside the timing
    # (for --op tensor: H2D of u and v, the tensor call, D2H of the values, through the same API)
    nu = m.n_dof if world == 1 else asm.n_rows
    u_pin = torch.empty(nu, dtype=torch.float64, pin_memory=True)
    u_pin.copy_(us[0].cpu())
    outs = [torch.empty(max(nnz_local, 1), dtype=torch.float64, pin_memory=True) if cfg.which & b else None
            for b in (MASS, STIFF)]
    outs_np = [o.numpy() if o is not None else None for o in outs]
    e2e_steps = max(3, min(args.steps, 20))
    if tensor:
        v_pin = torch.empty(nu, dtype=torch.float64, pin_memory=True)
        v_pin.copy_(vs[0].cpu())
        ud, vd = torch.empty_like(us[0]), torch.empty_like(vs[0])

        def e2e_once():
            ud.copy_(u_pin, non_blocking=True)
            vd.copy_(v_pin, non_blocking=True)
            asm.ctx.assemble_tensor(ud, vd, mt, ct)
            for o, d in zip(outs, (mt, ct)):
                if o is not None:
                    o.copy_(d[: o.shape[0]], non_blocking=True)
            torch.cuda.synchronize()
    else:
        def e2e_once():
            asm.ctx.reassemble_host(u_pin.numpy(), *outs_np)
    e2e_once()
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_once()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    tmax = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(tmax, op=torch.distributed.ReduceOp.MAX)
    e2e_s = float(tmax.item())

    line = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cores = len(os.sched_getaffinity(0))
            tgt = float(os.environ.get("FEA_CPU_BASELINE_S", "10"))
            rate, desc, dt, t_pat = cpu_oracle_run(wl, cfg, tgt, cores, lib_to_user=asm.lib_to_user, tensor=tensor)
            cores = 1 if tensor else cores
            cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc,
                   "pattern_build_s_of_sample": round(t_pat, 4), "values_s_of_sample": round(dt, 4)}
            if not tensor and cores > 1:  # the same oracle on one core (SURVEY 8(d) "Oracle timing")
                rate1, desc1, dt1, t_pat1 = cpu_oracle_run(wl, cfg, tgt, 1, lib_to_user=asm.lib_to_user)
                cpu["one_core"] = {"value": rate1, "unit": UNIT, "cores": 1, "sample": desc1,
                                   "pattern_build_s_of_sample": round(t_pat1, 4), "values_s_of_sample": round(dt1, 4)}
        desc = workload_desc(cfg, wl)
        if args.scale:
            desc["workload"] = f"DIAGNOSTIC {cfg.name} scaled to N={cfg.N} (not a bench value)"
        if tensor:
            desc["op"] = "tensor contractions (M o2 v, C o2 v), NEXT-1/2: u = u_r, v = u_{r+1} - u_r"
        if world > 1:
            mi = asm.ctx.stat(14)
            rpr = -(-m.n_dof // world)
            desc["exchange"] = (f"interface-only ncclAllGather of {mi} float64 per rank "
                                f"({8 * mi * world} B received per GPU per step; the full-vector "
                                f"allgather would be {8 * rpr * world} B)")
        desc.update({"l2": f"flushed ({flush_mb} MiB write) before every timed step" if flush_mb >= 256 else
                     f"NOT flushed ({flush_mb} MiB write): diagnostic run, not a bench value", "parallelism": f"rows{world}",
                     "nnz": int(nnz_local) if world == 1 else None, "setup_s": round(t_setup, 3),
                     "tuning": tuning})
        sk = (16, 17, 18, 19, 13) if tensor else (1, 2, 3, 6, 8)  # tensor plan / matrix plan statistics
        desc.update({"blocks": asm.ctx.stat(sk[0]),
                     "elem_visits_over_owned": round(asm.ctx.stat(sk[1]) / max(1, asm.ctx.stat(sk[2])), 4),
                     "smem_per_cta": asm.ctx.stat(sk[3]), "grid": asm.ctx.stat(sk[4])})
        if os.environ.get("FEA_DEBUG_TIMING"):
            if asm.ctx.stat(11) == 5:  # per-warp timeline of k_reassemble5 (lane 0 of every warp)
                names = ["compute", "move_refill", "full_wait", "rec_wait", "phaseB", "free_wait", "prologue"]
            elif asm.ctx.stat(11) == 6:  # k_reassemble6: summed over the warps of each role
                names = ["A_lamfull_wait", "A_A1", "A2_", "A_vfree_wait", "A_A2", "A_loop", "A_phaseB", "A7_",
                         "B_loop", "B_vfull_wait", "B_phaseB", "B3_", "B4_", "B5_", "B_A1", "B_prefetch"]
                ph = [asm.ctx.stat(20 + i) for i in range(16)] + [asm.ctx.stat(40 + i) for i in range(2)]
                desc["phase_cycles"] = dict(zip(names + ["P_free_wait", "P_gather"], ph))
                names = []
            else:
                names = ["unused0", "unused1", "A2_dmma", "B_and_next_A1", "unused4", "barrier_wait"]
            if names:
                ph = [asm.ctx.stat(20 + i) for i in range(len(names))]
                tot = sum(ph) or 1
                desc["phase_cycles_pct"] = dict(zip(names, [round(100.0 * x / tot, 1) for x in ph]))
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": desc,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "algorithmic_bytes": B,
                         "kernel": kname,
                         "peak_source": peak_src,
                         "kernel_ms_median": kern_ms},
            "cpu_baseline": cpu,
            "e2e": {"value": entries_step / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 8 * nu * (2 if tensor else 1),
                    "d2h_bytes_per_step": 8 * nnz_local * nmat, "ms_per_step": e2e_s * 1e3},
            "gpu_launches": args.steps * asm.ctx.stat(5),
            "exchange_split": xsplit,
            "clocks": sampler.summary(),
        }
        print(json.dumps(line), flush=True)
    asm.close()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=os.environ.get("FEA_BENCH_CONFIG", DEFAULT_CONFIG), choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--op", default="reassemble", choices=["reassemble", "tensor"],
                    help="reassemble: the per-iteration M, K reassembly (default); tensor: NEXT-1/2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scale", type=int, default=0, help="diagnostics: run the config's recipe on an N x N grid")
    ap.add_argument("--tune", action="append", default=[], help="libfea tuning key=value (fea.h FEA_TUNE_*)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: at least 3 warm-up steps
    if "WORLD_SIZE" in os.environ:
        if int(os.environ["WORLD_SIZE"]) != args.gpus and args.impl == "ours":
            raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}")
    elif args.gpus > 1:
        # one process per GPU: re-launch under torchrun (rendezvous on 127.0.0.1)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
        os.execv(sys.executable, cmd)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
