"""GPU parity of the tensor contractions:
(M o2 v) and (C o2 v) through fea_assemble_tensor vs the oracle's element-by-element assembly
(oracle.assemble_tensor_contraction) on the same seeded inputs.  Bar: pattern identical to the
matrices' (bit-exact), values max|gpu - oracle| <= 1e-12 max|oracle| (reading 12)."""
import copy

import numpy as np
import pytest

import oracle
from fea_inputs import CONFIGS, K_EXP, K_POLY, K_PWL, make_workload, scaled, single_element_mesh, triangle_rule
from fea_inputs.mesh import random_mesh_from_structured
from tests.helpers import lib_numbering, maxabs_rel

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _run(mesh, q_xy, q_w, u_user, v_user, p, mcoef, ccoef, do_m=True, do_c=True, reorder=True, tker=0):
    import torch
    from paper_2204_03893_b200.fea import FEA_MASS, FEA_STIFF, FEA_TUNE_TENSOR_KERNEL, Context
    if tker == 5 and not (p == 1 and len(q_w) == 3):
        pytest.skip("k_tensor5 covers P1 with its 3-point rule")
    ctx = Context(device=0)
    ctx.set_element(p, q_xy, q_w)
    ctx.mesh_upload(mesh.vert_xy, mesh.elem_vert, mesh.n_dof, mesh.elem_dof, reorder=reorder)
    ctx.set_tuning(FEA_TUNE_TENSOR_KERNEL, tker)
    ctx.build_pattern()
    ctx.set_coefficient(FEA_MASS, mcoef[0], mcoef[1])
    ctx.set_coefficient(FEA_STIFF, ccoef[0], ccoef[1])
    perm = ctx.get_dof_perm()
    dev = "cuda:0"
    u = torch.tensor(u_user[perm], dtype=torch.float64, device=dev)
    v = torch.tensor(v_user[perm], dtype=torch.float64, device=dev)
    n = max(ctx.nnz, 1)
    mt = torch.full((n,), np.nan, dtype=torch.float64, device=dev) if do_m else None
    ct = torch.full((n,), np.nan, dtype=torch.float64, device=dev) if do_c else None
    ctx.assemble_tensor(u, v, mt, ct)
    ctx.sync()
    assert ctx.stat(12) == (tker or ctx.stat(12)) and ctx.stat(12) in (1, 4, 5)
    rp, ci = ctx.get_pattern()
    mlib = copy.copy(mesh)
    mlib.elem_dof = lib_numbering(mesh, perm)
    ref = oracle.assemble_tensor_contraction(mlib, q_xy, q_w, np.ascontiguousarray(u_user[perm]),
                                             np.ascontiguousarray(v_user[perm]),
                                             m_coef=mcoef if do_m else None, c_coef=ccoef if do_c else None)
    assert np.array_equal(rp, ref.row_ptr) and np.array_equal(ci, ref.col_idx)
    out = {}
    if do_m:
        g = mt[: ctx.nnz].cpu().numpy()
        assert np.isfinite(g).all()
        out["M"] = maxabs_rel(g, ref.M)
    if do_c:
        g = ct[: ctx.nnz].cpu().numpy()
        assert np.isfinite(g).all()
        out["C"] = maxabs_rel(g, ref.K)
    ctx.close()
    return out


# FEA_TUNE_TENSOR_KERNEL: k_tensor (lane per element), k_tensor4 (DMMA), k_tensor5 (lane per element,
# pipelined; P1 with the 3-point rule only: other cases skip)
TKER = [1, 4, 5]


@pytest.mark.parametrize("tker", TKER)
@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_tensor_parity_random_mesh(p, tker):
    """Both contractions, every order, the configs' minimal rule, polynomial and exp k."""
    m = random_mesh_from_structured(8, p, seed=300 + p)
    rng = np.random.default_rng(p)
    u = rng.uniform(-1, 1, m.n_dof)
    v = rng.normal(size=m.n_dof)
    xy, w = triangle_rule(2 * p)
    for mc, cc in (((K_POLY, (1.0, 0.0, 1.0)), (K_POLY, (1.0, 0.0, 0.0, 0.0, 1.0))),
                   ((K_EXP, (1.3, 0.5)), (K_EXP, (0.7, -0.3)))):
        err = _run(m, xy, w, u, v, p, mc, cc, tker=tker)
        assert err["M"] <= TOL and err["C"] <= TOL, err


@pytest.mark.parametrize("tker", TKER)
@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_tensor_modes_generic_rule_pwl(p, tker):
    """Mass-only / conductivity-only launches, a non-minimal rule (generic kernel), PWL k
    (k' = segment slope), user numbering."""
    m = random_mesh_from_structured(6, p, seed=310 + p)
    rng = np.random.default_rng(10 + p)
    u = rng.uniform(-1, 1, m.n_dof)
    v = rng.uniform(-2, 2, m.n_dof)
    pwl = (K_PWL, (-1.0, 1.5, 0.0, 0.7, 1.0, 0.5))
    xy, w = triangle_rule(min(8, 2 * p + 2))
    assert _run(m, xy, w, u, v, p, pwl, pwl, do_c=False, reorder=False, tker=tker)["M"] <= TOL
    assert _run(m, xy, w, u, v, p, pwl, pwl, do_m=False, reorder=False, tker=tker)["C"] <= TOL


@pytest.mark.parametrize("tker", TKER)
@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_tensor_single_element(p, tker):
    for mesh in (single_element_mesh((0.0, 0.0), (1.0, 0.0), (0.0, 1.0), p=p),
                 single_element_mesh((0.3, -0.2), (1.7, 0.4), (0.1, 2.0), p=p)):
        rng = np.random.default_rng(p)
        u = rng.uniform(0, 1, mesh.n_dof)
        v = rng.normal(size=mesh.n_dof)
        xy, w = triangle_rule(2 * p)
        err = _run(mesh, xy, w, u, v, p, (K_POLY, (1.0, 0.0, 1.0)), (K_POLY, (1.0, 0.0, 1.0)), tker=tker)
        assert err["M"] <= TOL and err["C"] <= TOL, err


@pytest.mark.parametrize("tker", TKER)
@pytest.mark.parametrize("name,N", [("C2", 40), ("C3", 20), ("C5", 10)])
def test_tensor_config_shapes(name, N, tker):
    """Config-shaped meshes (several blocks, ragged tail): u, v = two iterates of the workload."""
    cfg = scaled(CONFIGS[name], N)
    wl = make_workload(cfg)
    us = list(wl.u_sequence(2))
    coef = (cfg.k_kind, tuple(cfg.k_par))
    err = _run(wl.mesh, wl.q_xy, wl.q_w, us[0], us[1] - us[0], cfg.p, coef, coef, tker=tker)
    assert err["M"] <= TOL and err["C"] <= TOL, err


@pytest.mark.parametrize("p", [2, 3, 4])
def test_tensor4_deterministic_across_tilings(p):
    """k_tensor4: bit-identical values across runs and element caps per block (FEA_TUNE_EMAX):
    per-element DMMA arithmetic does not depend on the element's tile position, and phase B sums
    every slot in ascending library element order (reading 11)."""
    import torch
    from paper_2204_03893_b200.fea import FEA_MASS, FEA_STIFF, FEA_TUNE_EMAX, FEA_TUNE_TENSOR_KERNEL, Context
    m = random_mesh_from_structured(10, p, seed=330 + p)
    xy, w = triangle_rule(2 * p)
    rng = np.random.default_rng(30 + p)
    u = rng.uniform(-1, 1, m.n_dof)
    v = rng.normal(size=m.n_dof)
    outs = []
    for cap in (0, 0, 24, 40):
        ctx = Context(device=0)
        ctx.set_element(p, xy, w)
        ctx.mesh_upload(m.vert_xy, m.elem_vert, m.n_dof, m.elem_dof)
        ctx.set_tuning(FEA_TUNE_TENSOR_KERNEL, 4)
        ctx.set_tuning(FEA_TUNE_EMAX, cap)
        ctx.build_pattern()
        ctx.set_coefficient(FEA_MASS, K_EXP, (1.3, 0.5))
        ctx.set_coefficient(FEA_STIFF, K_POLY, (1.0, 0.0, 1.0))
        perm = ctx.get_dof_perm()
        mt = torch.empty(ctx.nnz, dtype=torch.float64, device="cuda:0")
        ct = torch.empty(ctx.nnz, dtype=torch.float64, device="cuda:0")
        ctx.assemble_tensor(torch.tensor(u[perm], device="cuda:0"), torch.tensor(v[perm], device="cuda:0"), mt, ct)
        ctx.sync()
        outs.append((ctx.stat(16), mt.cpu().numpy(), ct.cpu().numpy()))
        ctx.close()
    assert outs[2][0] > outs[0][0]  # a finer tiling
    for nb, mt, ct in outs[1:]:
        assert np.array_equal(outs[0][1], mt) and np.array_equal(outs[0][2], ct)


def test_tensor5_replan_and_tilings():
    """k_tensor5 (P1, 3-point rule): a first call with one channel plans shared memory for it only;
    a later call with both re-plans.  Values are bit-identical across calls, element caps per block
    (FEA_TUNE_EMAX) and against a fresh context, and match the oracle (reading 11)."""
    import torch
    from paper_2204_03893_b200.fea import FEA_MASS, FEA_STIFF, FEA_TUNE_EMAX, FEA_TUNE_TENSOR_KERNEL, Context
    m = random_mesh_from_structured(24, 1, seed=341)
    xy, w = triangle_rule(2)
    assert len(w) == 3
    rng = np.random.default_rng(41)
    u = rng.uniform(-1, 1, m.n_dof)
    v = rng.normal(size=m.n_dof)
    dev = "cuda:0"
    runs = []
    for cap, seq in ((0, ("C", "MC")), (0, ("M", "MC")), (40, ("MC",)), (64, ("C", "M"))):
        ctx = Context(device=0)
        ctx.set_element(1, xy, w)
        ctx.mesh_upload(m.vert_xy, m.elem_vert, m.n_dof, m.elem_dof)
        ctx.set_tuning(FEA_TUNE_TENSOR_KERNEL, 5)
        ctx.set_tuning(FEA_TUNE_EMAX, cap)
        ctx.build_pattern()
        ctx.set_coefficient(FEA_MASS, K_EXP, (1.3, 0.5))
        ctx.set_coefficient(FEA_STIFF, K_POLY, (1.0, 0.0, 1.0))
        perm = ctx.get_dof_perm()
        ut, vt = torch.tensor(u[perm], device=dev), torch.tensor(v[perm], device=dev)
        got = {}
        for which in seq:
            mt = torch.full((ctx.nnz,), np.nan, dtype=torch.float64, device=dev) if "M" in which else None
            ct = torch.full((ctx.nnz,), np.nan, dtype=torch.float64, device=dev) if "C" in which else None
            ctx.assemble_tensor(ut, vt, mt, ct)
            ctx.sync()
            assert ctx.stat(12) == 5
            for k, t in (("M", mt), ("C", ct)):
                if t is not None:
                    g = t.cpu().numpy()
                    assert np.isfinite(g).all()
                    if k in got:
                        assert np.array_equal(got[k], g)
                    got[k] = g
        runs.append((ctx.stat(16), got))
        if cap == 0 and seq[0] == "C":
            mlib = copy.copy(m)
            mlib.elem_dof = lib_numbering(m, perm)
            ref = oracle.assemble_tensor_contraction(mlib, xy, w, np.ascontiguousarray(u[perm]),
                                                     np.ascontiguousarray(v[perm]),
                                                     m_coef=(K_EXP, (1.3, 0.5)), c_coef=(K_POLY, (1.0, 0.0, 1.0)))
            assert maxabs_rel(got["M"], ref.M) <= TOL and maxabs_rel(got["C"], ref.K) <= TOL
        ctx.close()
    assert runs[2][0] > runs[0][0]  # a finer tiling
    for _, got in runs[1:]:
        assert np.array_equal(runs[0][1]["M"], got["M"]) and np.array_equal(runs[0][1]["C"], got["C"])
