"""GPU parity: the CUDA path (through the C ABI) vs the oracle on the same seeded inputs.

Bar (BASELINE.json north_star, reading 12): CSR row_ptr / col_idx bit-exact; values
max|gpu - oracle| <= 1e-12 * max|oracle| per matrix, FP64.
"""
import numpy as np
import pytest

import oracle
from fea_inputs import CONFIGS, K_EXP, K_POLY, K_PWL, MASS, STIFF, make_workload, scaled, single_element_mesh, \
    structured_mesh, triangle_rule, two_element_mesh
from fea_inputs.mesh import random_mesh_from_structured
from tests.helpers import coef_of, coefs_of, library_assemble, maxabs_rel, oracle_for

pytestmark = pytest.mark.gpu
TOL = 1e-12


def _check(res, ref, which):
    assert np.array_equal(res["row_ptr"], ref.row_ptr), "row_ptr not bit-exact"
    assert np.array_equal(res["col_idx"], ref.col_idx), "col_idx not bit-exact"
    if which & MASS:
        assert np.isfinite(res["M"]).all()
        assert maxabs_rel(res["M"], ref.M) <= TOL, maxabs_rel(res["M"], ref.M)
    if which & STIFF:
        assert np.isfinite(res["K"]).all()
        assert maxabs_rel(res["K"], ref.K) <= TOL, maxabs_rel(res["K"], ref.K)


# configs at sizes the oracle finishes in seconds; several CTA blocks and a ragged tail each
SMALL = [("C1", 32), ("C2", 48), ("C3", 24), ("C4", 96), ("C5", 12), ("E2", 43)]


@pytest.mark.parametrize("name,N", SMALL)
@pytest.mark.parametrize("kernel", [0, 4])
def test_config_parity_small(name, N, kernel):
    """kernel 0: automatic (v5 for p <= 2, v6 for p >= 3 with the native rule), 4: v4 forced
    (FEA_TUNE_KERNEL)."""
    cfg = scaled(CONFIGS[name], N)
    w = make_workload(cfg)
    mcoef, ccoef = coefs_of(cfg)
    for u in w.u_sequence(min(cfg.reassemblies, 2)):
        res = library_assemble(w.mesh, w.q_xy, w.q_w, u, cfg.p, mcoef, ccoef, which=cfg.which,
                               tuning={2: kernel} if kernel else None)
        auto = 5 if cfg.p <= 2 else 6  # the automatic kernel for the native rules
        assert res["ctx"].stat(11) == (auto if kernel == 0 else kernel)
        assert res["ctx"].stat(1) >= 2  # several blocks
        ref = oracle_for(w.mesh, w.q_xy, w.q_w, u, res["perm"], mcoef, ccoef, cfg.which)
        _check(res, ref, cfg.which)


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_single_and_two_element_meshes(p):
    for m in (single_element_mesh((0.0, 0.0), (1.0, 0.0), (0.0, 1.0), p=p),
              single_element_mesh((0.3, -0.2), (1.7, 0.4), (0.1, 2.0), p=p),
              single_element_mesh((0.0, 0.0), (0.0, 1.0), (1.0, 0.0), p=p)):  # clockwise
        xy, w = triangle_rule(2 * p)
        u = np.random.default_rng(p).uniform(-1, 1, m.n_dof)
        coef = (K_POLY, (1.0, 0.0, 1.0))
        res = library_assemble(m, xy, w, u, p, coef, coef)
        _check(res, oracle_for(m, xy, w, u, res["perm"], coef, coef, 3), 3)
    if p == 1:
        m = two_element_mesh()
        xy, w = triangle_rule(2)
        res = library_assemble(m, xy, w, np.zeros(4), 1, (K_POLY, (1.0,)), (K_POLY, (1.0,)))
        _check(res, oracle_for(m, xy, w, np.zeros(4), res["perm"], (K_POLY, (1.0,)), (K_POLY, (1.0,)), 3), 3)


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_distinct_coefficients_generic_rule_and_modes(p):
    """M and C with different k (two Lambda), a non-native rule (generic kernel), PWL k,
    mass-only and stiffness-only launches, user numbering (no reorder)."""
    m = random_mesh_from_structured(7, p, seed=50 + p)
    u = np.random.default_rng(p).uniform(-1, 1, m.n_dof)
    km, kc = (K_EXP, (1.3, 0.5)), (K_PWL, (-1.0, 1.5, 0.0, 0.7, 1.0, 0.5))
    for deg in sorted({2 * p, min(8, 2 * p + 2)}):
        xy, w = triangle_rule(deg)
        for which in (MASS | STIFF, MASS, STIFF):
            for reorder in (True, False):
                res = library_assemble(m, xy, w, u, p, km, kc, which=which, reorder=reorder)
                _check(res, oracle_for(m, xy, w, u, res["perm"], km, kc, which), which)


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_deterministic_across_runs_and_tilings(p):
    """Bit-identical values across repeated runs and across CTA tilings (smem budgets):
    per-slot summation in ascending library element order (reading 11)."""
    m = random_mesh_from_structured(10, p, seed=70 + p)
    xy, w = triangle_rule(2 * p)
    u = np.random.default_rng(p).uniform(0, 1, m.n_dof)
    coef = (K_POLY, (1.0, 0.0, 0.0, 0.0, 1.0))
    base = library_assemble(m, xy, w, u, p, coef, coef)
    again = library_assemble(m, xy, w, u, p, coef, coef)
    assert np.array_equal(base["M"], again["M"]) and np.array_equal(base["K"], again["K"])
    if p >= 3:
        # v6 ghost row-tile skipping relabels ghost elements per block (FEA_TUNE_SKIP): reproducible
        # run to run (above) but not bit-identical across tilings; without it every tiling and
        # kernel generation sums the same products in the same order
        base = library_assemble(m, xy, w, u, p, coef, coef, tuning={12: 0})
    # smem budgets (v4 and v5) and element caps per block (v5, FEA_TUNE_EMAX = 3)
    # ... and v5 without the zero-padded single-contributor items (FEA_TUNE_PAD1 = 10); p >= 3:
    # kernel v6 (default) and v4 (FEA_TUNE_KERNEL = 4) sum in the same order: bit-identical
    tunings = {1: [{1: 24000}, {3: 64}, {3: 120}, {10: 0}], 2: [{1: 40000}, {3: 48}, {3: 120}, {10: 0}],
               3: [{1: 100000}, {1: 150000}, {3: 24}, {2: 4}], 4: [{1: 150000}, {1: 190000}, {3: 16}, {2: 4}]}[p]
    for tu in tunings:
        if p >= 3:
            tu = {**tu, 12: 0}
        r = library_assemble(m, xy, w, u, p, coef, coef, tuning=tu)
        if 1 in tu or 3 in tu:
            assert r["ctx"].stat(1) > max(1, base["ctx"].stat(1) // 2)  # a different, finer tiling
        assert np.array_equal(base["M"], r["M"]) and np.array_equal(base["K"], r["K"])


@pytest.mark.parametrize("p,world", [(1, 2), (2, 3), (3, 4), (4, 2)])
def test_fake_world_bit_identical(p, world):
    """Row partition over `world` ranks (each rank: its rows + ghost elements), run one rank
    after another on one GPU with the full u: concatenated rows are bit-identical to world 1."""
    m = random_mesh_from_structured(9, p, seed=90 + p)
    xy, w = triangle_rule(2 * p)
    u = np.random.default_rng(p).uniform(0, 1, m.n_dof)
    coef = (K_POLY, (1.0, 0.0, 1.0))
    tu = {12: 0} if p >= 3 else None  # (bit-identity needs the same element labelling: no v6 skipping)
    base = library_assemble(m, xy, w, u, p, coef, coef, tuning=tu)
    Ms, Ks, rps, cis = [], [], [], []
    nxt = 0
    for r in range(world):
        res = library_assemble(m, xy, w, u, p, coef, coef, rank=r, world=world, tuning=tu)
        assert res["row_begin"] == nxt
        nxt += res["n_rows"]
        Ms.append(res["M"])
        Ks.append(res["K"])
        cis.append(res["col_idx"])
        rps.append(res["row_ptr"][1:] + (rps[-1][-1] if rps else 0))
    assert nxt == m.n_dof
    assert np.array_equal(np.concatenate([[0]] + rps), base["row_ptr"])
    assert np.array_equal(np.concatenate(cis), base["col_idx"])
    assert np.array_equal(np.concatenate(Ms), base["M"]) and np.array_equal(np.concatenate(Ks), base["K"])


def test_permutation_export_against_user_numbering():
    """Oracle in USER numbering, mapped through lib_to_user, equals the library result."""
    cfg = scaled(CONFIGS["C4"], 40)
    wl = make_workload(cfg)
    coef = coef_of(cfg)
    res = library_assemble(wl.mesh, wl.q_xy, wl.q_w, wl.u0, 1, coef, coef, which=STIFF)
    ref = oracle.assemble(wl.mesh, wl.q_xy, wl.q_w, wl.u0, m_coef=coef, c_coef=coef, which=STIFF)
    perm = res["perm"]
    n = wl.mesh.n_dof
    Du = ref.dense("K", n)
    Dl = np.zeros((n, n))
    for r in range(n):
        a, b = res["row_ptr"][r], res["row_ptr"][r + 1]
        Dl[r, res["col_idx"][a:b]] = res["K"][a:b]
    assert np.abs(Dl - Du[np.ix_(perm, perm)]).max() <= TOL * np.abs(Du).max()


def test_error_paths():
    import torch
    from paper_2204_03893_b200.fea import Context, FeaError
    ctx = Context(device=0)
    xy, w = triangle_rule(2)
    with pytest.raises(FeaError, match="FEA_E_ARG"):
        ctx.set_element(1, xy, w * 2)  # weights sum to 1, not 1/2
    with pytest.raises(FeaError, match="FEA_E_UNSUPPORTED"):
        ctx.set_element(5, xy, w)
    with pytest.raises(FeaError, match="FEA_E_STATE"):
        ctx.mesh_upload(np.zeros((3, 2)), np.zeros((1, 3)), 3, np.zeros((1, 3)))
    ctx.set_element(1, xy, w)
    with pytest.raises(FeaError, match="degenerate element 0"):
        ctx.mesh_upload(np.array([[0.0, 0], [1, 0], [2, 0]]), np.array([[0, 1, 2]]), 3, np.array([[0, 1, 2]]))
    m = structured_mesh(3, 1)
    ctx.mesh_upload(m.vert_xy, m.elem_vert, m.n_dof, m.elem_dof)
    u = torch.zeros(m.n_dof, dtype=torch.float64, device="cuda")
    with pytest.raises(FeaError, match="FEA_E_STATE"):
        ctx.assemble(u, torch.zeros(100, dtype=torch.float64, device="cuda"))
    ctx.build_pattern()
    buf = torch.zeros(ctx.nnz + 1, dtype=torch.float64, device="cuda")
    with pytest.raises(FeaError, match="16-byte aligned"):
        ctx.assemble(u, buf[1:])
    m3 = structured_mesh(2, 3)
    ctx.set_element(3, *triangle_rule(6))
    bad = m3.elem_dof.copy()
    bad[0, [3, 4]] = bad[0, [4, 3]]  # wrong edge orientation in element 0
    with pytest.raises(FeaError, match="inconsistently"):
        ctx.mesh_upload(m3.vert_xy, m3.elem_vert, m3.n_dof, bad)
    ctx.close()


def test_reassemble_and_host_entry_points():
    cfg = scaled(CONFIGS["C2"], 20)
    wl = make_workload(cfg)
    import torch
    from paper_2204_03893_b200 import Assembler
    coef = coef_of(cfg)
    asm = Assembler(cfg.p, wl.q_xy, wl.q_w, wl.mesh.vert_xy, wl.mesh.elem_vert, wl.mesh.n_dof, wl.mesh.elem_dof,
                    coef_m=coef, coef_c=coef)
    u_lib = asm.to_library(wl.u0)
    M, K = asm.reassemble(torch.tensor(u_lib, device="cuda"))
    asm.ctx.sync()
    Mh = np.zeros(asm.nnz)
    Kh = np.zeros(asm.nnz)
    asm.ctx.reassemble_host(u_lib, Mh, Kh)
    assert np.array_equal(Mh, M.cpu().numpy()) and np.array_equal(Kh, K.cpu().numpy())
    ref = oracle_for(wl.mesh, wl.q_xy, wl.q_w, wl.u0, asm.lib_to_user, coef, coef, 3)
    assert maxabs_rel(Mh, ref.M) <= TOL and maxabs_rel(Kh, ref.K) <= TOL


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_separate_rules_per_matrix(p):
    """NEXT-4 / PAPER.md:137: M with one rule, C with another (fea_set_rule); each matrix must
    equal the oracle run with its own rule.  Also the tensor contractions (M o2 v with M's rule,
    C o2 v with C's rule), and going back to one common rule."""
    import copy

    import torch
    from paper_2204_03893_b200.fea import FEA_MASS, FEA_STIFF, Context
    m = random_mesh_from_structured(6, p, seed=400 + p)
    rng = np.random.default_rng(40 + p)
    u = rng.uniform(-1, 1, m.n_dof)
    v = rng.normal(size=m.n_dof)
    km, kc = (K_POLY, (1.0, 0.0, 1.0)), (K_EXP, (0.8, 0.4))
    rm, rc = triangle_rule(2 * p), triangle_rule(min(8, 2 * p + 2))
    ctx = Context(device=0)
    ctx.set_element(p, *rm)
    ctx.mesh_upload(m.vert_xy, m.elem_vert, m.n_dof, m.elem_dof)
    ctx.set_rule(FEA_STIFF, *rc)
    ctx.build_pattern()
    ctx.set_coefficient(FEA_MASS, *km)
    ctx.set_coefficient(FEA_STIFF, *kc)
    perm = ctx.get_dof_perm()
    dev = "cuda:0"
    ul = torch.tensor(u[perm], dtype=torch.float64, device=dev)
    vl = torch.tensor(v[perm], dtype=torch.float64, device=dev)
    n = max(ctx.nnz, 1)
    M = torch.zeros(n, dtype=torch.float64, device=dev)
    K = torch.zeros(n, dtype=torch.float64, device=dev)
    ctx.assemble(ul, M, K)
    MT = torch.zeros(n, dtype=torch.float64, device=dev)
    CT = torch.zeros(n, dtype=torch.float64, device=dev)
    ctx.assemble_tensor(ul, vl, MT, CT)
    ctx.sync()
    mlib = copy.copy(m)
    from tests.helpers import lib_numbering
    mlib.elem_dof = lib_numbering(m, perm)
    refm = oracle.assemble(mlib, *rm, u[perm], m_coef=km, c_coef=kc, which=MASS)
    refc = oracle.assemble(mlib, *rc, u[perm], m_coef=km, c_coef=kc, which=STIFF)
    assert maxabs_rel(M[: ctx.nnz].cpu().numpy(), refm.M) <= TOL
    assert maxabs_rel(K[: ctx.nnz].cpu().numpy(), refc.K) <= TOL
    tm = oracle.assemble_tensor_contraction(mlib, *rm, u[perm], v[perm], m_coef=km)
    tc = oracle.assemble_tensor_contraction(mlib, *rc, u[perm], v[perm], c_coef=kc)
    assert maxabs_rel(MT[: ctx.nnz].cpu().numpy(), tm.M) <= TOL
    assert maxabs_rel(CT[: ctx.nnz].cpu().numpy(), tc.K) <= TOL
    # a different rule for M, then one common rule again
    ctx.set_rule(FEA_MASS, *rc)
    ctx.build_pattern()
    ctx.assemble(ul, M, K)
    ctx.sync()
    refm2 = oracle.assemble(mlib, *rc, u[perm], m_coef=km, c_coef=kc, which=MASS)
    assert maxabs_rel(M[: ctx.nnz].cpu().numpy(), refm2.M) <= TOL
    assert maxabs_rel(K[: ctx.nnz].cpu().numpy(), refc.K) <= TOL
    ctx.set_rule(FEA_MASS | FEA_STIFF, *rm)
    ctx.build_pattern()
    ctx.assemble(ul, M, K)
    ctx.sync()
    refb = oracle.assemble(mlib, *rm, u[perm], m_coef=km, c_coef=kc, which=MASS | STIFF)
    assert maxabs_rel(M[: ctx.nnz].cpu().numpy(), refb.M) <= TOL
    assert maxabs_rel(K[: ctx.nnz].cpu().numpy(), refb.K) <= TOL
    ctx.close()


@pytest.mark.parametrize("p", [1, 2, 3])
@pytest.mark.parametrize("kernel", [0, 4])
def test_assembling_more_than_planned(p, kernel):
    """A plan sized for one matrix (FEA_TUNE_PLAN_WHICH) serves the other matrix too (fea.h: one
    pass per matrix; the unplanned matrix takes the planned matrix's shared-memory V region)."""
    import torch
    from paper_2204_03893_b200.fea import Context
    m = random_mesh_from_structured(9, p, seed=70 + p)
    xy, w = triangle_rule(2 * p)
    u = np.random.default_rng(70 + p).uniform(-1, 1, m.n_dof)
    km, kc = (K_POLY, (1.0, 0.0, 1.0)), (K_EXP, (1.0, 0.5))
    for plan in (MASS, STIFF):
        ctx = Context(device=0)
        ctx.set_element(p, xy, w)
        ctx.mesh_upload(m.vert_xy, m.elem_vert, m.n_dof, m.elem_dof, reorder=True)
        ctx.set_tuning(4, plan)
        if kernel:
            ctx.set_tuning(2, kernel)
        _, _, nnz = ctx.build_pattern()
        ctx.set_coefficient(MASS, *km)
        ctx.set_coefficient(STIFF, *kc)
        perm = ctx.get_dof_perm()
        ul = torch.tensor(u[perm], dtype=torch.float64, device="cuda:0")
        ref = oracle_for(m, xy, w, u, perm, km, kc, MASS | STIFF)
        vm = torch.full((nnz,), np.nan, dtype=torch.float64, device="cuda:0")
        vc = torch.full((nnz,), np.nan, dtype=torch.float64, device="cuda:0")
        ctx.assemble(ul, vm, vc)
        ctx.sync()
        assert maxabs_rel(vm.cpu().numpy(), ref.M) <= TOL and maxabs_rel(vc.cpu().numpy(), ref.K) <= TOL
        vm.fill_(np.nan)
        vc.fill_(np.nan)
        ctx.assemble_stiffness(ul, vc)
        ctx.assemble_mass(ul, vm)
        ctx.sync()
        assert maxabs_rel(vm.cpu().numpy(), ref.M) <= TOL and maxabs_rel(vc.cpu().numpy(), ref.K) <= TOL
        ctx.close()
