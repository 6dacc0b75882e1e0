"""C-ABI checks that need no GPU: every function declared in include/fea.h is exported by
libfea.so, and the planning-only context (device -1) reproduces the oracle's pattern."""
import os
import re

import numpy as np
import pytest

import oracle
from fea_inputs import CONFIGS, make_workload, scaled, structured_mesh, triangle_rule
from fea_inputs.mesh import random_mesh_from_structured
from paper_2204_03893_b200 import fea
from tests.helpers import lib_numbering

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "fea.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fea_[a-z_0-9]+)\s*\(", src)))


def test_header_symbols_exported():
    lib = fea.load_library()
    names = _declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), f"{n} declared in fea.h but not exported"
    assert sorted(fea.SYMBOLS) == names


def _plan(m, p, world=1, rank=0, reorder=True, budget=0):
    ctx = fea.Context(device=-1, rank=rank, world=world)
    xy, w = triangle_rule(2 * p)
    ctx.set_element(p, xy, w)
    ctx.mesh_upload(m.vert_xy, m.elem_vert, m.n_dof, m.elem_dof, reorder=reorder)
    if budget:
        ctx.set_tuning(1, budget)
    ctx.build_pattern()
    return ctx


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_planning_pattern_bit_exact_vs_oracle(p):
    m = random_mesh_from_structured(6, p, seed=500 + p)
    for reorder in (True, False):
        ctx = _plan(m, p, reorder=reorder)
        perm = ctx.get_dof_perm()
        assert sorted(perm) == list(range(m.n_dof))
        if not reorder:
            assert np.array_equal(perm, np.arange(m.n_dof))
        rp, ci = ctx.get_pattern()
        orp, oci = oracle.pattern(m.n_dof, lib_numbering(m, perm))
        assert np.array_equal(rp, orp) and np.array_equal(ci, oci)
        assert ctx.stat(2) >= ctx.stat(3) == m.n_e  # visits >= owned = every element once
        eperm = ctx.get_elem_perm()
        assert sorted(eperm) == list(range(m.n_e))


@pytest.mark.parametrize("p,world", [(1, 3), (2, 2), (3, 4), (4, 3)])
def test_row_partition_concatenates(p, world):
    m = random_mesh_from_structured(5, p, seed=600 + p)
    base = _plan(m, p)
    brp, bci = base.get_pattern()
    rows, cols, nxt = [0], [], 0
    owned = 0
    for r in range(world):
        ctx = _plan(m, p, world=world, rank=r)
        assert ctx.row_begin == nxt
        nxt += ctx.n_rows
        rp, ci = ctx.get_pattern()
        rows += list(rp[1:] + rows[-1])
        cols.append(ci)
        owned += ctx.stat(3)
    assert nxt == m.n_dof and owned == m.n_e  # every element owned by exactly one block
    assert np.array_equal(np.array(rows), brp) and np.array_equal(np.concatenate(cols), bci)


def test_small_budgets_give_finer_tilings():
    m = random_mesh_from_structured(12, 2, seed=9)
    a = _plan(m, 2)
    b = _plan(m, 2, budget=40000)
    assert b.stat(1) > a.stat(1)
    assert np.array_equal(a.get_pattern()[1], b.get_pattern()[1])


def test_p1_blocks_in_whole_unit_rounds():
    """P1 (kernel v5): e_max is a multiple of 32 * 20 warps, so a block's 32-element units fill whole
    rounds over the warps (DESIGN 7.2); an explicit FEA_TUNE_EMAX is taken as given."""
    m = random_mesh_from_structured(40, 1, seed=11)
    a = _plan(m, 1)
    assert a.stat(7) >= 640 and a.stat(7) % 640 == 0
    ctx = fea.Context(device=-1)
    xy, w = triangle_rule(2)
    ctx.set_element(1, xy, w)
    ctx.mesh_upload(m.vert_xy, m.elem_vert, m.n_dof, m.elem_dof, reorder=True)
    ctx.set_tuning(3, 700)
    ctx.build_pattern()
    assert ctx.stat(7) == 696  # 700 rounded down to a multiple of 8 only
    assert ctx.stat(1) <= a.stat(1)
    assert np.array_equal(a.get_pattern()[1], ctx.get_pattern()[1])


def test_planning_errors():
    ctx = fea.Context(device=-1)
    xy, w = triangle_rule(2)
    with pytest.raises(fea.FeaError, match="FEA_E_ARG"):
        ctx.set_element(1, xy, 2 * w)
    with pytest.raises(fea.FeaError, match="FEA_E_STATE"):
        ctx.build_pattern()
    ctx.set_element(1, xy, w)
    with pytest.raises(fea.FeaError, match="degenerate element 0"):
        ctx.mesh_upload(np.array([[0.0, 0], [1, 0], [2, 0]]), np.array([[0, 1, 2]]), 3, np.array([[0, 1, 2]]))
    with pytest.raises(fea.FeaError, match="out of range"):
        ctx.mesh_upload(np.array([[0.0, 0], [1, 0], [0, 1]]), np.array([[0, 1, 2]]), 3, np.array([[0, 1, 5]]))
    with pytest.raises(fea.FeaError, match="not referenced"):
        ctx.mesh_upload(np.array([[0.0, 0], [1, 0], [0, 1]]), np.array([[0, 1, 2]]), 4, np.array([[0, 1, 2]]))
    m = structured_mesh(2, 3)
    ctx.set_element(3, *triangle_rule(6))
    bad = m.elem_dof.copy()
    bad[0, [3, 4]] = bad[0, [4, 3]]
    with pytest.raises(fea.FeaError, match="inconsistently"):
        ctx.mesh_upload(m.vert_xy, m.elem_vert, m.n_dof, bad)
    with pytest.raises(fea.FeaError, match="FEA_E_ARG"):
        ctx.set_coefficient(3, 2, [0.0, 1.0, -1.0, 2.0])  # PWL breakpoints must increase
    with pytest.raises(fea.FeaError, match="FEA_E_STATE"):
        ctx.mesh_upload(m.vert_xy, m.elem_vert, m.n_dof, m.elem_dof)
        ctx.build_pattern()
        ctx.sync()  # planning-only contexts have no device


def test_config_nnz_matches_survey():
    """Structural nnz of the configs at a reduced size and the formula."""
    for name in ("C1", "C2"):
        cfg = CONFIGS[name]
        w = make_workload(cfg)
        ctx = _plan(w.mesh, cfg.p)
        assert ctx.nnz == {"C1": 7361, "C2": 3018753}[name]


def test_pattern_rows_window_matches_full_pattern():
    """fea_get_pattern_rows returns the rows [r0, r1) of the full local pattern (planning-only)."""
    from fea_inputs import triangle_rule
    from fea_inputs.mesh import random_mesh_from_structured
    from paper_2204_03893_b200.fea import Context
    m = random_mesh_from_structured(9, 2, seed=5)
    ctx = Context(device=-1)
    ctx.set_element(2, *triangle_rule(4))
    ctx.mesh_upload(m.vert_xy, m.elem_vert, m.n_dof, m.elem_dof)
    ctx.build_pattern()
    rp, ci = ctx.get_pattern()
    for r0, r1 in ((0, 5), (17, 60), (m.n_dof - 9, m.n_dof), (12, 12)):
        wrp, wci = ctx.get_pattern_rows(r0, r1)
        assert np.array_equal(wrp, rp[r0:r1 + 1])
        assert np.array_equal(wci, ci[rp[r0]:rp[r1]])
    ctx.close()


def test_tuning_keys_validated_and_plan_invariant():
    """fea_set_tuning rejects unknown keys and out-of-range values (FEA_E_ARG) and leaves the
    context usable; tuning keys that only change the kernel-side plan (v5 padding, tensor kernel)
    keep the CSR pattern bit-identical."""
    m = random_mesh_from_structured(6, 2, seed=520)
    base = _plan(m, 2)
    rp0, ci0 = base.get_pattern()
    for key, bad in ((2, 3), (3, -1), (4, 0), (5, 2), (7, 2), (8, 2), (10, 2), (99, 0)):
        ctx = fea.Context(device=-1)
        xy, w = triangle_rule(4)
        ctx.set_element(2, xy, w)
        ctx.mesh_upload(m.vert_xy, m.elem_vert, m.n_dof, m.elem_dof)
        with pytest.raises(fea.FeaError):
            ctx.set_tuning(key, bad)
        ctx.build_pattern()  # still usable after the rejected value
        rp, ci = ctx.get_pattern()
        assert np.array_equal(rp, rp0) and np.array_equal(ci, ci0)
    for key, val in ((10, 0), (8, 1), (8, 4), (2, 4)):
        ctx = fea.Context(device=-1)
        xy, w = triangle_rule(4)
        ctx.set_element(2, xy, w)
        ctx.mesh_upload(m.vert_xy, m.elem_vert, m.n_dof, m.elem_dof)
        ctx.set_tuning(key, val)
        ctx.build_pattern()
        rp, ci = ctx.get_pattern()
        assert np.array_equal(rp, rp0) and np.array_equal(ci, ci0)
