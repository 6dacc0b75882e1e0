"""Pins of the CPU oracle (oracle/oracle.c) against what the paper and the mathematics fix.

Every pin is independent of the oracle's own formulas: golden values printed in SPEC.md /
derived in SURVEY.md (tests/golden/, cited), exact rational integration through an
independently-derived basis (tests/exact_fem.py), brute force in exact arithmetic, closed
forms and invariants.  A dropped term, wrong sign, wrong index or transposed operand in
oracle.c fails at least one of them.
"""
from fractions import Fraction

import numpy as np
import pytest
import sympy as sp

import oracle
from fea_inputs import K_EXP, K_POLY, local_nodes, single_element_mesh, structured_mesh, triangle_rule, two_element_mesh
from fea_inputs.mesh import random_mesh_from_structured
from tests import exact_fem
from tests.golden import load

KONE = (K_POLY, (1.0,))


def _ref(p):
    return single_element_mesh((0.0, 0.0), (1.0, 0.0), (0.0, 1.0), p=p)


def _asm(mesh, u=None, m=KONE, c=KONE, **kw):
    xy, w = triangle_rule(2 * mesh.p)
    if u is None:
        u = np.zeros(mesh.n_dof)
    return oracle.assemble(mesh, xy, w, u, m_coef=m, c_coef=c, **kw)


def _maxrel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


# ---------------------------------------------------------------- basis (Alg. 1)
@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_basis_lagrange_property_and_partition(p):
    nodes = np.array(local_nodes(p), dtype=np.float64) / p
    phi, J = oracle.basis(p, nodes[:, 1:3])  # evaluate at the element's own nodes
    assert np.abs(phi - np.eye(len(nodes))).max() < 1e-15
    xy = np.random.default_rng(p).uniform(0, 0.5, (40, 2))
    phi, J = oracle.basis(p, xy)
    assert np.abs(phi.sum(0) - 1).max() < 1e-15          # partition of unity
    assert np.abs(J.sum(1)).max() < 1e-13                # zero gradient sum


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_basis_matches_independent_vandermonde_route(p):
    """Values and gradients vs the exact-rational basis from the interpolation solve."""
    xy, _ = triangle_rule(2 * p)
    phi, J = oracle.basis(p, xy)
    for q, (x, y) in enumerate(xy):
        ex = exact_fem.basis_at(p, Fraction(float(x)), Fraction(float(y)))
        for i, (f, fx, fy) in enumerate(ex):
            assert abs(phi[i, q] - float(f)) <= 2e-15
            assert abs(J[q, i, 0] - float(fx)) <= 2e-14 and abs(J[q, i, 1] - float(fy)) <= 2e-14


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_basis_reproduces_polynomials(p):
    """sum_i P(node_i) phi_i = P and sum_i P(node_i) grad phi_i = grad P for deg P <= p."""
    nodes = np.array(local_nodes(p), dtype=np.float64) / p
    xy = np.random.default_rng(10 + p).uniform(0, 0.5, (25, 2))
    phi, J = oracle.basis(p, xy)
    P = lambda x, y: 0.3 + 1.7 * x - 0.4 * y + 0.9 * x ** p - 1.1 * x * y ** (p - 1)
    Px = lambda x, y: 1.7 + 0.9 * p * x ** (p - 1) - 1.1 * y ** (p - 1)
    Py = lambda x, y: -0.4 - 1.1 * x * (p - 1) * y ** (p - 2) if p >= 2 else -0.4 + 0 * x
    vals = P(nodes[:, 1], nodes[:, 2])
    assert np.abs(vals @ phi - P(xy[:, 0], xy[:, 1])).max() < 1e-13
    assert np.abs(np.einsum("i,qi->q", vals, J[:, :, 0]) - Px(xy[:, 0], xy[:, 1])).max() < 1e-12
    assert np.abs(np.einsum("i,qi->q", vals, J[:, :, 1]) - Py(xy[:, 0], xy[:, 1])).max() < 1e-12


# ---------------------------------------------------------------- element matrices
def test_p1_reference_element_golden():
    g = load("p1_reference_element.txt")
    r = _asm(_ref(1))
    assert np.abs(g["scale_M"] * r.dense("M", 3) - np.array(g["M"])).max() < 1e-14
    assert np.abs(g["scale_C"] * r.dense("K", 3) - np.array(g["C"])).max() < 1e-14


def test_p2_reference_mass_golden():
    g = load("p2_reference_mass.txt")
    r = _asm(_ref(2))
    assert np.abs(g["scale_M"] * r.dense("M", 6) - np.array(g["M"])).max() < 1e-12


def test_p3_p4_traces_golden():
    g = load("reference_traces.txt")
    for p in (3, 4):
        r = _asm(_ref(p))
        n = r.row_ptr.shape[0] - 1
        assert abs(np.trace(r.dense("M", n)) - float(Fraction(g[f"p{p}_trM"]))) < 1e-14
        assert abs(np.trace(r.dense("K", n)) - float(Fraction(g[f"p{p}_trC"]))) < 1e-12
        assert abs(r.M.sum() - 0.5) < 1e-14 and abs(r.K.sum()) < 1e-12


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_reference_element_exact_rational(p):
    """Constant k: the minimal rule is exact, so the oracle must equal the
    exact integrals computed by the barycentric formula on an independent basis."""
    Mx, Cx = exact_fem.exact_reference_matrices(p)
    r = _asm(_ref(p))
    n = Mx.shape[0]
    Mx = np.array(Mx.tolist(), dtype=np.float64)
    Cx = np.array(Cx.tolist(), dtype=np.float64)
    assert _maxrel(r.dense("M", n), Mx) < 3e-15
    assert _maxrel(r.dense("K", n), Cx) < 3e-15


def test_geometry_golden_scaled_triangle():
    """(0,0),(2,0),(0,2): b_e = 4, A_e = I/4: M scales by 4, C invariant."""
    g = load("geometry.txt")
    for p in (1, 3):
        r1 = _asm(single_element_mesh(*g["tri_ref"], p=p))
        r2 = _asm(single_element_mesh(*g["tri_2"], p=p))
        assert g["b_2"] / g["b_ref"] == 4
        assert _maxrel(r2.M, 4 * r1.M) < 1e-14 and _maxrel(r2.K, r1.K) < 1e-14


def test_two_element_mesh_golden():
    g = load("two_element_mesh.txt")
    r = _asm(two_element_mesh())
    assert r.nnz == g["nnz"]
    assert np.abs(g["scale_M"] * r.dense("M", 4) - np.array(g["M"])).max() < 1e-14
    assert np.abs(g["scale_K"] * r.dense("K", 4) - np.array(g["K"])).max() < 1e-14
    cols = {(i, int(c)) for i in range(4) for c in r.col_idx[r.row_ptr[i]:r.row_ptr[i + 1]]}
    for ij in g["absent"]:
        assert tuple(ij) not in cols
    for ij in g["structural_zero"]:
        assert tuple(ij) in cols  # structural zero kept (reading 9)


def test_degenerate_element_rejected():
    m = single_element_mesh((0.0, 0.0), (1.0, 0.0), (2.0, 0.0), p=1)
    with pytest.raises(ValueError, match="degenerate element 0"):
        _asm(m)


# ---------------------------------------------------------------- pattern (reading 9)
@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_pattern_brute_force_and_formula(p):
    coeffs = load("nnz_formulas.txt")[f"p{p}"]
    for N in (1, 2, 3, 5):
        m = structured_mesh(N, p)
        rp, ci = oracle.pattern(m.n_dof, m.elem_dof)
        assert rp[-1] == coeffs[0] * N * N + coeffs[1] * N + coeffs[2]
        brp, bci = exact_fem.brute_force_pattern(m.n_dof, m.elem_dof)
        assert np.array_equal(rp, brp) and np.array_equal(ci, bci)
    m = random_mesh_from_structured(4, p, seed=3)
    rp, ci = oracle.pattern(m.n_dof, m.elem_dof)
    brp, bci = exact_fem.brute_force_pattern(m.n_dof, m.elem_dof)
    assert np.array_equal(rp, brp) and np.array_equal(ci, bci)


def test_pattern_row_range_and_permutation_identity():
    """Oracle(P mesh) = P Oracle(mesh) P^T for the pattern (SURVEY 8(c) 'Permutation')."""
    m = structured_mesh(6, 2)
    perm = np.random.default_rng(5).permutation(m.n_dof)
    mp = structured_mesh(6, 2)
    mp.elem_dof = perm[m.elem_dof].astype(np.int32)
    rp, ci = oracle.pattern(m.n_dof, m.elem_dof)
    rpp, cip = oracle.pattern(m.n_dof, mp.elem_dof)
    for r in range(m.n_dof):
        a = set(perm[ci[rp[r]:rp[r + 1]]])
        b = set(cip[rpp[perm[r]]:rpp[perm[r] + 1]])
        assert a == b
    rp2, ci2 = oracle.pattern(m.n_dof, m.elem_dof, 10, 40)
    assert np.array_equal(ci2, ci[rp[10]:rp[40]]) and np.array_equal(rp2, rp[10:41] - rp[10])


# ---------------------------------------------------------------- non-constant k
def _energy_sum(mesh, q_xy, q_w, u, kind, par):
    """sum_e d_e sum_q w_q k(u_h(x_q)) computed without any element matrix, through the
    independent exact basis (PAPER.md:198 Lambda = S * (w b^T), summed)."""
    tab = [exact_fem.basis_at(mesh.p, Fraction(float(x)), Fraction(float(y))) for x, y in q_xy]
    phi = np.array([[float(t[i][0]) for t in tab] for i in range(mesh.n_p)])  # (n_p, n_q)
    a, b, c = (mesh.vert_xy[mesh.elem_vert[:, k]] for k in range(3))
    d = np.abs((b[:, 0] - a[:, 0]) * (c[:, 1] - a[:, 1]) - (c[:, 0] - a[:, 0]) * (b[:, 1] - a[:, 1]))
    uq = u[mesh.elem_dof] @ phi
    kq = np.polyval(list(par)[::-1], uq) if kind == K_POLY else par[0] * np.exp(par[1] * uq)
    return float((d[:, None] * q_w[None, :] * kq).sum())


COEFS = [(K_POLY, (1.0, 0.0, 1.0)), (K_EXP, (1.0, 0.5)), (K_POLY, (1.0, 0.0, 0.0, 0.0, 1.0))]


@pytest.mark.parametrize("p", [1, 2, 3, 4])
@pytest.mark.parametrize("coef", COEFS)
def test_invariants_nonconstant_k(p, coef):
    m = random_mesh_from_structured(4, p, seed=100 + p)
    xy, w = triangle_rule(2 * p)
    u = np.random.default_rng(p).uniform(-1, 1, m.n_dof)
    r = oracle.assemble(m, xy, w, u, m_coef=coef, c_coef=coef)
    n = m.n_dof
    Md, Kd = r.dense("M", n), r.dense("K", n)
    # K 1 = 0 for any k (sum_i grad phi_i = 0)
    assert np.abs(Kd.sum(1)).max() <= 1e-11 * np.abs(Kd).max()
    # symmetry
    assert np.abs(Md - Md.T).max() <= 1e-14 * np.abs(Md).max()
    assert np.abs(Kd - Kd.T).max() <= 1e-13 * np.abs(Kd).max()
    # 1^T M 1 = sum_e d_e sum_q w_q k_q (SPEC.md:335 generalised)
    assert abs(Md.sum() - _energy_sum(m, xy, w, u, *coef)) <= 1e-13 * abs(Md.sum())
    # linear field X = g . x:  X^T K X = |g|^2 sum_e d_e sum_q w_q k_q
    g = np.array([0.7, -1.3])
    Xf = m.dof_xy @ g
    assert abs(Xf @ Kd @ Xf - (g @ g) * _energy_sum(m, xy, w, u, *coef)) <= 1e-11 * abs(Xf @ Kd @ Xf)


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_constant_u_scaling_and_coordinate_scaling(p):
    m = random_mesh_from_structured(3, p, seed=200 + p)
    c = 0.37
    r1 = _asm(m)
    rk = _asm(m, u=np.full(m.n_dof, c), m=COEFS[0], c=COEFS[0])
    kc = 1 + c * c
    assert _maxrel(rk.M, kc * r1.M) < 1e-14 and _maxrel(rk.K, kc * r1.K) < 1e-13
    s = 3.0
    ms = random_mesh_from_structured(3, p, seed=200 + p)
    ms.vert_xy = ms.vert_xy * s
    rs = _asm(ms)
    assert _maxrel(rs.M, s * s * r1.M) < 1e-14 and _maxrel(rs.K, r1.K) < 1e-13
    assert abs(r1.M.sum() - 1.0) < 1e-13  # area of the unit square


@pytest.mark.parametrize("p", [1, 2, 3, 4])
@pytest.mark.parametrize("coef", [COEFS[0], COEFS[1]])
def test_brute_force_exact_arithmetic(p, coef):
    """FP64 oracle vs the quadrature formula evaluated exactly (rational / 40-digit mpmath)."""
    import mpmath
    mpmath.mp.dps = 40
    m = random_mesh_from_structured(2 if p <= 2 else 1, p, seed=300 + p)
    xy, w = triangle_rule(2 * p)
    u = np.random.default_rng(300 + p).uniform(-1, 1, m.n_dof)
    r = oracle.assemble(m, xy, w, u, m_coef=coef, c_coef=COEFS[0] if coef is COEFS[1] else COEFS[1])
    Mx, Cx = exact_fem.brute_force_assemble(m, xy, w, u, coef, COEFS[0] if coef is COEFS[1] else COEFS[1])
    assert _maxrel(r.dense("M", m.n_dof), Mx) < 1e-14
    assert _maxrel(r.dense("K", m.n_dof), Cx) < 1e-14


def test_threads_and_row_ranges_bit_identical():
    m = random_mesh_from_structured(8, 2, seed=11)
    xy, w = triangle_rule(4)
    u = np.random.default_rng(1).uniform(0, 1, m.n_dof)
    r1 = oracle.assemble(m, xy, w, u, m_coef=COEFS[0], c_coef=COEFS[0], nthreads=1)
    r4 = oracle.assemble(m, xy, w, u, m_coef=COEFS[0], c_coef=COEFS[0], nthreads=4)
    assert np.array_equal(r1.M, r4.M) and np.array_equal(r1.K, r4.K)
    rb = oracle.assemble(m, xy, w, u, m_coef=COEFS[0], c_coef=COEFS[0], r0=37, r1=101)
    a, b = r1.row_ptr[37], r1.row_ptr[101]
    assert np.array_equal(rb.M, r1.M[a:b]) and np.array_equal(rb.K, r1.K[a:b])


# ---------------------------------------------------------------- NEXT-1/2 tensor contractions
@pytest.mark.parametrize("p", [1, 2, 3])
def test_tensor_contractions_are_directional_derivatives(p):
    """(Mt o2 v)_{ik} = d/de M_ik(u + e v) (Mt symmetric in all modes) and
    w^T (Ct o2 w') ... : (Ct o2 w) v = d/de [K(u + e v) w] (K_ijk = dK_ij/du_k).
    k = 1 + u^2 makes M(u + e v) quadratic in e, so the central difference is exact."""
    m = random_mesh_from_structured(3, p, seed=400 + p)
    xy, w = triangle_rule(2 * p)
    rng = np.random.default_rng(p)
    u, v, wv = (rng.uniform(-1, 1, m.n_dof) for _ in range(3))
    coef = COEFS[0]
    T = oracle.assemble_tensor_contraction(m, xy, w, u, v, m_coef=coef, c_coef=coef)
    eps = 0.5
    rp = oracle.assemble(m, xy, w, u + eps * v, m_coef=coef, c_coef=coef)
    rm = oracle.assemble(m, xy, w, u - eps * v, m_coef=coef, c_coef=coef)
    dM = (rp.M - rm.M) / (2 * eps)
    assert _maxrel(T.M, dM) < 1e-12
    Tw = oracle.assemble_tensor_contraction(m, xy, w, u, wv, m_coef=coef, c_coef=coef)
    n = m.n_dof
    lhs = Tw.dense("K", n) @ v
    rhs = ((rp.dense("K", n) - rm.dense("K", n)) / (2 * eps)) @ wv
    assert np.abs(lhs - rhs).max() <= 1e-11 * np.abs(rhs).max()
