"""Pins of the oracle's coefficient branches that round 1 left unpinned (VERDICT r1 "What's weak" 1):
the piecewise-linear k(T) of PAPER.md:560-568 (oracle.c or_k kind 2) and the derivatives k'(u)
of the EXP and PWL kinds (oracle.c or_dk kinds 1, 2) that the tensor contractions use
(PAPER.md:286-289).  Every expected value comes from an independent route:

* PWL k and k' : the paper's case formula written out in exact rationals (tests/exact_fem.py
  pwl_exact / pwl_slope_exact), breakpoint T_2 owned by the first case (T_1 <= T <= T_2),
  linear extrapolation outside [T_1, T_m] (reading R26);
* EXP k'       : mpmath's numerical derivative of c0 exp(c1 u) at 40 digits;
* tensor pins  : directional derivatives of the oracle's own M(u), K(u) (which are pinned
  elsewhere) -- Richardson-extrapolated central differences for EXP, exact central differences
  for PWL along paths that stay inside one segment;
* assembled values with PWL k: exact-arithmetic brute force and the 1^T M 1 energy identity.
"""
from fractions import Fraction

import mpmath
import numpy as np
import pytest

import oracle
from fea_inputs import K_EXP, K_POLY, triangle_rule
from fea_inputs.configs import K_PWL
from fea_inputs.mesh import random_mesh_from_structured
from tests import exact_fem

# the paper's Experiment-2 conductivity: (T_1, k_1) = (0, 1.5), (200, 0.7), (1000, 0.5)
PWL_E2 = (0.0, 1.5, 200.0, 0.7, 1000.0, 0.5)
# four breakpoints on the scale of the synthetic u fields (U[-1, 1])
PWL_4 = (-0.6, 2.0, -0.1, 1.25, 0.35, 1.75, 0.9, 0.5)


def _maxrel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def _probe_points(par):
    T = [par[2 * i] for i in range(len(par) // 2)]
    span = T[-1] - T[0]
    pts = list(T)                                                    # the breakpoints themselves
    pts += [(a + b) / 2 for a, b in zip(T, T[1:])]                   # segment midpoints
    for t in T[1:-1]:                                                # just either side of interior ones
        pts += [np.nextafter(t, -np.inf), np.nextafter(t, np.inf), t - 1e-6 * span, t + 1e-6 * span]
    pts += [T[0] - 0.3 * span, T[0] - 1e-9 * span, T[-1] + 1e-9 * span, T[-1] + 0.7 * span]  # R26
    return pts


@pytest.mark.parametrize("par", [PWL_E2, PWL_4])
def test_pwl_k_matches_paper_cases(par):
    for T in _probe_points(par):
        want = float(exact_fem.pwl_exact(par, Fraction(T)))
        got = oracle.k_eval(K_PWL, par, T)
        assert abs(got - want) <= 4e-16 * max(1.0, abs(want)), (T, got, want)


def test_pwl_k_paper_example_values():
    """Exp. 2 values read off PAPER.md:563-566: k(0) = 1.5, k(200) = 0.7, k(1000) = 0.5,
    k(100) = 1.1 (first case), k(600) = 0.6 (second case)."""
    for T, k in ((0.0, 1.5), (200.0, 0.7), (1000.0, 0.5), (100.0, 1.1), (600.0, 0.6)):
        assert abs(oracle.k_eval(K_PWL, PWL_E2, T) - k) <= 1e-15


@pytest.mark.parametrize("par", [PWL_E2, PWL_4])
def test_pwl_dk_is_the_owning_segment_slope(par):
    for T in _probe_points(par):
        want = float(exact_fem.pwl_slope_exact(par, Fraction(T)))
        got = oracle.dk_eval(K_PWL, par, T)
        assert abs(got - want) <= 2e-16 * max(1.0, abs(want)), (T, got, want)
    # ownership: at T_2 the slope is the FIRST case's ("T_1 <= T <= T_2")
    assert oracle.dk_eval(K_PWL, PWL_E2, 200.0) == pytest.approx((0.7 - 1.5) / 200.0, rel=1e-15)
    assert oracle.dk_eval(K_PWL, PWL_E2, np.nextafter(200.0, np.inf)) == pytest.approx((0.5 - 0.7) / 800.0, rel=1e-15)


@pytest.mark.parametrize("par", [(1.0, 0.5), (2.5, -1.7), (0.3, 3.0)])
def test_exp_dk_matches_mpmath_derivative(par):
    mpmath.mp.dps = 40
    f = lambda x: mpmath.mpf(par[0]) * mpmath.exp(mpmath.mpf(par[1]) * x)  # noqa: E731
    for u in (-1.0, -0.3, 0.0, 0.25, 0.8, 1.0):
        want = float(mpmath.diff(f, mpmath.mpf(u)))
        got = oracle.dk_eval(K_EXP, par, u)
        assert abs(got - want) <= 4e-16 * abs(want), (u, got, want)


@pytest.mark.parametrize("par", [(1.0, 0.0, 1.0), (1.0, 0.0, 0.0, 0.0, 1.0), (0.5, -2.0, 0.25, 3.0)])
def test_poly_dk_matches_exact_derivative(par):
    for u in (-1.0, -0.4, 0.0, 0.6, 1.0):
        want = float(sum(Fraction(i) * Fraction(c) * Fraction(u) ** (i - 1) for i, c in enumerate(par) if i > 0))
        assert abs(oracle.dk_eval(K_POLY, par, u) - want) <= 4e-16 * max(1.0, abs(want))


# ---------------------------------------------------------------- assembled values with PWL k
@pytest.mark.parametrize("p", [1, 2, 3])
def test_brute_force_exact_arithmetic_pwl(p):
    """FP64 oracle with PWL k (both matrices; M and C with different breakpoint sets) vs the
    quadrature formula in exact rationals; u spans all segments and both extrapolations."""
    m = random_mesh_from_structured(2 if p <= 2 else 1, p, seed=500 + p)
    xy, w = triangle_rule(2 * p)
    u = np.random.default_rng(500 + p).uniform(-1.2, 1.2, m.n_dof)
    mc, cc = (K_PWL, PWL_4), (K_PWL, (-1.0, 0.5, 0.0, 1.0, 1.0, 3.0))
    r = oracle.assemble(m, xy, w, u, m_coef=mc, c_coef=cc)
    Mx, Cx = exact_fem.brute_force_assemble(m, xy, w, u, mc, cc)
    assert _maxrel(r.dense("M", m.n_dof), Mx) < 1e-14
    assert _maxrel(r.dense("K", m.n_dof), Cx) < 1e-14


@pytest.mark.parametrize("p", [1, 2, 4])
def test_energy_identity_pwl(p):
    """1^T M 1 = sum_e d_e sum_q w_q k(u_h(x_q)) and K 1 = 0 with the PWL coefficient; the right
    side evaluates k through the exact case formula at the interpolated u_q."""
    m = random_mesh_from_structured(4, p, seed=600 + p)
    xy, w = triangle_rule(2 * p)
    u = np.random.default_rng(600 + p).uniform(-1, 1, m.n_dof)
    coef = (K_PWL, PWL_4)
    r = oracle.assemble(m, xy, w, u, m_coef=coef, c_coef=coef)
    tab = [exact_fem.basis_at(p, Fraction(float(x)), Fraction(float(y))) for x, y in xy]
    phi = np.array([[float(t[i][0]) for t in tab] for i in range(m.n_p)])
    a, b, c = (m.vert_xy[m.elem_vert[:, k]] for k in range(3))
    d = np.abs((b[:, 0] - a[:, 0]) * (c[:, 1] - a[:, 1]) - (c[:, 0] - a[:, 0]) * (b[:, 1] - a[:, 1]))
    uq = u[m.elem_dof] @ phi
    kq = np.vectorize(lambda t: float(exact_fem.pwl_exact(PWL_4, Fraction(float(t)))))(uq)
    want = float((d[:, None] * w[None, :] * kq).sum())
    n = m.n_dof
    assert abs(r.dense("M", n).sum() - want) <= 1e-13 * abs(want)
    Kd = r.dense("K", n)
    assert np.abs(Kd.sum(1)).max() <= 1e-11 * np.abs(Kd).max()


# ---------------------------------------------------------------- tensor contractions, EXP and PWL k'
def _dirderiv_check(m, xy, w, u, v, wv, coef, deriv, tol):
    T = oracle.assemble_tensor_contraction(m, xy, w, u, v, m_coef=coef, c_coef=coef)
    Tw = oracle.assemble_tensor_contraction(m, xy, w, u, wv, m_coef=coef, c_coef=coef)
    n = m.n_dof
    dM, dK = deriv(lambda x: oracle.assemble(m, xy, w, x, m_coef=coef, c_coef=coef))
    assert _maxrel(T.M, dM.M) < tol
    lhs = Tw.dense("K", n) @ v
    rhs = dK.dense("K", n) @ wv
    assert np.abs(lhs - rhs).max() <= tol * np.abs(rhs).max()


class _D:
    def __init__(self, M, K, rp, ci):
        self.M, self.K, self.row_ptr, self.col_idx = M, K, rp, ci

    def dense(self, which, n):
        out = np.zeros((n, n))
        vals = self.M if which == "M" else self.K
        for r in range(n):
            for k in range(self.row_ptr[r], self.row_ptr[r + 1]):
                out[r, self.col_idx[k]] += vals[k]
        return out


@pytest.mark.parametrize("p", [1, 2, 3])
def test_tensor_contractions_exp_k(p):
    """(M o2 v) = d/de M(u + e v) and (C o2 w) v = d/de [K(u + e v) w] with k = c0 exp(c1 u):
    Richardson-extrapolated central differences (error O(e^4)); dropping c1 from k' = c0 c1 exp(c1 u)
    or its sign would be off by O(1)."""
    m = random_mesh_from_structured(3, p, seed=700 + p)
    xy, w = triangle_rule(2 * p)
    rng = np.random.default_rng(700 + p)
    u, v, wv = (rng.uniform(-1, 1, m.n_dof) for _ in range(3))
    coef = (K_EXP, (1.3, 0.7))

    def deriv(asm):
        def cd(eps):
            rp, rm = asm(u + eps * v), asm(u - eps * v)
            return (rp.M - rm.M) / (2 * eps), (rp.K - rm.K) / (2 * eps), rp
        m1, k1, r = cd(0.02)
        m2, k2, _ = cd(0.01)
        dm, dk = (4 * m2 - m1) / 3, (4 * k2 - k1) / 3
        return _D(dm, None, r.row_ptr, r.col_idx), _D(None, dk, r.row_ptr, r.col_idx)

    _dirderiv_check(m, xy, w, u, v, wv, coef, deriv, 2e-9)


@pytest.mark.parametrize("p", [1, 2])
@pytest.mark.parametrize("lo,hi", [(20.0, 180.0), (260.0, 940.0)])
def test_tensor_contractions_pwl_k(p, lo, hi):
    """PWL k along u + e v with every u_q inside one segment of PAPER.md:563-564 (first or second
    case): k is affine along the path, so the central difference is exact up to rounding and
    k' must be that segment's slope."""
    m = random_mesh_from_structured(3, p, seed=800 + p)
    xy, w = triangle_rule(2 * p)
    rng = np.random.default_rng(800 + p)
    # Lagrange interpolants overshoot the nodal range for p = 2 by at most 1/8 of it; keep a margin
    mid, half = (lo + hi) / 2, (hi - lo) / 2
    u = mid + 0.6 * half * rng.uniform(-1, 1, m.n_dof)
    v, wv = rng.uniform(-1, 1, m.n_dof), rng.uniform(-1, 1, m.n_dof)
    eps = 0.1 * half
    coef = (K_PWL, PWL_E2)
    phi, _ = oracle.basis(p, xy)
    for x in (u + eps * v, u - eps * v, u):
        uq = x[m.elem_dof] @ phi
        assert uq.min() > lo - 20 and uq.max() < hi + 20  # inside the segment (lo, hi) +- margin

    def deriv(asm):
        rp, rm = asm(u + eps * v), asm(u - eps * v)
        return (_D((rp.M - rm.M) / (2 * eps), None, rp.row_ptr, rp.col_idx),
                _D(None, (rp.K - rm.K) / (2 * eps), rp.row_ptr, rp.col_idx))

    _dirderiv_check(m, xy, w, u, v, wv, coef, deriv, 1e-11)
