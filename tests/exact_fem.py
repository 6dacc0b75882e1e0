"""Independent exact-arithmetic finite-element helpers used to PIN the oracle.

Nothing here is shared with oracle/oracle.c or with the CUDA path.  The routes are
deliberately different from the oracle's:
  * the Lagrange basis is obtained by solving the interpolation (Vandermonde) system in
    exact rationals (the oracle uses the barycentric product formula in long double);
  * exact element integrals use the barycentric-monomial formula
      int_T l1^a l2^b l3^c = a! b! c! 2|T| / (a+b+c+2)!
    on the reference triangle (no quadrature at all);
  * the quadrature-formula brute force evaluates PAPER.md:134-135 in exact rationals
    (all FP64 inputs taken as exact binary fractions), with mpmath only for exp().
"""
from __future__ import annotations

from fractions import Fraction
from functools import lru_cache
from math import factorial

import mpmath
import numpy as np
import sympy as sp

from fea_inputs.mesh import local_nodes

X, Y = sp.symbols("x y")


@lru_cache(maxsize=None)
def monomials(p: int):
    return [(a, d - a) for d in range(p + 1) for a in range(d, -1, -1)]


@lru_cache(maxsize=None)
def lagrange_coeffs(p: int):
    """Coefficient matrix Cf (n_p x n_mono) of phi_i = sum_m Cf[i,m] x^a y^b, exact rationals,
    from Vandermonde V[node, mono] and phi(node_j) = delta_ij  =>  Cf = V^{-T}."""
    mons = monomials(p)
    nodes = local_nodes(p)
    V = sp.Matrix([[sp.Rational(k1, p) ** a * sp.Rational(k2, p) ** b for (a, b) in mons]
                   for (_k0, k1, k2) in nodes])
    Cf = V.inv().T
    return Cf, mons


def basis_polys(p: int):
    Cf, mons = lagrange_coeffs(p)
    n = Cf.shape[0]
    return [sp.expand(sum(Cf[i, m] * X ** a * Y ** b for m, (a, b) in enumerate(mons))) for i in range(n)]


@lru_cache(maxsize=None)
def _poly_dicts(p: int):
    """phi_i and their x/y derivatives as {(a, b): Fraction} dicts."""
    out = []
    for f in basis_polys(p):
        fx, fy = sp.diff(f, X), sp.diff(f, Y)
        ds = []
        for g in (f, fx, fy):
            P = sp.Poly(g, X, Y)
            ds.append({m: Fraction(int(c.p), int(c.q)) for m, c in zip(P.monoms(), P.coeffs())})
        out.append(tuple(ds))
    return out


def _ev(d, x, y):
    return sum(c * x ** a * y ** b for (a, b), c in d.items())


def basis_at(p: int, x: Fraction, y: Fraction):
    """(phi_i, dphi_i/dx, dphi_i/dy) exact at a rational point."""
    return [(_ev(f, x, y), _ev(fx, x, y), _ev(fy, x, y)) for (f, fx, fy) in _poly_dicts(p)]


def _int_ref_monomial(a: int, b: int) -> Fraction:
    """int over reference triangle of x^a y^b = a! b! / (a+b+2)!  (barycentric formula, |T|=1/2)."""
    return Fraction(factorial(a) * factorial(b), factorial(a + b + 2))


def exact_reference_matrices(p: int):
    """Exact M and C (k = 1) on the reference triangle (0,0),(1,0),(0,1) as sympy Rationals."""
    phis = basis_polys(p)
    n = len(phis)

    def integ(expr):
        P = sp.Poly(sp.expand(expr), X, Y)
        return sum(sp.Rational(c) * sp.Rational(_int_ref_monomial(a, b).numerator, _int_ref_monomial(a, b).denominator)
                   for (a, b), c in zip(P.monoms(), P.coeffs()))

    M = sp.zeros(n, n)
    C = sp.zeros(n, n)
    for i in range(n):
        for j in range(i, n):
            M[i, j] = M[j, i] = integ(phis[i] * phis[j])
            C[i, j] = C[j, i] = integ(sp.diff(phis[i], X) * sp.diff(phis[j], X) + sp.diff(phis[i], Y) * sp.diff(phis[j], Y))
    return M, C


def k_exact(kind: int, par, u):
    """k(u) exactly (Fraction) for polynomials; mpmath (current dps) for exp."""
    if kind == 0:
        r = Fraction(0)
        for c in reversed(par):
            r = r * u + Fraction(c)
        return r
    if kind == 1:
        return mpmath.mpf(par[0]) * mpmath.exp(mpmath.mpf(par[1]) * mpmath.mpf(u.numerator) / u.denominator)
    if kind == 2:
        return pwl_exact(par, u)
    raise ValueError(kind)


def _pwl_pairs(par):
    pts = [(Fraction(par[2 * i]), Fraction(par[2 * i + 1])) for i in range(len(par) // 2)]
    assert all(pts[i][0] < pts[i + 1][0] for i in range(len(pts) - 1))
    return pts


def _pwl_segment(pts, T):
    """Segment index s of T: the first case is T_1 <= T <= T_2 (T_2 belongs to
    it), the following ones T_s < T <= T_{s+1}.  Outside [T_1, T_m] (where the paper is silent)
    reading R26: the end segments continue (linear extrapolation)."""
    for s in range(len(pts) - 1):
        if T <= pts[s + 1][0]:
            return s
    return len(pts) - 2


def pwl_exact(par, T):
    """k(T) = k_s + (k_{s+1} - k_s) / (T_{s+1} - T_s) (T - T_s) in exact rationals."""
    pts = _pwl_pairs(par)
    T = Fraction(T)
    s = _pwl_segment(pts, T)
    (T0, k0), (T1, k1) = pts[s], pts[s + 1]
    return k0 + (k1 - k0) / (T1 - T0) * (T - T0)


def pwl_slope_exact(par, T):
    """k'(T) of the piecewise-linear k: the slope of the segment that owns T (breakpoints belong to
    the segment on their left, as in the paper's closed first case), exact."""
    pts = _pwl_pairs(par)
    s = _pwl_segment(pts, Fraction(T))
    (T0, k0), (T1, k1) = pts[s], pts[s + 1]
    return (k1 - k0) / (T1 - T0)


def brute_force_assemble(mesh, q_xy, q_w, u, m_coef, c_coef):
    """Dense n x n M, C of the quadrature formula PAPER.md:134-135 in exact arithmetic
    (rational, or mpmath for exp).  Returns numpy float arrays (rounded once)."""
    p = mesh.p
    n = mesh.n_dof
    n_p = mesh.n_p
    qx = [(Fraction(float(a)), Fraction(float(b))) for a, b in q_xy]
    qw = [Fraction(float(w)) for w in q_w]
    tabs = [basis_at(p, x, y) for (x, y) in qx]
    M = [[0] * n for _ in range(n)]
    Cm = [[0] * n for _ in range(n)]
    for e in range(mesh.n_e):
        a, b, c = (tuple(Fraction(float(t)) for t in mesh.vert_xy[v]) for v in mesh.elem_vert[e])
        B = [[b[0] - a[0], c[0] - a[0]], [b[1] - a[1], c[1] - a[1]]]
        det = B[0][0] * B[1][1] - B[0][1] * B[1][0]
        ad = abs(det)
        # inverse of B: grad_x phi = B^{-T} grad_ref phi  (same as J A J^T)
        Binv = [[B[1][1] / det, -B[0][1] / det], [-B[1][0] / det, B[0][0] / det]]
        dofs = [int(d) for d in mesh.elem_dof[e]]
        ue = [Fraction(float(u[d])) for d in dofs]
        for q in range(len(qx)):
            tab = tabs[q]
            uq = sum(tab[i][0] * ue[i] for i in range(n_p))
            mq = k_exact(m_coef[0], m_coef[1], uq)
            cq = k_exact(c_coef[0], c_coef[1], uq)
            gphys = []
            for i in range(n_p):
                gx, gy = tab[i][1], tab[i][2]
                gphys.append((Binv[0][0] * gx + Binv[1][0] * gy, Binv[0][1] * gx + Binv[1][1] * gy))
            for i in range(n_p):
                for j in range(n_p):
                    mij = qw[q] * tab[i][0] * tab[j][0] * ad
                    cij = qw[q] * (gphys[i][0] * gphys[j][0] + gphys[i][1] * gphys[j][1]) * ad
                    M[dofs[i]][dofs[j]] = M[dofs[i]][dofs[j]] + mq * mij
                    Cm[dofs[i]][dofs[j]] = Cm[dofs[i]][dofs[j]] + cq * cij
    tofl = np.vectorize(lambda v: float(v))
    return tofl(np.array(M, dtype=object)).astype(np.float64), tofl(np.array(Cm, dtype=object)).astype(np.float64)


def brute_force_pattern(n_dof: int, elem_dof: np.ndarray):
    """Set-based structural pattern (reading 9): row -> sorted unique columns."""
    rows = [set() for _ in range(n_dof)]
    for dofs in elem_dof:
        for i in dofs:
            rows[int(i)].update(int(j) for j in dofs)
    row_ptr = np.zeros(n_dof + 1, dtype=np.int64)
    cols = []
    for r in range(n_dof):
        s = sorted(rows[r])
        cols += s
        row_ptr[r + 1] = row_ptr[r] + len(s)
    return row_ptr, np.array(cols, dtype=np.int32)
