"""Quadrature rules on the reference triangle -- INPUT DATA, shared by oracle and CUDA path.

The paper treats the rule as an input of both algorithms ("Quadrature weights {w_q} and
nodes {x_q}", Algorithm 1 input; Algorithm 2 input) and
delegates the values to a published listing.  The configs
(BASELINE.json) name the symmetric Dunavant rules of degree 2/4/6/8 with 3/6/12/16 points,
the minimal rules exact for constant coefficients.

Values: SURVEY.md Appendix A (barycentric orbits, 20 significant digits, area-normalised
weights).  This module holds no arithmetic of the assembly method: it expands orbits into
points and halves the weights so that sum(w) = |T_hat| = 1/2 (reading 4 in DESIGN.md).
The expansion is done in exact rational arithmetic from the decimal strings and rounded
once to float64.  The tables are *self-verifying*: tests/test_rules.py checks the moment
equations sum_q w_q x^a y^b = a! b! / (a+b+2)! for a+b <= degree and non-exactness at
degree+1.
"""
from __future__ import annotations

from decimal import Decimal
from fractions import Fraction

import numpy as np

# orbit kinds: ("c", w) centroid; ("3", a, w) permutations of (a, a, 1-2a);
# ("6", a, b, w) permutations of (a, b, 1-a-b).  Weights are area-normalised (sum 1).
_ORBITS = {
    2: [("3", "0.16666666666666666666666666666666666667", "0.33333333333333333333333333333333333333")],
    4: [
        ("3", "0.44594849091596488632", "0.22338158967801146570"),
        ("3", "0.091576213509770743460", "0.10995174365532186764"),
    ],
    6: [
        ("3", "0.24928674517091042129", "0.11678627572637936603"),
        ("3", "0.063089014491502228340", "0.050844906370206816921"),
        ("6", "0.053145049844816947353", "0.31035245103378440542", "0.082851075618373575194"),
    ],
    8: [
        ("c", "0.14431560767778716825"),
        ("3", "0.45929258829272315603", "0.095091634267284624794"),
        ("3", "0.17056930775176020662", "0.10321737053471825028"),
        ("3", "0.050547228317030975458", "0.032458497623198080311"),
        ("6", "0.0083947774099576053372", "0.26311282963463811342", "0.027230314174434994265"),
    ],
}

# degree -> number of points
RULE_POINTS = {2: 3, 4: 6, 6: 12, 8: 16}


def _frac(s: str) -> Fraction:
    return Fraction(Decimal(s))


def _expand(degree: int):
    """Return list of (beta0, beta1, beta2, w_area) as exact Fractions.

    Fixed point order (reading 6 in DESIGN.md): orbits in table order; within a
    3-orbit the odd coordinate moves beta0 -> beta1 -> beta2; within a 6-orbit the six
    permutations of (a, b, c) in lexicographic order of the index permutation.
    The deg-2 orbit value 1/6 and weight 1/3 are stored as exact fractions.
    """
    pts = []
    for orb in _ORBITS[degree]:
        if orb[0] == "c":
            w = _frac(orb[1])
            t = Fraction(1, 3)
            pts.append((t, t, t, w))
        elif orb[0] == "3":
            a = Fraction(1, 6) if degree == 2 else _frac(orb[1])
            w = Fraction(1, 3) if degree == 2 else _frac(orb[2])
            o = 1 - 2 * a
            pts += [(o, a, a, w), (a, o, a, w), (a, a, o, w)]
        else:
            a, b, w = _frac(orb[1]), _frac(orb[2]), _frac(orb[3])
            c = 1 - a - b
            for perm in ((a, b, c), (a, c, b), (b, a, c), (b, c, a), (c, a, b), (c, b, a)):
                pts.append((*perm, w))
    assert len(pts) == RULE_POINTS[degree]
    return pts


def triangle_rule_exact(degree: int):
    """Exact-rational rule from the decimal table: list of ((x, y), w) with sum w = 1/2."""
    return [((b1, b2), w / 2) for (_b0, b1, b2, w) in _expand(degree)]


def triangle_rule(degree: int):
    """Rule as float64 arrays: xy (n_q, 2) reference coordinates (x, y) = (beta1, beta2),
    w (n_q,) weights with sum 1/2 (reference-triangle measure)."""
    ex = triangle_rule_exact(degree)
    xy = np.array([[float(x), float(y)] for (x, y), _ in ex], dtype=np.float64)
    w = np.array([float(wq) for _, wq in ex], dtype=np.float64)
    return xy, w


def rule_degree_for_order(p: int) -> int:
    """Minimal rule exact for the constant-coefficient mass matrix: degree 2p."""
    return 2 * p
