"""Pins of the quadrature-rule INPUT data ("Gaussian quadrature"; reading 4-6).

Moment equations: sum_q w_q x^a y^b = a! b! / (a+b+2)! for a+b <= degree,
evaluated in exact rationals on the float64 table values; the rule must NOT be exact at
degree+1 (so a wrong-degree rule or a dropped orbit fails); sum w = 1/2.
"""
from fractions import Fraction
from math import factorial

import numpy as np
import pytest

from fea_inputs.rules import RULE_POINTS, triangle_rule


def _moment_residuals(deg_max, xy, w):
    res = {}
    for d in range(deg_max + 1):
        for a in range(d + 1):
            b = d - a
            s = sum(Fraction(float(wq)) * Fraction(float(x)) ** a * Fraction(float(y)) ** b
                    for (x, y), wq in zip(xy, w))
            exact = Fraction(factorial(a) * factorial(b), factorial(a + b + 2))
            res[(a, b)] = abs(float(s - exact))
    return res


@pytest.mark.parametrize("degree", [2, 4, 6, 8])
def test_rule_moments_exact(degree):
    xy, w = triangle_rule(degree)
    assert xy.shape == (RULE_POINTS[degree], 2) and w.shape == (RULE_POINTS[degree],)
    res = _moment_residuals(degree, xy, w)
    assert max(res.values()) <= 1e-15, max(res.items(), key=lambda kv: kv[1])


@pytest.mark.parametrize("degree", [2, 4, 6, 8])
def test_rule_not_exact_one_degree_higher(degree):
    xy, w = triangle_rule(degree)
    res = _moment_residuals(degree + 1, xy, w)
    top = [res[(a, degree + 1 - a)] for a in range(degree + 2)]
    assert max(top) > 1e-9  # >> the 1e-15 exactness residual


@pytest.mark.parametrize("degree", [2, 4, 6, 8])
def test_rule_weights_points(degree):
    xy, w = triangle_rule(degree)
    assert abs(w.sum() - 0.5) <= 1e-15
    assert (w > 0).all()
    assert (xy > 0).all() and (xy.sum(1) < 1).all()
    # symmetric rule: invariant under the barycentric permutation (x, y) -> (y, x)
    pts = {(round(x, 14), round(y, 14)) for x, y in xy}
    assert {(b, a) for a, b in pts} == pts


def test_deg2_is_interior_rule():
    """Reading 5: the 3-point degree-2 rule is Dunavant's interior rule (2/3, 1/6, 1/6), w = 1/6."""
    xy, w = triangle_rule(2)
    assert np.allclose(np.sort(xy[:, 0]), [1 / 6, 1 / 6, 2 / 3], atol=1e-16)
    assert np.allclose(w, 1 / 6, atol=1e-17)
