"""Pins of the oracle's smoothing kernel -- CPU only."""
import math

import numpy as np
import pytest


def test_normalisation_quadrature(orc):
    """Pin-1: int W 4 pi r^2 dr = 1.  Gauss-Legendre on each polynomial
    piece of the oracle's own W is exact to rounding."""
    xs, ws = np.polynomial.legendre.leggauss(20)
    for h in (0.37, 1.0, 2.5):
        tot = 0.0
        for a, b in ((0.0, h), (h, 2.0 * h)):
            r = 0.5 * (b - a) * xs + 0.5 * (b + a)
            tot += 0.5 * (b - a) * sum(wi * orc.kernel(ri, h)[0] * 4 * math.pi * ri * ri for ri, wi in zip(r, ws))
        assert abs(tot - 1.0) < 1e-12


def test_closed_form_values(orc):
    """Textbook M4 values: w(0)=1, w(1)=1/4, w(2)=0, w'(1)=-3/4 (both pieces agree),
    sigma = 1/pi so W(0,h) = 1/(pi h^3)."""
    assert orc.w(0.0) == 1.0
    assert abs(orc.w(1.0) - 0.25) < 1e-15
    assert orc.w(2.0) == 0.0 and orc.w(2.5) == 0.0
    assert abs(orc.dw(1.0) + 0.75) < 1e-15
    assert abs(orc.dw(1.0 - 1e-12) + 0.75) < 1e-9
    W, dr, dh = orc.kernel(0.0, 0.5)
    assert abs(W - 1.0 / (math.pi * 0.125)) < 1e-12
    assert dr == 0.0  # S:46 radial symmetry at the origin
    # continuity of w and w' at q = 1 and q = 2
    for q in (1.0, 2.0):
        assert abs(orc.w(q - 1e-9) - orc.w(q + 1e-9)) < 1e-8
        assert abs(orc.dw(q - 1e-9) - orc.dw(q + 1e-9)) < 1e-8


def test_compact_support(orc):
    """Pin-2: W, dW/dr, dW/dh are exactly 0 for r >= 2h."""
    for h in (0.1, 1.0, 3.0):
        for r in (2.0 * h, 2.0000001 * h, 3.0 * h):
            assert orc.kernel(r, h) == (0.0, 0.0, 0.0) or all(abs(x) == 0.0 for x in orc.kernel(r, h))


@pytest.mark.parametrize("seed", [0, 1])
def test_derivatives_finite_difference(orc, seed):
    """Pin-3: dW/dr and dW/dh (Eq. 6 summand) equal central differences of W at random
    (r, h), 1e-6 relative -- except q = 1 where dW/dh is exactly 0 (SPEC S:54 is degenerate
    there), checked with an absolute tolerance."""
    rng = np.random.default_rng(seed)
    for _ in range(20):
        h = rng.uniform(0.2, 2.0)
        r = rng.uniform(0.02, 1.95) * h
        if abs(r / h - 1.0) < 1e-3:
            continue
        W, dr, dh = orc.kernel(r, h)
        e = 1e-6 * h
        fd_r = (orc.kernel(r + e, h)[0] - orc.kernel(r - e, h)[0]) / (2 * e)
        fd_h = (orc.kernel(r, h + e)[0] - orc.kernel(r, h - e)[0]) / (2 * e)
        scale = 1.0 / h ** 4
        assert abs(dr - fd_r) < 1e-6 * scale
        assert abs(dh - fd_h) < 1e-6 * scale
    # q = 1: dW/dh = -(3W + r dW/dr)/h = -(3/4 - 3/4)/(pi h^4) = 0
    _, _, dh1 = orc.kernel(0.7, 0.7)
    assert abs(dh1) < 1e-14


def test_homogeneity(orc):
    """Pin-4: dW/dh(lambda r, lambda h) = lambda^-4 dW/dh(r, h)."""
    rng = np.random.default_rng(3)
    for _ in range(20):
        h = rng.uniform(0.2, 2.0)
        r = rng.uniform(0.0, 2.0) * h
        lam = rng.uniform(0.1, 10.0)
        a = orc.kernel(lam * r, lam * h)[2]
        b = orc.kernel(r, h)[2] / lam ** 4
        assert abs(a - b) <= 1e-12 * max(abs(b), 1e-300) + 1e-300
