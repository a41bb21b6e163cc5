"""Gresho-Chan vortex to t = 0.1 (Fig. 6, Eqs. 27-28):
the KDK integrator with all three loops and both switches, judged against the analytic
solution.  At 64^3 the L1 error of v_theta is 0.027 and of P 0.032 (128^3: 0.040 / 0.038,
profiles/r01/gresho128.json); the bounds below catch a broken loop (a wrong sign or factor
in the force loop puts L1(v_theta) above 0.2 within a few steps) while leaving room for the
scheme's own smoothing of the v_theta kink at r = 0.2.  Total momentum and energy are
conserved by the pairwise-antisymmetric force loop and the KDK integrator."""
import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))

pytestmark = pytest.mark.gpu


def test_gresho_vortex_t01():
    from gresho_validate import run

    res = run(n=64, t_end=0.1)
    assert res["L1_vtheta"] < 0.08, res["L1_vtheta"]
    assert res["L1_P"] < 0.08, res["L1_P"]
    assert res["momentum_drift_rel"] < 1e-6
    assert res["energy_drift_rel"] < 1e-3
    b = res["bins"]
    # the vortex survives: the peak stays near v_theta(0.2) = 1 (SPH smooths the kink)
    assert 0.8 < max(b["vtheta_mean"]) < 1.05
