"""Parity at BASELINE.json's full size, in the configuration bench.py times.

C4 (Gresho-Chan vortex, 256^3 = 16.8 M particles, the bench workload; also C3 Sedov 128^3 and
the clustered C5s 128^3 on the adaptive grid): the GPU runs the whole hydro pass -- density with the h iteration, gradient (+ ghost), force (+ dt) -- over every
particle, with the same cell grid, tiles and kernels as the bench.  The oracle cannot sum 16.8 M
particles in test time, so it recomputes a sample of particles one by one (their 2-hop
neighbourhoods, `Oracle.hydro(sample=...)`) at the GPU's converged h: the sampled outputs must
meet the same bars as the small parity cases (neighbour counts bit-exact; rho, P, c, v_sig
within 1e-4; a and du/dt within 1e-4 of their term scales).  The h iteration itself is checked
by the converged residual of every particle (|g_i| <= h_tol eta^3, the paper's closure,
P:90) and, at sizes the oracle finishes, by test_gpu_parity.test_h_iteration_end_to_end.
"""
import numpy as np
import pytest

import workloads as W
from parity_util import RTOL, assert_close, gpu_hydro, oracle_hydro

pytestmark = pytest.mark.gpu


FULL = {
    # the bench workloads (bench.py WORKLOADS) at their full sizes
    "C4_gresho256": lambda: W.gresho(256),
    "C3_sedov128": lambda: W.sedov(128),  # adaptive grid, wide particles
    "C5s_clustered128": lambda: W.clustered(128 ** 3),  # mostly empty / all-wide blocks skipped
}


@pytest.mark.parametrize("case", list(FULL))
def test_fullsize_sampled(case):
    p = FULL[case]()
    n = p["X"].shape[0]
    g = gpu_hydro(p, dt_ghost=1e-3, h_tol=1e-4)
    assert g["stats"]["unconverged"] == 0
    # every particle's smoothing length solves the closure (Eq. 5 + P:90) to the tolerance
    eta3 = float(np.float32(1.2348)) ** 3  # sph_config_default's eta
    resid = g["nhat"].astype(np.float64) * g["h"].astype(np.float64) ** 3 - eta3
    assert np.abs(resid).max() <= 1.01e-4 * eta3 + 1e-6
    # the oracle at the GPU's h, on a sample: random particles plus the extremes of |a|
    rng = np.random.default_rng(len(case))
    amag = np.linalg.norm(g["a"], axis=1)
    sample = np.unique(np.concatenate([rng.choice(n, 32, replace=False), np.argsort(amag)[-6:]]))
    q = dict(p)
    q["h"] = g["h"].astype(np.float32)
    o = oracle_hydro(q, dt_ghost=1e-3, fixed_h=True, sample=sample)
    d, fin, gr, fo = o["density"], o["finalize"], o["gradient"], o["force"]
    s = sample
    assert np.array_equal(g["count"][s], d["count"][s])
    assert np.array_equal(g["count_force"][s], fo["count"][s].astype(np.int32))
    for k in ("rho", "nhat"):
        assert_close(k, g[k][s], d[k][s], rtol=RTOL)
    for k in ("P", "c"):
        assert_close(k, g[k][s], fin[k][s], rtol=RTOL)
    assert_close("v_sig_grad", g["v_sig_grad"][s], gr["v_sig"][s], rtol=RTOL)
    assert_close("v_sig", g["v_sig"][s], fo["v_sig"][s], rtol=RTOL)
    assert_close("a", g["a"][s], fo["a"][s], atol_scale=fo["scale_a"][s])
    # du: the term scale plus the f32 sensitivities of v_c and of w' near the support edge,
    # as in test_gpu_parity.test_full_pass_fixed_h
    assert_close("du", g["du"][s], fo["du"][s],
                 atol_scale=(fo["scale_u"] + 10.0 * fo["scale_cond"] + 0.01 * fo["scale_tail"])[s])
