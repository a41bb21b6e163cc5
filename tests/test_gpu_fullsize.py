"""Parity at BASELINE.json's full sizes, in the configuration bench.py times.

C4 (Gresho-Chan vortex, 256^3 = 16.8 M particles, the bench workload), C2 (Sod, 2 x 64^3), C3
(Sedov 128^3) and the clustered C5s 128^3 on the adaptive grid: the GPU runs the whole hydro pass
-- density with the h iteration, gradient (+ ghost), force (+ dt) -- over every particle, with the
same cell grid, tiles and kernels as the bench.

1. At the bench's h_tol = 1e-4 (the paper's tolerance): every particle's smoothing length solves
   the closure |nhat h^3 - eta^3| <= h_tol eta^3 (Eq. 5 + P:90).
2. Parity: the same run at h_tol = 1e-6 against the oracle on a sample of >= 2000 particles
   (random ones plus the extremes of |a|, |du/dt| and |div v|).  The oracle cannot sum 16.8 M
   particles in test time, so it computes the sample one by one with ITS OWN h iteration (tol
   1e-13) over the samples' 2-hop neighbourhoods (`Oracle.hydro(sample=...)`); nothing the GPU
   computed enters the oracle.  Bars: neighbour counts exact except pairs within 1e-6 h of the
   support radius (north star); h, rho, nhat, P, c, v_sig within 1e-4 relative; div, curl, lap u,
   a and du/dt within 1e-4 of the oracle's per-particle term-magnitude scales (+ du's two f32
   sensitivities).
"""
import numpy as np
import pytest

import workloads as W
from parity_util import (RTOL, assert_close, assert_counts_in_band, du_tolerance, dv_tolerance, gpu_hydro,
                         lap_tolerance, oracle_count_band, oracle_sampled)

pytestmark = pytest.mark.gpu


FULL = {
    # the bench workloads (bench.py WORKLOADS) at their full sizes
    "C4_gresho256": lambda: W.gresho(256),
    "C2_sod2x64": lambda: W.sod(64),
    "C3_sedov128": lambda: W.sedov(128),  # adaptive grid, wide particles
    "C5s_clustered128": lambda: W.clustered(128 ** 3),  # mostly empty / all-wide blocks skipped
}
N_RANDOM = 2000
N_EXTREME = 32


@pytest.mark.parametrize("case", list(FULL))
def test_fullsize_sampled(case):
    p = FULL[case]()
    n = p["X"].shape[0]
    eta3 = float(np.float32(1.2348)) ** 3  # sph_config_default's eta
    # 1. the bench's tolerance: every particle closes (only the GPU's own residual is read)
    g4 = gpu_hydro(p, dt_ghost=1e-3, h_tol=1e-4)
    assert g4["stats"]["unconverged"] == 0
    resid = g4["nhat"].astype(np.float64) * g4["h"].astype(np.float64) ** 3 - eta3
    assert np.abs(resid).max() <= 1.01e-4 * eta3 + 1e-6
    del g4
    # 2. parity against the oracle's own root on a sample
    g = gpu_hydro(p, dt_ghost=1e-3, h_tol=1e-6)
    assert g["stats"]["unconverged"] == 0
    rng = np.random.default_rng(len(case))
    ext = [np.argsort(np.linalg.norm(g["a"], axis=1))[-N_EXTREME:], np.argsort(np.abs(g["du"]))[-N_EXTREME:],
           np.argsort(np.abs(g["div"]))[-N_EXTREME:]]
    s = np.unique(np.concatenate([rng.choice(n, N_RANDOM, replace=False)] + ext))
    # (the oracle's cell list: side ~ a typical support radius, not the largest: Sedov's centre and
    # a clustered box's voids have h ~ 10-100x the dense regions', whose particles would then share
    # a handful of huge cells)
    cs = 2.0 * float(np.percentile(p["h"], 75))
    o = oracle_sampled(p, s, dt_ghost=1e-3, cell_side=cs)
    d, fin, gr, fo = o["density"], o["finalize"], o["gradient"], o["force"]
    s0, s1, s2 = o["sets"]
    assert np.array_equal(s0, s)
    # counts: exact except pairs within 1e-6 h of the support radius (north star), from fixed-h
    # oracle runs at the oracle's root scaled by 1 -+ 5e-7 (h outside the closure set: unused)
    hroot = p["h"].astype(np.float64).copy()
    hroot[s2] = d["h"][s2]
    dlo, dhi, flo, fhi = oracle_count_band(p, hroot, dt_ghost=1e-3, sample=s, hop_radius=o["hop_radius"],
                                           cell_side=cs)
    assert_counts_in_band("count", g["count"], dlo, dhi, idx=s)
    assert_counts_in_band("count_force", g["count_force"], flo, fhi, idx=s)
    assert_close("h", g["h"][s], d["h"][s], rtol=1e-5)
    for k in ("rho", "nhat"):
        assert_close(k, g[k][s], d[k][s], rtol=RTOL)
    for k in ("P", "c"):
        assert_close(k, g[k][s], fin[k][s], rtol=RTOL)
    assert_close("div", g["div"][s], d["div"][s], atol_scale=dv_tolerance(d)[s])
    assert_close("curl", g["curl"][s], d["curl"][s], atol_scale=dv_tolerance(d)[s])
    assert_close("v_sig_grad", g["v_sig_grad"][s], gr["v_sig"][s], rtol=RTOL)
    assert_close("lap_u", g["lap_u"][s], gr["lap_u"][s], atol_scale=lap_tolerance(gr)[s])
    assert_close("v_sig", g["v_sig"][s], fo["v_sig"][s], rtol=RTOL)
    assert_close("a", g["a"][s], fo["a"][s], atol_scale=fo["scale_a"][s])
    sc_u, at_u = du_tolerance(fo)
    assert_close("du", g["du"][s], fo["du"][s], atol_scale=sc_u[s], atol=at_u[s])
