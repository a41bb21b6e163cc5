"""Helpers shared by the GPU parity tests: run the CUDA path and the oracle on the same
seeded inputs and compare element by element."""
from __future__ import annotations

import numpy as np

import oracle

# north-star tolerances (BASELINE.json): rho, h, P, accelerations 1e-4 relative (fp32 vs fp64)
RTOL = 1e-4


def gpu_hydro(p, dt_ghost=1e-3, fixed_h=False, h_tol=1e-6, **cfg):
    """density (+h iteration) -> gradient -> force on the GPU, fields in input order."""
    from paper_2505_14538_b200 import Context

    if fixed_h:
        cfg["h_max_iter"] = 0
    ctx = Context(p, h_tol=h_tol, **cfg)
    st = ctx.density()
    ctx.gradient(dt_ghost)
    dt = ctx.force()
    out = {k: ctx.get(k) for k in ("h", "rho", "drho_dh", "nhat", "dn_dh", "div", "curl", "count", "f", "P", "c",
                                   "B", "v_sig_grad", "lap_u", "alpha_v", "alpha_c", "a", "du", "v_sig",
                                   "count_force", "iters")}
    out["stats"] = st
    out["dt"] = dt
    out["counters"] = ctx.counters()
    ctx.close()
    return out


def oracle_hydro(p, dt_ghost=1e-3, fixed_h=False, h_tol=1e-13, mode="cells", sample=None, hop_radius=None,
                 allow_unconverged=False, cell_side=None, **prm):
    """The oracle's hydro pass; its status codes are asserted (a sampled run whose 2-hop
    closure missed a neighbour reports ORC_ERR_MISSING, an h iteration that did not close
    ORC_ERR_NOT_CONVERGED)."""
    o = oracle.Oracle(oracle.Params(h_tol=h_tol, h_max_iter=64, **prm), mode=mode, cell_side=cell_side)
    st = oracle.State.from_particles(p)
    r = o.hydro(st, dt_ghost=dt_ghost, first_step=True, fixed_h=fixed_h, sample=sample, hop_radius=hop_radius)
    assert r["density"]["status"] == 0 or (allow_unconverged and r["density"]["status"] == ORC_NOT_CONVERGED), \
        f"oracle density status {r['density']['status']}"
    assert r["gradient"]["status"] == 0, f"oracle gradient status {r['gradient']['status']}"
    assert r["force"]["status"] == 0, f"oracle force status {r['force']['status']}"
    return r


ORC_NOT_CONVERGED, ORC_MISSING = 5, 9  # oracle.c status codes


def oracle_sampled(p, sample, dt_ghost=1e-3, **kw):
    """The oracle's own h iteration and hydro pass on a sample (2-hop closure): the hop radius
    starts at 1.5 gamma_k max(h0) and grows until it exceeds 1.25 gamma_k times the largest
    converged h of the closure set, so the sampled particles' supports (and their neighbours')
    are covered; a neighbour outside the closure would still fail the status check."""
    R = 1.5 * 2.0 * float(np.max(p["h"]))
    for _ in range(4):
        o = oracle_hydro(p, dt_ghost=dt_ghost, sample=sample, hop_radius=R, **kw)
        s2 = o["sets"][2]
        if 1.25 * 2.0 * float(np.max(o["density"]["h"][s2])) <= R:
            o["hop_radius"] = R
            return o
        R *= 1.5
    raise AssertionError("sampled oracle: hop radius did not cover the converged supports")


# North star: neighbour counts bit-exact "excluding pairs within 1e-6 h of the support radius".
# A GPU h iteration stopped at h_tol = 1e-6 is within h_tol/(3 Omega) ~ 4e-7 relative of the
# exact root, i.e. its support radius 2h within ~8e-7 h of the oracle's: inside that band.
COUNT_BAND_H = 5e-7  # relative change of h that moves the support radius 2h by 1e-6 h


def oracle_count_band(p, h, dt_ghost=1e-3, sample=None, hop_radius=None, band=COUNT_BAND_H, **prm):
    """Bounds of the oracle's density and force neighbour counts over supports within the
    north star's exclusion band: (lo, hi) for N_i (r < H_i) and for N_force (r < max(H_i, H_j))
    at every h scaled by (1 - band) and (1 + band).  h is the ORACLE's converged h."""
    out = []
    for f in (1.0 - band, 1.0 + band):
        q = dict(p)
        q["h"] = (np.asarray(h, dtype=np.float64) * f).astype(np.float32)
        o = oracle_hydro(q, dt_ghost=dt_ghost, fixed_h=True, sample=sample, hop_radius=hop_radius, **prm)
        fc = o["force"]["count"]
        out.append((o["density"]["count"], np.where(np.isnan(fc), -1, fc).astype(np.int64)))  # (-1: not sampled)
    (dlo, flo), (dhi, fhi) = out
    return dlo, dhi, flo, fhi


def assert_counts_in_band(name, got, lo, hi, idx=None):
    got = np.asarray(got, dtype=np.int64)
    if idx is not None:
        got, lo, hi = got[idx], lo[idx], hi[idx]
    bad = (got < lo) | (got > hi)
    if bad.any():
        k = int(np.flatnonzero(bad)[0])
        raise AssertionError(f"{name}: {bad.sum()} particles outside the band counts; first at {k}: got {got[k]} "
                             f"band [{lo[k]}, {hi[k]}]")


def dv_tolerance(d):
    """atol_scale for div v and curl v: 1e-4 of the sum of term magnitudes plus the edge
    sensitivity (a pair near the support edge, w' ~ (2-q)^2, under a 1e-6 relative rounding of q)."""
    return d["scale_dv"] + 0.01 * d["scale_dv_tail"]


def lap_tolerance(gr):
    """atol_scale for lap u (the same two parts as dv_tolerance)."""
    return gr["scale_lap"] + 0.01 * gr["scale_lap_tail"]


def du_tolerance(fo):
    """(atol_scale, atol) for du/dt: 1e-4 of the term scale plus two f32
    sensitivities of the terms -- w'(q) near the support edge (1e-6 scale_tail) and the rounding
    of v_ij . r_ij (1e-6 scale_v: rigid rotation makes it rounding-level) -- plus the absolute
    bound scale_cond of the conduction term's v_c = sqrt(2|P_i - P_j|/rho) under a 1e-6 relative
    pressure error (oracle.c)."""
    return fo["scale_u"] + 0.01 * (fo["scale_tail"] + fo["scale_v"]), fo["scale_cond"]


def assert_close(name, got, ref, rtol=RTOL, atol_scale=None, mask=None, atol=None):
    """|got - ref| <= max(rtol |ref|, rtol atol_scale + atol) element by element (atol_scale and
    atol per particle; 2-D fields take the particle's scale for every component)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if mask is not None:
        got, ref = got[mask], ref[mask]
        if atol_scale is not None and np.ndim(atol_scale):
            atol_scale = np.asarray(atol_scale)[mask]
        if atol is not None and np.ndim(atol):
            atol = np.asarray(atol)[mask]
    tol = rtol * np.abs(ref)
    if atol_scale is not None or atol is not None:
        a = rtol * np.asarray(atol_scale if atol_scale is not None else 0.0, dtype=np.float64)
        a = a + np.asarray(atol if atol is not None else 0.0, dtype=np.float64)
        if got.ndim == 2 and a.ndim == 1:
            a = a[:, None]
        tol = np.maximum(tol, a)
    err = np.abs(got - ref)
    bad = err > tol
    if bad.any():
        k = np.argmax(err - tol)
        kk = np.unravel_index(k, err.shape)
        raise AssertionError(f"{name}: {bad.sum()} / {bad.size} elements outside tolerance; worst at {kk}: "
                             f"got {got[kk]!r} ref {ref[kk]!r} tol {tol[kk]!r}")
