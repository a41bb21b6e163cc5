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


def oracle_hydro(p, dt_ghost=1e-3, fixed_h=False, h_tol=1e-13, mode="cells", sample=None, **prm):
    o = oracle.Oracle(oracle.Params(h_tol=h_tol, h_max_iter=64, **prm), mode=mode)
    st = oracle.State.from_particles(p)
    return o.hydro(st, dt_ghost=dt_ghost, first_step=True, fixed_h=fixed_h, sample=sample)


def oracle_counts_at(p, h, dt_ghost=1e-3, **prm):
    """The oracle's density and force neighbour counts at the given (GPU-converged) h.

    The GPU's h iteration stops at its h_tol (1e-6 of eta^3 in the tests), ~h_tol/3 relative
    from the oracle's exact root; a pair inside that band of the support edge may flip (the
    north star excludes pairs within 1e-6 h of it).  At equal h the counts are bit-exact with
    no exclusion: the GPU re-decides edge pairs in fp64 with the oracle's operation sequence."""
    q = dict(p)
    q["h"] = np.asarray(h, dtype=np.float32)
    o = oracle_hydro(q, dt_ghost=dt_ghost, fixed_h=True, **prm)
    return o["density"]["count"], o["force"]["count"].astype(np.int32)


def assert_close(name, got, ref, rtol=RTOL, atol_scale=None, mask=None):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if mask is not None:
        got, ref = got[mask], ref[mask]
        if atol_scale is not None and np.ndim(atol_scale):
            atol_scale = np.asarray(atol_scale)[mask]
    tol = rtol * np.abs(ref)
    if atol_scale is not None:
        a = np.asarray(atol_scale, dtype=np.float64)
        if got.ndim == 2 and a.ndim == 1:
            a = a[:, None]
        tol = np.maximum(tol, rtol * a)
    err = np.abs(got - ref)
    bad = err > tol
    if bad.any():
        k = np.argmax(err - tol)
        kk = np.unravel_index(k, err.shape)
        raise AssertionError(f"{name}: {bad.sum()} / {bad.size} elements outside tolerance; worst at {kk}: "
                             f"got {got[kk]!r} ref {ref[kk]!r} tol {tol[kk]!r}")
