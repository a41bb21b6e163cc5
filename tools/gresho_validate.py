#!/usr/bin/env python
"""Gresho-Chan vortex run to t = 0.1 through the C-ABI (PAPER.md
P:335-363, Fig. 6): KDK steps at the CFL dt, then v_theta and P binned in the vortex radius
and compared with the analytic Eqs. 27-28; total momentum and energy tracked over the run.

  python tools/gresho_validate.py [--n 64] [--t-end 0.1] [--out file.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402


def totals(ctx, m):
    v = ctx.get("v").astype(np.float64)
    u = ctx.get("u").astype(np.float64)
    P = (m[:, None] * v).sum(0)
    E = float((m * (0.5 * (v * v).sum(1) + u)).sum())
    return P, E, float((m * np.abs(v).sum(1)).sum())


def run(n=64, t_end=0.1, bins=25, jitter=0.0):
    from paper_2505_14538_b200 import Context

    p = W.gresho(n, jitter=jitter)
    m = p["m"].astype(np.float64)
    ctx = Context(p, h_tol=1e-4)
    ctx.density()
    ctx.gradient(1e-4)
    dt = ctx.force()
    P0, E0, pscale = totals(ctx, m)
    t, steps = 0.0, 0
    t0 = time.perf_counter()
    while t < t_end - 1e-12:
        dt = min(dt, t_end - t)
        ctx.kick_drift(0.5 * dt, dt)
        ctx.density()
        ctx.gradient(dt)
        dt_next = ctx.force()
        ctx.kick_drift(0.5 * dt, 0.0)
        t += dt
        steps += 1
        dt = min(dt_next, 2.0 * dt)
    wall = time.perf_counter() - t0
    P1, E1, _ = totals(ctx, m)
    X = ctx.get("X").astype(np.float64) / 2.0 ** 32
    v = ctx.get("v").astype(np.float64)
    Pr = ctx.get("P").astype(np.float64)
    ctx.close()
    dxy = X[:, :2] - 0.5
    r = np.sqrt((dxy ** 2).sum(1))
    vt = (-dxy[:, 1] * v[:, 0] + dxy[:, 0] * v[:, 1]) / np.maximum(r, 1e-12)
    edges = np.linspace(0.0, 0.5, bins + 1)
    idx = np.clip(np.digitize(r, edges) - 1, 0, bins - 1)
    rc = 0.5 * (edges[1:] + edges[:-1])
    sel = r < 0.5
    cnt = np.bincount(idx[sel], minlength=bins)
    vt_mean = np.bincount(idx[sel], weights=vt[sel], minlength=bins) / np.maximum(cnt, 1)
    P_mean = np.bincount(idx[sel], weights=Pr[sel], minlength=bins) / np.maximum(cnt, 1)
    vt_std = np.sqrt(np.bincount(idx[sel], weights=vt[sel] ** 2, minlength=bins) / np.maximum(cnt, 1) - vt_mean ** 2)
    vt_a, P_a = W.gresho_analytic(rc)
    # L1 norm over all particles with r < 0.5 (the standard Gresho error measure)
    vta_p, Pa_p = W.gresho_analytic(r[sel])
    l1_v = float(np.mean(np.abs(vt[sel] - vta_p)))
    l1_P = float(np.mean(np.abs(Pr[sel] - Pa_p)))
    return {
        "n": n, "particles": int(n ** 3), "t_end": t, "steps": steps, "wall_s": wall,
        "L1_vtheta": l1_v, "L1_P": l1_P,
        "momentum_drift_rel": float(np.abs(P1 - P0).max() / pscale),
        "energy_drift_rel": float(abs(E1 - E0) / abs(E0)),
        "bins": {"r": rc.tolist(), "vtheta_mean": vt_mean.tolist(), "vtheta_std": vt_std.tolist(),
                 "vtheta_analytic": vt_a.tolist(), "P_mean": P_mean.tolist(), "P_analytic": P_a.tolist(),
                 "count": cnt.tolist()},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--t-end", type=float, default=0.1)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    res = run(a.n, a.t_end)
    s = json.dumps(res, indent=1)
    if a.out:
        open(a.out, "w").write(s)
    print(json.dumps({k: v for k, v in res.items() if k != "bins"}))
    b = res["bins"]
    for i in range(len(b["r"])):
        print(f"r={b['r'][i]:.3f} vt={b['vtheta_mean'][i]:.4f}+-{b['vtheta_std'][i]:.4f} (an {b['vtheta_analytic'][i]:.4f})"
              f"  P={b['P_mean'][i]:.4f} (an {b['P_analytic'][i]:.4f})")


if __name__ == "__main__":
    main()
