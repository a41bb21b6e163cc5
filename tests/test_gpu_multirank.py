"""Multi-rank slab decomposition on one GPU
through the loopback transport: R contexts, one thread each, exchanging migrants, ghost
planes (X1-X3) and the global scalars (X4) exactly as the NCCL transport does between
processes.  Bars:
  - every particle owned by exactly one rank after any number of steps;
  - one hydro pass: the same per-particle results as the fp64 oracle on the whole box, to the
    single-GPU parity bars (neighbour counts bit-exact);
  - one hydro pass vs the single-context GPU run: counts exact, floats to f32 summation-order
    rounding (the ghost copies make each rank's tiles hold the same neighbours);
  - KDK steps with particles crossing slab boundaries: trajectories track the single-context
    run to f32 rounding growth.
"""
import numpy as np
import pytest

import workloads as W
from multirank_util import run_ranks
from parity_util import (RTOL, assert_close, assert_counts_in_band, du_tolerance, dv_tolerance, gpu_hydro,
                         lap_tolerance, oracle_count_band, oracle_hydro, oracle_sampled)

pytestmark = pytest.mark.gpu


def _switches(p, seed):
    rng = np.random.default_rng(seed)
    n = p["X"].shape[0]
    p = dict(p)
    p["alpha_v"] = rng.uniform(0.0, 2.0, n).astype(np.float32)
    p["alpha_c"] = rng.uniform(0.0, 0.5, n).astype(np.float32)
    return p


def _hydro(dt_ghost):
    def prog(ctx):
        st = ctx.density()
        ctx.gradient(dt_ghost)
        dt = ctx.force()
        return {"stats": st, "dt": dt, "counters": ctx.counters()}

    return prog


@pytest.mark.parametrize("R", [2, 3, 4])
def test_multirank_hydro_matches_oracle(R):
    p = _switches(W.jittered_lattice(20, seed=61, vel_sigma=0.05, u_sigma=0.3), 3)
    p["h"] = (p["h"] * 1.1).astype(np.float32)
    g, parts = run_ranks(p, R, _hydro(2e-4), h_tol=1e-6)
    o = oracle_hydro(p, dt_ghost=2e-4)
    d, fin, gr, fo = o["density"], o["finalize"], o["gradient"], o["force"]
    # counts: exact except pairs within 1e-6 h of the support radius (north star)
    dlo, dhi, flo, fhi = oracle_count_band(p, d["h"], dt_ghost=2e-4)
    assert_counts_in_band("count", g["count"], dlo, dhi)
    assert_counts_in_band("count_force", g["count_force"], flo, fhi)
    assert_close("h", g["h"], d["h"], rtol=1e-5)
    assert_close("rho", g["rho"], d["rho"], rtol=2e-5)
    assert_close("P", g["P"], fin["P"], rtol=2e-5)
    assert_close("v_sig_grad", g["v_sig_grad"], gr["v_sig"], rtol=1e-4)
    assert_close("a", g["a"], fo["a"], atol_scale=fo["scale_a"])
    sc_u, at_u = du_tolerance(fo)
    assert_close("du", g["du"], fo["du"], atol_scale=sc_u, atol=at_u)
    assert_close("v_sig", g["v_sig"], fo["v_sig"])
    # every rank sees the global CFL minimum (X4)
    dts = {q["dt"] for q in parts}
    assert len(dts) == 1 and abs(parts[0]["dt"] - o["dt"]) <= RTOL * o["dt"]
    assert sum(q["counters"]["pairs_force"] for q in parts) == int(g["count_force"].sum())


@pytest.mark.parametrize("case,R", [("poisson", 2), ("jitter", 3), ("jitter", 5)])
def test_multirank_matches_single_gpu(case, R):
    if case == "poisson":
        p = _switches(W.poisson(30000, seed=62, vel_sigma=0.2, u_sigma=0.4), 4)
    else:
        p = _switches(W.jittered_lattice(40, seed=64, vel_sigma=0.2, u_sigma=0.4), 4)
    # the same h on both sides (no iteration): neighbour sets identical by construction
    one = gpu_hydro(p, dt_ghost=1e-3, fixed_h=True)
    g, parts = run_ranks(p, R, _hydro(1e-3), h_max_iter=0)
    assert np.array_equal(g["count"], one["count"])
    assert np.array_equal(g["count_force"], one["count_force"])
    for k in ("h", "rho", "P", "c", "f", "v_sig_grad", "v_sig", "alpha_v"):
        assert_close(k, g[k], one[k], rtol=2e-5, atol_scale=np.abs(one[k]).max() * 1e-3 if k == "alpha_v" else None)
    assert {q["dt"] for q in parts} == {parts[0]["dt"]}
    # accelerations are sums with cancellation: judge both runs against the oracle on a
    # sample holding the particles where they differ most (+ random ones)
    diff = np.abs(g["a"] - one["a"]).max(1)
    rng = np.random.default_rng(7)
    sample = np.unique(np.concatenate([np.argsort(diff)[-24:], rng.choice(len(diff), 40, replace=False)]))
    o = oracle_hydro(p, dt_ghost=1e-3, fixed_h=True, sample=sample)
    fo = o["force"]
    for run in (g, one):
        assert_close("a", run["a"][sample], fo["a"][sample], atol_scale=fo["scale_a"][sample])


@pytest.mark.parametrize("R", [1, 2, 3])
def test_halo_put_matches_send_recv(R):
    """X3 by peer stores from the gradient epilogue (halo_put = 1, NEXT#4) against X3 by
    send/recv of the ghost planes after the loop (halo_put = 0): the force loop sees the same
    ghost records, so counts agree exactly and a, du/dt to the summation order."""
    p = _switches(W.jittered_lattice(30, seed=66, vel_sigma=0.2, u_sigma=0.4), 5)
    res = {}
    for put in (0, 1):
        res[put], _ = run_ranks(p, R, _hydro(1e-3), h_max_iter=0, halo_put=put)
    a, b = res[0], res[1]
    assert np.array_equal(a["count"], b["count"])
    assert np.array_equal(a["count_force"], b["count_force"])
    for k in ("rho", "P", "v_sig_grad", "v_sig", "alpha_v"):
        assert np.array_equal(a[k], b[k]), k
    for k in ("a", "du"):
        scale = np.abs(a[k]).max()
        assert np.abs(a[k] - b[k]).max() <= 1e-5 * scale, k


@pytest.mark.parametrize("G", [2, 3])
def test_multirank_more_ghost_planes(G, monkeypatch):
    """The [G ghost | owned | G ghost] plane layout (the one wide particles need)
    holds the same neighbours as G = 1: results identical to the single-context run."""
    monkeypatch.setenv("SPH_GHOST_PLANES", str(G))
    p = _switches(W.jittered_lattice(40, seed=64, vel_sigma=0.2, u_sigma=0.4), 4)
    one = gpu_hydro(p, dt_ghost=1e-3, fixed_h=True)
    g, parts = run_ranks(p, 3, _hydro(1e-3), h_max_iter=0)
    assert np.array_equal(g["count"], one["count"])
    assert np.array_equal(g["count_force"], one["count_force"])
    for k in ("rho", "P", "v_sig_grad", "v_sig"):
        assert_close(k, g[k], one[k], rtol=2e-5)
    assert sum(q["counters"]["pairs_force"] for q in parts) == int(one["count_force"].sum())
    # accelerations (sums with cancellation): both runs against the oracle where they differ most
    diff = np.abs(g["a"] - one["a"]).max(1)
    sample = np.unique(np.argsort(diff)[-48:])
    fo = oracle_hydro(p, dt_ghost=1e-3, fixed_h=True, sample=sample)["force"]
    for run in (g, one):
        assert_close("a", run["a"][sample], fo["a"][sample], atol_scale=fo["scale_a"][sample])


@pytest.mark.parametrize("R", [2, 3, 4])
def test_multirank_adaptive_sedov(R):
    """C3-like Sedov blast on the slab path: the adaptive grid with wide particles on every rank
    (DESIGN.md §9, §11).  The blast centre's wide particles reach several cell planes into the
    neighbouring slabs (G ghost planes per side).
      (a) fixed h: the same neighbour sets as the single-context run (counts exact, floats to
          f32 summation order);
      (b) the h iteration: a sample (random, the largest h, the particles nearest the slab faces)
          against the oracle's own root, at the single-GPU parity bars."""
    p = _switches(W.sedov(64), 8)
    n = p["X"].shape[0]
    one = gpu_hydro(p, dt_ghost=1e-3, fixed_h=True)
    g, parts = run_ranks(p, R, _hydro(1e-3), h_max_iter=0)
    wide = [q["counters"]["wide_particles"] for q in parts]
    assert min(wide) > 0 and one["counters"]["wide_particles"] > 0
    assert np.array_equal(g["count"], one["count"])
    assert np.array_equal(g["count_force"], one["count_force"])
    for k in ("rho", "P", "c", "f", "v_sig_grad", "v_sig"):
        assert_close(k, g[k], one[k], rtol=2e-5)
    assert sum(q["counters"]["pairs_force"] for q in parts) == int(one["count_force"].sum())
    assert {q["dt"] for q in parts} == {parts[0]["dt"]}
    # (b)
    g, parts = run_ranks(p, R, _hydro(1e-3), h_tol=1e-6)
    assert all(q["stats"]["unconverged"] == 0 for q in parts)
    x = p["X"][:, 0].astype(np.float64) / 2.0 ** 32
    face = np.min(np.abs(((x[:, None] - np.arange(R)[None, :] / R) + 0.5) % 1.0 - 0.5), axis=1)
    rng = np.random.default_rng(R)
    s = np.unique(np.concatenate([rng.choice(n, 400, replace=False), np.argsort(g["h"])[-48:],
                                  np.argsort(face)[:96]]))
    cs = 2.0 * float(np.percentile(p["h"], 75))
    o = oracle_sampled(p, s, dt_ghost=1e-3, cell_side=cs)
    d, fin, gr, fo = o["density"], o["finalize"], o["gradient"], o["force"]
    s2 = o["sets"][2]
    hroot = p["h"].astype(np.float64).copy()
    hroot[s2] = d["h"][s2]
    dlo, dhi, flo, fhi = oracle_count_band(p, hroot, dt_ghost=1e-3, sample=s, hop_radius=o["hop_radius"],
                                           cell_side=cs)
    assert_counts_in_band("count", g["count"], dlo, dhi, idx=s)
    assert_counts_in_band("count_force", g["count_force"], flo, fhi, idx=s)
    assert_close("h", g["h"][s], d["h"][s], rtol=1e-5)
    assert_close("rho", g["rho"][s], d["rho"][s], rtol=RTOL)
    assert_close("P", g["P"][s], fin["P"][s], rtol=RTOL)
    assert_close("div", g["div"][s], d["div"][s], atol_scale=dv_tolerance(d)[s])
    assert_close("v_sig_grad", g["v_sig_grad"][s], gr["v_sig"][s], rtol=RTOL)
    assert_close("lap_u", g["lap_u"][s], gr["lap_u"][s], atol_scale=lap_tolerance(gr)[s])
    assert_close("v_sig", g["v_sig"][s], fo["v_sig"][s], rtol=RTOL)
    assert_close("a", g["a"][s], fo["a"][s], atol_scale=fo["scale_a"][s])
    sc_u, at_u = du_tolerance(fo)
    assert_close("du", g["du"][s], fo["du"][s], atol_scale=sc_u[s], atol=at_u[s])


def _kdk(steps, log):
    def prog(ctx):
        ctx.density()
        ctx.gradient(1e-3)
        dt = ctx.force()
        n0 = ctx.n
        id0 = ctx.get("id")
        for _ in range(steps):
            ctx.kick_drift(0.5 * dt, dt)
            ctx.density()
            ctx.gradient(dt)
            dt_new = ctx.force()
            ctx.kick_drift(0.5 * dt, 0.0)
            dt = dt_new
            log.append(ctx.n)
        return {"n0": n0, "id0": id0, "dt": dt, "counters": ctx.counters()}

    return prog


def test_multirank_kdk_migration():
    """Bulk flow along x pushes particles across the slab boundaries every step."""
    from paper_2505_14538_b200 import Context

    p = _switches(W.jittered_lattice(24, seed=63, vel_sigma=0.05, u_sigma=0.2), 5)
    p["v"] = p["v"].copy()
    p["v"][:, 0] += 3.0  # ~3 sound speeds: ~0.5 h per step at the CFL dt
    steps = 6
    log = []
    g, parts = run_ranks(p, 3, _kdk(steps, log), h_tol=1e-5)
    moved = sum(len(set(q["id0"].tolist()) ^ set(q["id"].tolist())) for q in parts)
    assert moved > 0, "no particle migrated"
    ctx = Context(p, h_tol=1e-5)
    ref = _kdk(steps, [])(ctx)
    X1, rho1, v1 = ctx.get("X"), ctx.get("rho"), ctx.get("v")
    ctx.close()
    dX = (g["X"].astype(np.int64) - X1.astype(np.int64) + 2 ** 31) % 2 ** 32 - 2 ** 31
    assert np.abs(dX).max() < 2 ** 32 * 1e-6, "positions drifted apart"
    assert_close("rho", g["rho"], rho1, rtol=1e-4)
    assert_close("v", g["v"], v1, rtol=1e-4, atol_scale=np.full(len(rho1), 0.05))  # vel_sigma
    assert abs(parts[0]["dt"] - ref["dt"]) <= 1e-4 * ref["dt"]


def test_multirank_balanced_slabs():
    """sph_config.balance (the 1-D ORB of the slab path): with two thirds of the
    particles in x < 1/2 the fixed slabs own 44 / 33 / 22 % of them; every rebuild moves the
    cuts toward equal counts (a quarter plane at a time), particles migrate across the moving
    cuts, and the run still tracks the single-context run."""
    from paper_2505_14538_b200 import Context

    p = _switches(W.poisson(24000, seed=67, vel_sigma=0.02, u_sigma=0.2), 6)
    x = p["X"][:, 0].astype(np.float64) / 2.0 ** 32
    xs = np.where(x < 2.0 / 3.0, 0.75 * x, 0.5 + 1.5 * (x - 2.0 / 3.0))  # density 4/3 left, 2/3 right
    p["X"] = p["X"].copy()
    p["X"][:, 0] = np.minimum(np.floor(xs * 2.0 ** 32), 2.0 ** 32 - 1).astype(np.uint32)
    steps = 8
    kdk = _kdk(steps, [])

    def prog(ctx):
        n_start = ctx.n  # (the creation's rebuild keeps the fixed cuts)
        out = kdk(ctx)
        out["n_start"] = n_start
        return out

    g, parts = run_ranks(p, 3, prog, h_tol=1e-5, balance=1)
    n0 = [q["n_start"] for q in parts]
    n1 = [q["n_local"] for q in parts]
    assert sum(n1) == p["X"].shape[0]
    assert max(n0) > 10000 and max(n1) < 8400, (n0, n1)  # 44 / 33 / 22 % -> about a third each
    ctx = Context(p, h_tol=1e-5)
    ref = _kdk(steps, [])(ctx)
    X1, rho1 = ctx.get("X"), ctx.get("rho")
    ctx.close()
    dX = (g["X"].astype(np.int64) - X1.astype(np.int64) + 2 ** 31) % 2 ** 32 - 2 ** 31
    assert np.abs(dX).max() < 2 ** 32 * 1e-6, "positions drifted apart"
    assert_close("rho", g["rho"], rho1, rtol=1e-4)
    assert abs(parts[0]["dt"] - ref["dt"]) <= 1e-4 * ref["dt"]


def test_multirank_too_thin_slab_is_an_error():
    """Two ranks need two planes each (ghost planes distinct): explicit error, no hang."""
    from paper_2505_14538_b200 import SphError

    p = W.lattice(8, h_factor=1.0)  # ~3 cells per axis -> 1 plane per slab at R = 2
    with pytest.raises(SphError):
        run_ranks(p, 2, _hydro(1e-3), timeout=60)


@pytest.mark.parametrize("transport", ["loopback", "nccl"])
def test_single_rank_slab_path(transport):
    """One rank through the slab path: its ghost planes are copies of its own edge planes,
    exchanged with itself -- over NCCL (send/recv to self + allreduce, the only NCCL run a
    single GPU allows) or the loopback group."""
    from paper_2505_14538_b200 import Context, LoopbackGroup, nccl_unique_id

    p = _switches(W.jittered_lattice(24, seed=65, vel_sigma=0.1, u_sigma=0.3), 6)
    n = p["X"].shape[0]
    one = gpu_hydro(p, dt_ghost=1e-3, fixed_h=True)
    grp = LoopbackGroup(1) if transport == "loopback" else None
    kw = {"loopback": grp} if grp else {"nccl_uid": nccl_unique_id()}
    ctx = Context(p, rank=0, nranks=1, n_total=n, h_max_iter=0, **kw)
    ctx.density()
    ctx.gradient(1e-3)
    dt = ctx.force()
    got = {k: ctx.get(k) for k in ("count", "count_force", "rho", "P", "a", "du", "v_sig")}
    # a KDK step with drift: rebuild + self-migration bookkeeping
    ctx.kick_drift(0.5 * dt, dt)
    ctx.density()
    ctx.close()
    if grp:
        grp.close()
    assert np.array_equal(got["count"], one["count"])
    assert np.array_equal(got["count_force"], one["count_force"])
    for k in ("rho", "P", "v_sig"):
        assert_close(k, got[k], one[k], rtol=2e-6)
    # accelerations (sums with cancellation): both runs against the oracle where they differ most
    diff = np.abs(got["a"] - one["a"]).max(1)
    sample = np.unique(np.concatenate([np.argsort(diff)[-16:], np.arange(0, n, n // 16)]))
    fo = oracle_hydro(p, dt_ghost=1e-3, fixed_h=True, sample=sample)["force"]
    for run in (got, one):
        assert_close("a", run["a"][sample], fo["a"][sample], atol_scale=fo["scale_a"][sample])
    assert abs(dt - one["dt"]) <= 1e-6 * one["dt"]


@pytest.mark.parametrize("balance", [0, 1])
def test_multirank_kdk_sedov_wide(balance):
    """KDK steps of the C3-like Sedov blast on three ranks: migration, rebuilds with G ghost
    planes and wide particles on every rank (halo put on the loopback transport; balance = 1
    also moves the slab cuts at every rebuild).  Momentum: cross-rank pairs are evaluated on both
    ranks (each keeps its own side) from tile coordinates, so the two sides agree to f32
    rounding, not bitwise: |Delta P| <= 1e-6 sum m |v| per step (north star);
    the trajectories track the single-context run to f32 rounding growth."""
    from paper_2505_14538_b200 import Context

    p = _switches(W.sedov(48), 11)
    m = p["m"].astype(np.float64)
    steps = 3
    g, parts = run_ranks(p, 3, _kdk(steps, []), h_tol=1e-5, balance=balance)
    assert min(q["counters"]["wide_particles"] for q in parts) > 0
    ctx = Context(p, h_tol=1e-5)
    ref = _kdk(steps, [])(ctx)
    X1, rho1, v1 = ctx.get("X"), ctx.get("rho"), ctx.get("v")
    ctx.close()
    v0 = p["v"].astype(np.float64)
    pscale = float((m * (np.linalg.norm(v0, axis=1) + np.linalg.norm(g["v"].astype(np.float64), axis=1))).sum())
    dP = np.abs((m[:, None] * (g["v"].astype(np.float64) - v0)).sum(0)).max()
    assert dP <= 1e-6 * pscale * steps, (dP, pscale)
    dX = (g["X"].astype(np.int64) - X1.astype(np.int64) + 2 ** 31) % 2 ** 32 - 2 ** 31
    assert np.abs(dX).max() < 2 ** 32 * 1e-6, "positions drifted apart"
    assert_close("rho", g["rho"], rho1, rtol=1e-4)
    assert_close("v", g["v"], v1, rtol=1e-4, atol_scale=np.full(len(rho1), 1e-2))
    assert abs(parts[0]["dt"] - ref["dt"]) <= 1e-4 * ref["dt"]
