"""One whole KDK step (the bench's step: kick, drift, rebuild, density + h iteration, gradient,
force, kick) on the GPU against the fp64 oracle's same step from the same seeded state, with the
same dt (S:251-258 kick / drift).  North star: "total momentum and energy drift
within 1e-6 relative per step":
  - |Delta P_gpu - Delta P_oracle| and |Delta P_gpu| <= 1e-6 sum m |v| (pair forces are
    antisymmetric, so momentum is conserved up to rounding on both sides);
  - |Delta E_gpu - Delta E_oracle| <= 1e-6 E, E = sum m (v^2/2 + u);
  - per particle after the step: v and u within 1e-4 of the step's own change scale, X within a
    few units of the 2^-32 L grid.
The oracle's inputs are the generator's arrays and the oracle's own CFL dt; nothing the GPU
computed enters it."""
import numpy as np
import pytest

import oracle
import workloads as W
from parity_util import du_tolerance, oracle_hydro

pytestmark = pytest.mark.gpu


def _switches(p, seed):
    rng = np.random.default_rng(seed)
    n = p["X"].shape[0]
    p = dict(p)
    p["alpha_v"] = rng.uniform(0.0, 2.0, n).astype(np.float32)
    p["alpha_c"] = rng.uniform(0.0, 0.5, n).astype(np.float32)
    return p


def _energy(m, v, u):
    return float((m * (0.5 * (v * v).sum(1) + u)).sum())


def _oracle_step(p, dt):
    """kick(dt/2) + drift(dt) with the first pass's a, du; second pass; kick(dt/2)."""
    o = oracle.Oracle(oracle.Params(h_tol=1e-13, h_max_iter=64), mode="cells")
    st = oracle.State.from_particles(p)
    r0 = o.hydro(st, dt_ghost=dt, first_step=True)
    assert r0["density"]["status"] == 0 and r0["force"]["status"] == 0
    st.h = r0["density"]["h"].copy()
    st.alpha_v, st.alpha_c, st.div_prev = (r0["ghost"][k].copy() for k in ("alpha_v", "alpha_c", "div_prev"))
    o.kick_drift(st, r0["force"]["a"], r0["force"]["du"], 0.5 * dt, dt)
    r1 = o.hydro(st, dt_ghost=dt, first_step=False)
    assert r1["density"]["status"] == 0 and r1["force"]["status"] == 0
    o.kick_drift(st, r1["force"]["a"], r1["force"]["du"], 0.5 * dt, 0.0)
    return st, r0, r1


@pytest.mark.parametrize("case", ["poisson", "gresho", "sod"])
def test_kdk_step_conservation(case):
    from paper_2505_14538_b200 import Context

    if case == "poisson":
        p = _switches(W.poisson(4096, seed=71, vel_sigma=0.3, u_sigma=0.4), 8)
    elif case == "gresho":
        p = _switches(W.gresho(24, jitter=0.1), 9)
    else:
        p = _switches(W.sod(16), 10)
    m = p["m"].astype(np.float64)
    v0, u0 = p["v"].astype(np.float64), p["u"].astype(np.float64)
    dt = 0.5 * oracle_hydro(p, dt_ghost=1e-3)["dt"]  # half the oracle's CFL step
    st, r0, r1 = _oracle_step(p, dt)
    ctx = Context(p, h_tol=1e-6)
    ctx.density()
    ctx.gradient(dt)
    ctx.force()
    ctx.kick_drift(0.5 * dt, dt)
    ctx.density()
    ctx.gradient(dt)
    ctx.force()
    ctx.kick_drift(0.5 * dt, 0.0)
    v, u, X = (ctx.get(k).astype(np.float64) if k != "X" else ctx.get(k) for k in ("v", "u", "X"))
    ctx.close()
    # momentum
    P0 = (m[:, None] * v0).sum(0)
    dP_g = (m[:, None] * v).sum(0) - P0
    dP_o = (m[:, None] * st.v).sum(0) - P0
    # momentum scale: sum m |v| over the step (Sod starts at rest: its velocities are the step's own)
    pscale = float((m * (np.linalg.norm(v0, axis=1) + np.linalg.norm(st.v, axis=1))).sum())
    assert np.all(np.abs(dP_g) <= 1e-6 * pscale), (dP_g, pscale)
    assert np.all(np.abs(dP_g - dP_o) <= 1e-6 * pscale), (dP_g, dP_o)
    # energy
    E0 = _energy(m, v0, u0)
    dE_g = _energy(m, v, u) - E0
    dE_o = _energy(m, st.v, st.u) - E0
    assert abs(dE_g - dE_o) <= 1e-6 * abs(E0), (dE_g, dE_o, E0)
    # per particle: the step's change dt (a0 + a1)/2 to 1e-4 of its term scale
    sa = 0.5 * dt * (r0["force"]["scale_a"] + r1["force"]["scale_a"])
    err_v = np.abs(v - st.v).max(1)
    assert np.all(err_v <= 1e-4 * sa + 1e-6 * np.abs(st.v).max(1)), err_v.max()
    (s0, c0), (s1, c1) = du_tolerance(r0["force"]), du_tolerance(r1["force"])
    tol_u = 0.5 * dt * (1e-4 * (s0 + s1) + c0 + c1) + 1e-6 * np.abs(st.u)
    assert np.all(np.abs(u - st.u) <= tol_u), np.abs(u - st.u).max()
    # positions: the drift by dt (v0 + dt a0 / 2) carries a0's 1e-4 term-scale error and the f32
    # rounding of the displacement (2^32 / L grid units)
    unit = 2.0 ** 32 / np.asarray(p["box"], dtype=np.float64)[None, :]
    tol_x = (1e-4 * 0.5 * dt * dt * r0["force"]["scale_a"][:, None] + 1e-6 * np.abs(st.v) * dt) * unit + 2.0
    dX = (X.astype(np.int64) - st.X.astype(np.int64) + 2 ** 31) % 2 ** 32 - 2 ** 31
    assert np.all(np.abs(dX) <= tol_x), np.abs(dX).max()


def test_pipelined_host_io_matches_blocking():
    """sph_stage_particles / sph_set_particles_staged / sph_get_async (include/sph.h: the
    pipelined host I/O of bench.py's e2e) give the same particles and results as
    sph_set_particles / sph_get: staged uploads overlap the previous pass, reads overlap the
    next, and each pass sees exactly its own inputs."""
    from paper_2505_14538_b200 import Context

    ps = [W.jittered_lattice(16, seed=70 + k, vel_sigma=0.1, u_sigma=0.3) for k in range(3)]
    ref = []
    ctx = Context(ps[0], h_tol=1e-6, device=0)
    for p in ps:
        ctx.set_particles(p)
        ctx.density()
        ctx.gradient(1e-3)
        ctx.force()
        ref.append({k: ctx.get(k) for k in ("a", "du", "rho", "h")})
    n = ps[0]["X"].shape[0]
    outs = [{"a": np.zeros((n, 3), np.float32), "du": np.zeros(n, np.float32), "rho": np.zeros(n, np.float32),
             "h": np.zeros(n, np.float32)} for _ in ps]
    ctx.stage_particles(ps[0])
    for k in range(len(ps)):
        ctx.set_particles_staged()
        if k + 1 < len(ps):
            ctx.stage_particles(ps[k + 1])
        ctx.density()
        ctx.gradient(1e-3)
        ctx.force()
        for f in outs[k]:
            ctx.get_async(f, outs[k][f])
    ctx.synchronize()
    for k in range(len(ps)):
        for f in ("rho", "h"):
            assert np.array_equal(outs[k][f], ref[k][f]), (k, f)
        for f in ("a", "du"):  # (the pair-once force sums land in reduction order)
            scale = np.abs(ref[k][f]).max()
            assert np.abs(outs[k][f] - ref[k][f]).max() <= 1e-5 * scale, (k, f)
    with pytest.raises(Exception):
        ctx.set_particles_staged()  # nothing staged
    ctx.close()
