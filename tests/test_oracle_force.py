"""Pins of the oracle's finalize, gradient loop, gradient ghost, force loop, CFL dt and
kick/drift (SURVEY.md §8(c) Pins 5, 10, 13-16, 19-22) -- CPU only."""
import math

import numpy as np
import pytest

import workloads as W


def _state(orc, p):
    return orc.State.from_particles(p)


def _rand_set(seed=10, n=700):
    """Poisson positions with uneven h, u, v, alpha: every force term is active."""
    rng = np.random.default_rng(seed)
    p = W.poisson(n, seed=seed, vel_sigma=0.3, u_sigma=0.4)
    p["alpha_v"] = rng.uniform(0.0, 2.0, n).astype(np.float32)
    p["alpha_c"] = rng.uniform(0.0, 1.0, n).astype(np.float32)
    p["m"] = (p["m"] * rng.uniform(0.5, 1.5, n)).astype(np.float32)
    return p


def _forces(orc, p, fh_mode=0):
    o = orc.Oracle(orc.Params(fh_mode=fh_mode), mode="brute")
    st = _state(orc, p)
    r = o.hydro(st, dt_ghost=1e-3, first_step=True)
    return st, r


@pytest.mark.parametrize("fh_mode", [0, 1])
def test_momentum_and_energy_conservation(orc, fh_mode):
    """Pin-13: sum m a = 0 within 1e-10 of sum m|a|; Pin-14: sum m (v.a + du/dt) = 0
    within 1e-10 of sum m(|v.a| + |du|) (needs the viscous-heating term, R10).  Both
    f readings (R8) conserve exactly."""
    p = _rand_set()
    st, r = _forces(orc, p, fh_mode)
    a, du = r["force"]["a"], r["force"]["du"]
    m = st.m
    P = (m[:, None] * a).sum(0)
    assert np.all(np.abs(P) <= 1e-10 * (m[:, None] * np.abs(a)).sum(0))
    va = (st.v * a).sum(1)
    E = (m * (va + du)).sum()
    assert abs(E) <= 1e-10 * (m * (np.abs(va) + np.abs(du))).sum()
    assert np.abs(a).max() > 0 and np.abs(du).max() > 0


def test_lattice_at_rest_is_force_free(orc):
    """Pin-10: lattice at rest with uniform u -> a = 0, du/dt = 0,
    lap u = 0, no conduction (to 1e-12 of the term scales); v_sig = 2 c."""
    p = W.lattice(16, h_factor=1.0)  # power-of-two n: lattice exact on the 2^-32 grid
    st, r = _forces(orc, p)
    fo, gr = r["force"], r["gradient"]
    assert np.all(np.abs(fo["a"]) <= 1e-12 * fo["scale_a"][:, None])
    assert np.all(np.abs(fo["du"]) <= 1e-12 * np.maximum(fo["scale_u"], 1e-300))
    assert np.all(np.abs(gr["lap_u"]) < 1e-9)
    c = r["finalize"]["c"]
    assert np.allclose(gr["v_sig"], 2 * c, rtol=1e-15) and np.allclose(fo["v_sig"], 2 * c, rtol=1e-15)


def test_lap_of_quadratic_on_lattice(orc):
    """Pin-11: Brookshaw lap(x^2) on the lattice at h* = 1.962535969 (= Omega x 2) for
    interior particles (R16)."""
    n = 16
    p = W.lattice(n, h_factor=1.0)
    x = W.positions_f64(p)
    st = _state(orc, p)
    st.u = (x[:, 0] - 0.5) ** 2 + 1.0
    o = orc.Oracle(orc.Params(h_tol=1e-13), mode="cells")
    d = o.density(st)
    fin = o.finalize(st, d)
    g = o.gradient(st, d["h"], d["rho"], fin["c"])
    inside = np.all((x > 3.0 / n) & (x < 1 - 3.0 / n), axis=1)
    assert np.allclose(g["lap_u"][inside], 1.962535969, rtol=0, atol=1e-8)


def test_galilean_invariance_force(orc):
    """Pin-15 (R5, R12): a constant velocity shift leaves v_sig, a, du/dt unchanged."""
    p = _rand_set(seed=11, n=400)
    st1, r1 = _forces(orc, p)
    p2 = dict(p); p2["v"] = (p["v"] + np.array([2.0, -3.0, 1.0], np.float32)).astype(np.float32)
    # use the shifted float32 velocities in both to avoid float rounding differences
    p1 = dict(p); p1["v"] = (p2["v"] - np.array([2.0, -3.0, 1.0], np.float32)).astype(np.float32)
    _, r1 = _forces(orc, p1)
    st2 = _state(orc, p1); st2.v = st2.v + np.array([2.0, -3.0, 1.0])
    r2 = orc.Oracle(mode="brute").hydro(st2, dt_ghost=1e-3, first_step=True)
    for k in ("a", "du", "v_sig"):
        assert np.allclose(r1["force"][k], r2["force"][k], rtol=1e-8, atol=1e-8 * np.abs(r1["force"][k]).max())
    assert np.allclose(r1["gradient"]["v_sig"], r2["gradient"]["v_sig"], rtol=1e-12)


def test_signal_velocity_facts(orc):
    """Pin-16: in a uniformly expanding flow (v = H x about the centre, every
    pair receding) mu = 0 and v_sig = c_i + c_j = 2c; in a contracting flow v_sig > 2c."""
    n = 8
    p = W.lattice(n, h_factor=1.0)
    x = W.positions_f64(p)
    st = _state(orc, p)
    inside = np.all((x > 2.6 / n) & (x < 1 - 2.6 / n), axis=1)
    o = orc.Oracle(mode="cells")
    for sgn in (1.0, -1.0):
        st.v = sgn * 0.1 * (x - 0.5)
        d = o.density(st, fixed_h=True)
        fin = o.finalize(st, d)
        g = o.gradient(st, d["h"], d["rho"], fin["c"])
        if sgn > 0:
            assert np.allclose(g["v_sig"][inside], 2 * fin["c"][inside], rtol=1e-14)
        else:
            assert np.all(g["v_sig"][inside] > 2 * fin["c"][inside] * (1 + 1e-6))


def test_two_body_force_is_repulsive_and_antisymmetric(orc):
    """Two particles at rest, q = 1, positive pressure: m_i a_i = -m_j a_j, along r_ij,
    pointing apart (a_i . r_ij > 0, R4)."""
    L, h = 10.0, 0.5
    X = np.array([[0, 0, 0], [int(0.3 / L * 2 ** 32), int(0.4 / L * 2 ** 32), 0]], dtype=np.uint32)
    p = {"X": X, "v": np.zeros((2, 3), np.float32), "m": np.array([1.0, 2.0], np.float32),
         "u": np.array([1.0, 3.0], np.float32), "h": np.array([h, h], np.float32),
         "alpha_v": np.zeros(2, np.float32), "alpha_c": np.zeros(2, np.float32), "box": np.array([L, L, L])}
    st = _state(orc, p)
    o = orc.Oracle(mode="brute")
    d = o.density(st, fixed_h=True)
    fin = o.finalize(st, d)
    fo = o.force(st, d["h"], fin["f"], fin["P"], fin["c"], fin["B"], d["rho"], st.alpha_v, st.alpha_c)
    a = fo["a"]
    assert np.allclose(1.0 * a[0], -2.0 * a[1], rtol=1e-13, atol=0)
    rij = -X[1].astype(np.float64) * L / 2 ** 32  # r_0 - r_1 (R4), exact fixed-point value
    assert np.dot(a[0], rij) > 0
    assert abs(np.cross(a[0], rij)).max() < 1e-12 * np.linalg.norm(a[0])
    # no conduction (alpha_c = 0), no viscosity (at rest): du = 0
    assert np.allclose(fo["du"], 0.0, atol=1e-15)


def test_conduction_flows_hot_to_cold(orc):
    """Eq. 19 (R11): with alpha_c > 0, equal pressures, at rest: energy flows from the hot
    to the cold particle and the total is conserved."""
    L, h = 10.0, 0.5
    X = np.array([[0, 0, 0], [int(0.45 / L * 2 ** 32), 0, 0]], dtype=np.uint32)
    p = {"X": X, "v": np.zeros((2, 3), np.float32), "m": np.array([1.0, 1.0], np.float32),
         "u": np.array([4.0, 1.0], np.float32), "h": np.array([h, h], np.float32),
         "alpha_v": np.zeros(2, np.float32), "alpha_c": np.array([0.5, 0.5], np.float32), "box": np.array([L, L, L])}
    st = _state(orc, p)
    o = orc.Oracle(mode="brute")
    d = o.density(st, fixed_h=True)
    fin = o.finalize(st, d)
    fo = o.force(st, d["h"], fin["f"], fin["P"], fin["c"], fin["B"], d["rho"], st.alpha_v, st.alpha_c)
    # pressure work is zero at rest (v_ij = 0): du is conduction only
    assert fo["du"][0] < 0 < fo["du"][1]
    assert abs(fo["du"][0] + fo["du"][1]) < 1e-14 * abs(fo["du"][0])


def test_sod_interfaces_push_toward_low_pressure(orc):
    """C2 (Sod): the layers touching each interface are pushed from the high-pressure
    (left, P = 1) toward the low-pressure (right, P = 0.1) gas, the net momentum change of
    the gas around each interface points the same way, and particles farther than 2H from
    an interface feel no force (the force is a sum of pair terms inside the support)."""
    n = 8
    p = W.sod(n)
    st = _state(orc, p)
    r = orc.Oracle(mode="cells").hydro(st)
    x = W.positions_f64(p)[:, 0]
    ax = r["force"]["a"][:, 0]
    dx = 1.0 / n
    touch1 = np.abs(x - 1.0) < dx
    touch0 = (x < dx) | (x > 2.0 - dx)
    assert np.all(ax[touch1] > 1.0) and np.all(ax[touch0] < -1.0)
    around1 = np.abs(x - 1.0) < 0.5
    assert (st.m * ax)[around1].sum() > 0 > (st.m * ax)[~around1].sum()
    far = (np.abs(x - 0.5) < 0.1) | (np.abs(x - 1.5) < 0.1)
    assert np.all(np.abs(ax[far]) < 1e-1) and np.all(np.abs(ax[touch1]) > 1.0)


def test_finalize_eos_and_balsara(orc):
    """Pin-5: rho = 1, u = 7.5 -> P = 5; u = 0 -> P = c = 0.  Balsara (R14):
    div = 0 -> B = 0; curl = 0, div != 0 -> B = |div|/(|div| + 1e-4 c/h)."""
    o = orc.Oracle()
    st = orc.State(X=np.zeros((3, 3), np.uint32), box=np.ones(3), v=np.zeros((3, 3)), m=np.ones(3),
                   u=np.array([7.5, 0.0, 1.5]), h=np.array([0.1, 0.1, 0.1]), alpha_v=np.zeros(3),
                   alpha_c=np.zeros(3), div_prev=np.zeros(3))
    dens = np.zeros((3, 8))
    dens[:, 0] = 1.0
    dens[0, 5] = 2.0        # curl only
    dens[2, 4] = -3.0       # div only
    fin = o.finalize(st, {"h": st.h, "_dens": dens})
    assert abs(fin["P"][0] - 5.0) < 1e-15 and fin["P"][1] == 0.0 and fin["c"][1] == 0.0
    assert fin["B"][0] == 0.0 and fin["B"][1] == 0.0
    c2 = math.sqrt(5.0 / 3.0 * (2.0 / 3.0 * 1.5))
    assert abs(fin["B"][2] - 3.0 / (3.0 + 1e-4 * c2 / 0.1)) < 1e-15
    assert np.all(fin["f"] == 1.0)  # drho/dh = 0 -> Omega = 1


def test_gradient_ghost_switches(orc):
    """Pin-19 and S:248-250: constant div (Ddot = 0) -> alpha_loc = 0, alpha_v decays by
    exp(-ell c dt/H); strong compression raises alpha_v to alpha_loc <= alpha_v_max in one
    step; uniform u (lap u = 0) -> alpha_c decays and never goes below alpha_c_min; bounds hold."""
    o = orc.Oracle()
    n = 4
    st = orc.State(X=np.zeros((n, 3), np.uint32), box=np.ones(3), v=np.zeros((n, 3)), m=np.ones(n),
                   u=np.ones(n), h=np.full(n, 0.05), alpha_v=np.array([1.0, 0.1, 0.5, 1.9]),
                   alpha_c=np.array([0.5, 0.2, 0.9, 0.0]), div_prev=np.array([0.3, 0.0, 0.0, 0.0]))
    c = np.full(n, 1.2)
    div = np.array([0.3, -50.0, 0.0, 0.0])
    grad = {"_grad": np.stack([np.full(n, 2.4), np.array([0.0, 0.0, 0.0, 5.0])], 1)}
    dt = 0.01
    g = o.gradient_ghost(st, st.h, c, div, grad, dt, first_step=False)
    H = 0.1
    assert abs(g["alpha_v"][0] - 1.0 * math.exp(-0.05 * 1.2 * dt / H)) < 1e-15
    S = H * H * 50.0 / dt
    aloc = 2.0 * S / (2.4 ** 2 + S)
    assert abs(g["alpha_v"][1] - aloc) < 1e-15 and aloc <= 2.0
    assert g["alpha_c"][0] < 0.5 and g["alpha_c"][0] >= 0.0
    assert np.all((g["alpha_v"] >= 0) & (g["alpha_v"] <= 2.0))
    assert np.all((g["alpha_c"] >= 0) & (g["alpha_c"] <= 1.0))
    # ceiling alpha_c_max (1 - alpha_v/alpha_v_max): particle 3 has alpha_v ~ 1.9 -> ceiling ~0.05
    assert g["alpha_c"][3] <= 1.0 * (1 - g["alpha_v"][3] / 2.0) + 1e-15
    assert np.array_equal(g["div_prev"], div)


def test_dt_homogeneity(orc):
    """Pin-20: uniform h, v_sig -> dt = C_cfl 2 gamma_k h / v_sig; doubling
    v_sig halves dt."""
    o = orc.Oracle()
    h = np.full(10, 0.02)
    vs = np.full(10, 3.0)
    assert abs(o.dt(h, vs) - 0.1 * 4 * 0.02 / 3.0) < 1e-18
    assert abs(o.dt(h, 2 * vs) - 0.5 * o.dt(h, vs)) < 1e-18


def test_kdk_ballistic(orc):
    """Pin-21: with constant a, 100 KDK steps reproduce x0 + v0 t + a t^2/2 to
    round-off (positions on the 2^-32 grid, wrapped)."""
    p = W.poisson(50, seed=12)
    st = _state(orc, p)
    x0 = W.positions_f64(p)
    v0 = st.v.copy()
    a = np.tile(np.array([[0.3, -0.2, 0.1]]), (50, 1))
    du = np.zeros(50)
    dt = 1e-3
    for _ in range(100):
        o = orc.Oracle()
        o.kick_drift(st, a, du, 0.5 * dt, dt)
        o.kick_drift(st, a, du, 0.5 * dt, 0.0)
    t = 100 * dt
    exp = np.mod(x0 + v0 * t + 0.5 * a * t * t, 1.0)
    got = st.X.astype(np.float64) / 2 ** 32
    err = np.abs(((got - exp) + 0.5) % 1.0 - 0.5)
    assert err.max() < 1e-8
    assert np.allclose(st.v, v0 + a * t, rtol=0, atol=1e-12)


def test_gresho_initial_conditions():
    """Pin-22: v_theta(0.1) = 0.5, p(0.1) = 5.125, v_theta(0.2) = 1,
    v_theta(0.3) = 0.5, p(0) = 5, p(r >= 0.4) = 3 + 4 ln 2; continuity at 0.2 and 0.4."""
    vt, p = W.gresho_analytic(np.array([0.0, 0.1, 0.2, 0.3, 0.4, 0.7]))
    assert np.allclose(vt, [0, 0.5, 1.0, 0.5, 0, 0], atol=1e-14)
    assert abs(p[0] - 5) < 1e-14 and abs(p[1] - 5.125) < 1e-14
    assert abs(p[4] - (3 + 4 * math.log(2))) < 1e-12 and abs(p[5] - (3 + 4 * math.log(2))) < 1e-14
    a, b = W.gresho_analytic(np.array([0.4 - 1e-12, 0.4 + 1e-12]))
    assert abs(b[0] - b[1]) < 1e-9
    g = W.gresho(16)
    x = W.positions_f64(g)
    r = np.hypot(x[:, 0] - 0.5, x[:, 1] - 0.5)
    speed = np.hypot(g["v"][:, 0], g["v"][:, 1])
    assert np.allclose(speed, W.gresho_analytic(r)[0], atol=1e-6)
    assert np.allclose(g["u"], 1.5 * W.gresho_analytic(r)[1], rtol=1e-6)


def test_tolerance_scales_bound_their_sums(orc):
    """The per-particle tolerance scales the parity tests use are sums of term magnitudes, so
    each bounds its sum: |div|, |curl_a| <= scale_dv, |lap u| <= scale_lap, |a_a| <= scale_a,
    |du| <= scale_u; all vanish on the lattice at rest (where the sums are exactly 0).  The
    conduction bound scale_cond is 0 when alpha_c = 0 and grows like sqrt(eps) at P_i = P_j."""
    p = _rand_set(seed=12, n=600)
    st, r = _forces(orc, p)
    d, gr, fo = r["density"], r["gradient"], r["force"]
    assert np.all(np.abs(d["div"]) <= d["scale_dv"] * (1 + 1e-12))
    assert np.all(np.abs(d["curl"]) <= d["scale_dv"][:, None] * (1 + 1e-12))
    assert np.all(np.abs(gr["lap_u"]) <= gr["scale_lap"] * (1 + 1e-12))
    assert np.all(np.abs(fo["a"]) <= fo["scale_a"][:, None] * (1 + 1e-12))
    assert np.all(np.abs(fo["du"]) <= fo["scale_u"] * (1 + 1e-12))
    assert np.all(fo["scale_cond"] > 0)
    q = dict(p)
    q["alpha_c"] = np.zeros_like(p["alpha_c"])
    r0 = orc.Oracle(orc.Params(alpha_c_max=0.0), mode="brute").hydro(_state(orc, q), dt_ghost=1e-3, first_step=True)
    assert np.all(r0["force"]["scale_cond"] == 0)
    lat = W.lattice(8, h_factor=1.0)
    rl = orc.Oracle(orc.Params(h_max_iter=0), mode="brute").hydro(_state(orc, lat), dt_ghost=1e-3, first_step=True)
    assert np.all(rl["density"]["scale_dv"] == 0) and np.all(rl["gradient"]["scale_lap"] == 0)
