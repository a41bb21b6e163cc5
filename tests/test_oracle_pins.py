"""Value pins of the oracle's force loop and switches that conservation alone cannot fix
(VERDICT r1 "What's missing" 5): the f = 1/Omega reading (R8), the Pi_ij magnitude (Eq. 9,
R9) with the viscous heating (R10), the conduction term (Eqs. 19-22, R11-R13) and the
alpha_c source (Eq. 21, R20).  CPU only.

Expected values come from closed forms on the simple cubic lattice and from
tests/golden/pins_lattice.txt, written by tests/golden/gen_pins.py (numpy only, from the M4
kernel definition, no oracle import).  The pressure force is also pinned off-lattice by the
variational identity of grad-h SPH: with f = 1/Omega and equal masses, the accelerations are
exactly -(1/m) dE/dx_i of E = sum_i m u_i(rho_i) at fixed entropy (Price 2012), and du_i/dt
is exactly (P_i / rho_i^2) d rho_i/dt -- checked against central finite differences of an
independent numpy density + h solve.
"""
import math
import os

import numpy as np
import pytest

import workloads as W

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "pins_lattice.txt")
GAM = 5.0 / 3.0


def _gold():
    d = {}
    for ln in open(GOLD):
        if ln.startswith("#") or not ln.strip():
            continue
        k, *v = ln.split()
        d[k] = [float(x) for x in v] if len(v) > 1 else float(v[0])
    return d


def _lattice_state(orc, n=16):
    p = W.lattice(n, h_factor=1.0)
    st = orc.State.from_particles(p)
    x = W.positions_f64(p)
    return st, x


def _stages(orc, st, alpha_v, alpha_c, fh_mode=0):
    """density (h iteration) -> finalize -> gradient -> force with the given switches."""
    o = orc.Oracle(orc.Params(fh_mode=fh_mode, h_tol=1e-13), mode="brute")
    d = o.density(st)
    assert d["status"] == 0
    fin = o.finalize(st, d)
    gr = o.gradient(st, d["h"], d["rho"], fin["c"])
    fo = o.force(st, d["h"], fin["f"], fin["P"], fin["c"], fin["B"], d["rho"], alpha_v, alpha_c)
    return d, fin, gr, fo


def _interior(x, lo, hi, n=16, axes=(0,)):
    """particles whose lattice plane index lies in [lo, hi] along every axis in `axes`"""
    k = np.floor(x * n).astype(int)
    ok = np.ones(x.shape[0], dtype=bool)
    for a in axes:
        ok &= (k[:, a] >= lo) & (k[:, a] <= hi)
    return ok


@pytest.mark.parametrize("fh_mode", [0, 1])
def test_linear_pressure_field_gives_minus_grad_p_over_rho(orc, fh_mode):
    """Lattice at rest, u = u0 + g x (so P linear, rho uniform): Eq. 17 with f = 1/Omega gives
    a = -grad P / rho = -(gamma - 1) g x_hat EXACTLY (lattice symmetry: sum_j grad W_ij = 0
    and sum_j r_x^2 W'/r = (1/3) sum_j r W' = -rho Omega / m), du/dt = 0.  The literal Eq. 8
    (fh_mode = 1, f = Omega) gives -Omega^2 (gamma - 1) g instead.  Pins R8 and the
    A_i G_i + A_j G_j structure.  Planes within 2h of the periodic jump of u are excluded."""
    G = _gold()
    st, x = _lattice_state(orc)
    g = 0.8
    st.u[:] = 1.5 + g * x[:, 0]
    n = st.X.shape[0]
    _, _, _, fo = _stages(orc, st, np.zeros(n), np.zeros(n), fh_mode)
    ok = _interior(x, 3, 12)
    Omega = -G["Sq1"] / (3 * G["Sw"])
    want = -(GAM - 1) * g * (1.0 if fh_mode == 0 else Omega ** 2)
    a = fo["a"][ok]
    assert np.all(np.abs(a[:, 0] - want) <= 1e-11 * abs(want))
    assert np.all(np.abs(a[:, 1:]) <= 1e-11 * abs(want))
    assert np.all(np.abs(fo["du"][ok]) <= 1e-12)


def test_uniform_compression_viscous_heating_and_vsig(orc):
    """Lattice, uniform u, v = -k (x - c): interior particles feel a = 0 and
      du/dt = 3 k P / rho                                    (pressure work, exact with f = 1/Omega)
            - (m alpha B k^2 f / (2 rho)) (2 c Sq2 / (pi h^2) + beta k Sq3 / (pi h))   (R9, R10)
    from Pi_ij = -alpha_bar mu v_sig / rho_bar with mu = -k r, v_sig,ij = 2c + beta k r,
    gbar = f W'(r) / r, v_ij . r_ij = -k r^2; B = 3 k Omega / (3 k Omega + 1e-4 c / h)
    (div v = -3 k Omega on the lattice, curl = 0; R14).  v_sig (gradient and force loops)
    = 2 c + beta k r_max.  Lattice sums Sq2, Sq3, q_max: tests/golden/pins_lattice.txt."""
    G = _gold()
    st, x = _lattice_state(orc)
    k, alpha0, beta = 2.0, 1.5, 3.0
    st.v[:] = -k * (x - 0.5)
    n = st.X.shape[0]
    d, fin, gr, fo = _stages(orc, st, np.full(n, alpha0), np.zeros(n))
    # (B_j of a neighbour within 2h of the periodic jump of v differs: two supports from it)
    ok = _interior(x, 5, 10, axes=(0, 1, 2))
    assert ok.sum() == 216
    dx, m, u = 1.0 / 16, 1.0 / 16 ** 3, 1.5
    h = G["h_star"] * dx
    rho = m * G["Sw"] / (math.pi * h ** 3)
    Omega = -G["Sq1"] / (3 * G["Sw"])
    f = 1 / Omega
    P = (GAM - 1) * rho * u
    c = math.sqrt(GAM * P / rho)
    B = 3 * k * Omega / (3 * k * Omega + 1e-4 * c / h)
    du_p = 3 * k * P / rho
    du_v = -(m * alpha0 * B * k * k * f / (2 * rho)) * (2 * c * G["Sq2"] / (math.pi * h ** 2) +
                                                        beta * k * G["Sq3"] / (math.pi * h))
    assert du_v > 0.2 * du_p  # the viscous heating is a sizeable part of the check
    assert np.allclose(d["h"][ok], h, rtol=1e-12, atol=0)
    assert np.allclose(fin["B"][ok], B, rtol=1e-10, atol=0)
    assert np.all(np.abs(fo["du"][ok] - (du_p + du_v)) <= 1e-10 * (du_p + du_v))
    assert np.all(np.abs((fo["du"][ok] - du_p) - du_v) <= 1e-9 * du_v)  # the viscous part alone
    assert np.all(np.abs(fo["a"][ok]) <= 1e-11 * fo["scale_a"][ok][:, None])
    vs = 2 * c + beta * k * G["q_max"] * h
    assert np.allclose(gr["v_sig"][ok], vs, rtol=1e-12, atol=0)
    assert np.allclose(fo["v_sig"][ok], vs, rtol=1e-12, atol=0)


def test_conduction_cosine_field(orc):
    """Lattice at rest, u = 1.5 + 0.3 cos(2 pi x), alpha_c = 0.7 uniform, no viscosity: du/dt
    is the conduction sum alone (Eqs. 19-22 with R11-R13: bracket f_i W'(h_i) + f_j W'(h_j),
    denominator rho_i + rho_j, v_c = sqrt(2 |P_i - P_j| / (rho_i + rho_j)) at rest,
    alpha_c,ij the P-weighted mean); per-plane values from tests/golden/gen_pins.py."""
    G = _gold()
    st, x = _lattice_state(orc)
    st.u[:] = 1.5 + 0.3 * np.cos(2 * np.pi * x[:, 0])
    n = st.X.shape[0]
    _, _, _, fo = _stages(orc, st, np.zeros(n), np.full(n, 0.7))
    plane = np.floor(x[:, 0] * 16).astype(int)
    want = np.array([G[f"cond_du_{i}"] for i in range(16)])[plane]
    assert np.all(np.abs(fo["du"] - want) <= 1e-10 * np.abs(want).max())
    # (a finite pressure gradient is present too: the conduction pin checks du only)


def test_switches_from_cosine_field(orc):
    """The same field, one gradient loop + gradient ghost at the first step (Ddot = 0):
    Brookshaw lap u (R16), v_sig = max(2 c_i, max_j (c_i + c_j)) (R15), alpha_v decays by
    exp(-ell c dt / H) (R17 with alpha_loc = 0), alpha_c += dt (beta_c H lap u / sqrt(u) -
    (alpha_c - alpha_c_min) v_sig / H) clamped under the alpha_v ceiling (R20, R21); per-plane
    values from tests/golden/gen_pins.py."""
    G = _gold()
    st, x = _lattice_state(orc)
    st.u[:] = 1.5 + 0.3 * np.cos(2 * np.pi * x[:, 0])
    n = st.X.shape[0]
    st.alpha_v[:] = 0.5
    st.alpha_c[:] = 0.2
    o = orc.Oracle(orc.Params(h_tol=1e-13), mode="brute")
    d = o.density(st)
    fin = o.finalize(st, d)
    gr = o.gradient(st, d["h"], d["rho"], fin["c"])
    gh = o.gradient_ghost(st, d["h"], fin["c"], d["div"], gr, 1e-3, True)
    plane = np.floor(x[:, 0] * 16).astype(int)
    sw = np.array([G[f"switch_{i}"] for i in range(16)])[plane]
    assert np.allclose(gr["lap_u"], sw[:, 0], rtol=1e-10, atol=1e-10 * np.abs(sw[:, 0]).max())
    assert np.allclose(gr["v_sig"], sw[:, 1], rtol=1e-12, atol=0)
    assert np.allclose(gh["alpha_v"], sw[:, 2], rtol=1e-12, atol=0)
    assert np.allclose(gh["alpha_c"], sw[:, 3], rtol=1e-10, atol=0)
    assert np.abs(sw[:, 3] - 0.2).max() > 1e-3  # the source term moved alpha_c visibly


# ---- variational pin (off-lattice) ---------------------------------------------------------
def _w(q):
    return np.where(q < 1, 1 - 1.5 * q * q + 0.75 * q ** 3, np.where(q < 2, 0.25 * (2 - q) ** 3, 0.0))


def _dw(q):
    return np.where(q < 1, -3 * q + 2.25 * q * q, np.where(q < 2, -0.75 * (2 - q) ** 2, 0.0))


def _numpy_density(x, h0, eta=1.2348):
    """rho_i / m = nhat_i with h_i solving nhat_i h_i^3 = eta^3 (Eqs. 2, 5; R7), minimum image
    in the unit box; Newton on ln h to 1e-15 (independent of the oracle's iteration)."""
    d = x[:, None, :] - x[None, :, :]
    d -= np.round(d)
    r = np.sqrt((d * d).sum(-1))
    h = h0.copy()
    for _ in range(60):
        q = r / h[:, None]
        S0 = _w(q).sum(1)
        S1 = (q * _dw(q)).sum(1)
        g = S0 / math.pi - eta ** 3          # nhat h^3 - eta^3
        dg = -S1 / math.pi                   # h d(nhat h^3)/dh
        step = g / dg
        h = h * np.exp(-np.clip(step, -0.5, 0.5))
        if np.abs(step).max() < 1e-15:
            break
    q = r / h[:, None]
    return _w(q).sum(1) / (math.pi * h ** 3), h


@pytest.mark.parametrize("fh_mode", [0, 1])
def test_pressure_force_is_energy_gradient(orc, fh_mode):
    """Poisson set, equal masses, entropies K_i = (gamma-1) u_i / rho_i^(gamma-1): the oracle's
    a_i (no viscosity, no conduction) equals -(1/m) dE/dx_i, E = sum m K rho^(gamma-1)/(gamma-1),
    and its du_i/dt equals (P_i/rho_i^2) d rho_i/dt along v, to finite-difference accuracy --
    for f = 1/Omega only (fh_mode = 0); the literal Eq. 8 (fh_mode = 1) misses both by O(1 - Omega^2)."""
    N = 120
    p = W.poisson(N, seed=7, vel_sigma=0.3, u_sigma=0.3)
    st = orc.State.from_particles(p)
    x = W.positions_f64(p)
    m = 1.0 / N
    st.m[:] = m
    nh, h = _numpy_density(x, st.h.copy())
    rho = m * nh
    K = (GAM - 1) * st.u / rho ** (GAM - 1)
    zeros = np.zeros(N)
    st.h[:] = h
    _, fin, _, fo = _stages(orc, st, zeros, zeros, fh_mode)

    def energy(xx):
        r_, _ = _numpy_density(np.mod(xx, 1.0), h)
        return (m * K * (m * r_) ** (GAM - 1) / (GAM - 1)).sum()

    eps = 1e-6
    worst_a = 0.0
    for i in range(0, N, 17):
        for ax in range(3):
            xp, xm = x.copy(), x.copy()
            xp[i, ax] += eps
            xm[i, ax] -= eps
            a_fd = -(energy(xp) - energy(xm)) / (2 * eps) / m
            worst_a = max(worst_a, abs(fo["a"][i, ax] - a_fd) / np.abs(fo["a"]).max())
    rp, _ = _numpy_density(np.mod(x + eps * st.v, 1.0), h)
    rm, _ = _numpy_density(np.mod(x - eps * st.v, 1.0), h)
    drho = m * (rp - rm) / (2 * eps)
    du_fd = fin["P"] / rho ** 2 * drho
    worst_u = np.abs(fo["du"] - du_fd).max() / np.abs(du_fd).max()
    if fh_mode == 0:
        assert worst_a < 1e-6 and worst_u < 1e-6
    else:
        assert worst_a > 1e-3 and worst_u > 1e-3
