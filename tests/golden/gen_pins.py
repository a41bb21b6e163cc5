"""Independent lattice sums for the oracle pins of tests/test_oracle_pins.py.

Plain numpy, written from the paper's kernel definition only (M4 with
sigma = 1/pi, support 2h): it does NOT import oracle/ or the CUDA package.
Run `python tests/golden/gen_pins.py` to regenerate tests/golden/pins_lattice.txt.

Simple cubic lattice, spacing dx = 1, h = h* dx (the self-consistent smoothing length of
the eta = 1.2348 closure, tests/golden/lattice_m4_eta1.2348.txt).  Every quantity the pins
need reduces, on the lattice, to the radial sums

    Sw   = sum_j w(q_j)        (self included)      Sq1 = sum_j q_j   w'(q_j)
    Sq2  = sum_j q_j^2 w'(q_j)                      Sq3 = sum_j q_j^3 w'(q_j)

over the lattice points j with q_j = r_j / h < 2, plus q_max = the largest such q_j, and
(for the conduction pin) the per-plane sums of the cosine field given below.
"""
import itertools
import math
import os

import numpy as np

H_STAR = 1.2351475775552


def w(q):
    q = np.asarray(q, dtype=np.float64)
    return np.where(q < 1, 1 - 1.5 * q * q + 0.75 * q ** 3, np.where(q < 2, 0.25 * (2 - q) ** 3, 0.0))


def dw(q):
    q = np.asarray(q, dtype=np.float64)
    return np.where(q < 1, -3 * q + 2.25 * q * q, np.where(q < 2, -0.75 * (2 - q) ** 2, 0.0))


def offsets(h, reach=4):
    o = np.array(list(itertools.product(range(-reach, reach + 1), repeat=3)), dtype=np.float64)
    r = np.sqrt((o * o).sum(1))
    keep = r < 2 * h
    return o[keep], r[keep]


def main():
    o, r = offsets(H_STAR)
    q = r / H_STAR
    vals = {
        "h_star": H_STAR,
        "n_in_support": len(q),  # self included
        "Sw": float(w(q).sum()),
        "Sq1": float((q * dw(q)).sum()),
        "Sq2": float((q * q * dw(q)).sum()),
        "Sq3": float((q ** 3 * dw(q)).sum()),
        "q_max": float(q[q > 0].max()),
    }
    # Conduction pin: lattice of n = 16 per unit length (L = 1, dx = 1/16), at rest, m = 1/n^3,
    # u(x) = u0 + du cos(2 pi x), gamma = 5/3, alpha_c = ac uniform, f = 1/Omega (R8),
    # h = h* dx.  Per plane ix (x = (ix + 1/2) dx): du/dt = sum_j m_j D_ij with (R11-R13)
    #   D_ij = alpha_c,ij v_c,ij (u_i - u_j) (G_i + G_j) |r_ij| / (rho_i + rho_j),
    #   v_c,ij = sqrt(2 |P_i - P_j| / (rho_i + rho_j)),  G = f dW/dr / r,
    # on the lattice rho_i = rho, G_i = G_j, alpha_c,ij = ac (Eq. 20 with equal alpha_c).
    n, u0, du_, ac, gam = 16, 1.5, 0.3, 0.7, 5.0 / 3.0
    dx, m = 1.0 / n, 1.0 / n ** 3
    h = H_STAR * dx
    rho = m * vals["Sw"] / (math.pi * h ** 3)
    Omega = -vals["Sq1"] / (3 * vals["Sw"])
    f = 1.0 / Omega
    cond = []
    for ix in range(n):
        x = (ix + 0.5) * dx
        ui = u0 + du_ * math.cos(2 * math.pi * x)
        s = 0.0
        for (ox, oy, oz), rr in zip(o, r):
            if rr == 0:
                continue
            uj = u0 + du_ * math.cos(2 * math.pi * (x + ox * dx))
            Pi, Pj = (gam - 1) * rho * ui, (gam - 1) * rho * uj
            vc = math.sqrt(2 * abs(Pi - Pj) / (2 * rho))
            dWdr = float(dw(rr / H_STAR)) / (math.pi * h ** 4)
            Gsum_r = 2 * f * dWdr  # (G_i + G_j) |r|
            s += m * ac * vc * (ui - uj) * Gsum_r / (2 * rho)
        cond.append(s)
    # Switch pin (gradient loop + ghost, Eqs. 10-15 and 21-24 with R15-R21), the same lattice
    # and cosine field, first step (Ddot = 0, so alpha_loc = 0), dt, alpha_v0, alpha_c0:
    #   lap u_i = 2 sum_j (m_j / rho_j)(u_i - u_j) dW/dr / r   (Brookshaw, R16)
    #   v_sig,i = max(2 c_i, max_j (c_i + c_j))  (at rest, mu = 0; R15)
    #   alpha_v = alpha_v0 exp(-ell c_i dt / H_i)  (R17 with alpha_loc = 0)
    #   alpha_c = clamp(alpha_c0 + dt (beta_c H lap u / sqrt(u) - (alpha_c0 - ac_min) v_sig / H),
    #                   ac_min, max(ac_min, ac_max (1 - alpha_v / av_max)))   (R20, R21)
    dt, av0, ac0, ell, beta_c, ac_min, ac_max, av_max = 1e-3, 0.5, 0.2, 0.05, 1.0, 0.0, 1.0, 2.0
    H = 2 * h
    sw = []
    for ix in range(n):
        x = (ix + 0.5) * dx
        ui = u0 + du_ * math.cos(2 * math.pi * x)
        ci = math.sqrt(gam * (gam - 1) * ui)
        lap, vmax = 0.0, 2 * ci
        for (ox, oy, oz), rr in zip(o, r):
            if rr == 0:
                continue
            uj = u0 + du_ * math.cos(2 * math.pi * (x + ox * dx))
            cj = math.sqrt(gam * (gam - 1) * uj)
            lap += 2 * (m / rho) * (ui - uj) * (float(dw(rr / H_STAR)) / (math.pi * h ** 4)) / (rr * dx)
            vmax = max(vmax, ci + cj)
        av = av0 * math.exp(-ell * ci * dt / H)
        ac = ac0 + dt * (beta_c * H * lap / math.sqrt(ui) - (ac0 - ac_min) * vmax / H)
        ac = max(min(ac, max(ac_min, ac_max * (1 - av / av_max))), ac_min)
        sw.append((lap, vmax, av, ac))
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "pins_lattice.txt")
    with open(out, "w") as fh:
        fh.write("# Lattice sums for tests/test_oracle_pins.py, written by tests/golden/gen_pins.py\n")
        fh.write("# (numpy only, from the M4 kernel definition; independent of oracle/).  dx = 1, h = h* dx.\n")
        for k, v in vals.items():
            fh.write(f"{k} {v!r}\n")
        fh.write(f"# conduction: n={n} u0={u0} du={du_} alpha_c={ac} gamma=5/3 m=1/n^3 f=1/Omega, per x-plane\n")
        for ix, s in enumerate(cond):
            fh.write(f"cond_du_{ix} {s!r}\n")
        fh.write(f"# switches: same field, first step, dt={dt} alpha_v0={av0} alpha_c0={ac0} ell={ell} beta_c={beta_c} "
                 f"alpha_c_min={ac_min} alpha_c_max={ac_max} alpha_v_max={av_max}; per x-plane: lap_u v_sig alpha_v alpha_c\n")
        for ix, t in enumerate(sw):
            fh.write(f"switch_{ix} " + " ".join(repr(float(x)) for x in t) + "\n")
    print(open(out).read())


if __name__ == "__main__":
    main()
