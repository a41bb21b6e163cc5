"""Seeded generators for configs C1-C5 (BASELINE.json `configs`).

No SPH arithmetic lives here: positions, masses, velocities and internal energies are
laid out from the initial-condition recipes only.  The one physical formula used is the
ideal-gas inversion u = P/((gamma-1) rho) that turns a prescribed pressure profile into
the internal energy the solver takes as input ("rho_0=1 with polytropic
index gamma=5/3"); it is an input recipe, not a step of the hot path.
"""
from __future__ import annotations

import math

import numpy as np

TWO32 = 2.0 ** 32
GAMMA_EOS = 5.0 / 3.0
ETA = 1.2348
# Self-consistent smoothing length of the simple cubic lattice for the M4 kernel with
# eta = 1.2348.  Used only as an initial guess h0 = H_STAR*dx;
# the oracle tests re-derive it independently.
H_STAR_LATTICE = 1.2351475775552


def _fixed_point(x: np.ndarray, box) -> np.ndarray:
    """float64 positions [N,3] -> uint32 fixed point on a 2^-32 L grid (wrapped)."""
    box = np.asarray(box, dtype=np.float64)
    f = np.mod(x / box[None, :], 1.0)
    xi = np.floor(f * TWO32).astype(np.int64)
    return np.mod(xi, 1 << 32).astype(np.uint32)


def positions_f64(p) -> np.ndarray:
    """uint32 fixed point -> float64 positions in [0, L)."""
    return p["X"].astype(np.float64) * (np.asarray(p["box"], dtype=np.float64)[None, :] / TWO32)


def _pack(name, X, v, m, u, h, box, alpha_v=0.1, alpha_c=0.0):
    n = X.shape[0]
    return {
        "name": name,
        "X": np.ascontiguousarray(X, dtype=np.uint32),
        "v": np.ascontiguousarray(v, dtype=np.float32).reshape(n, 3),
        "m": np.ascontiguousarray(np.broadcast_to(m, (n,)), dtype=np.float32),
        "u": np.ascontiguousarray(np.broadcast_to(u, (n,)), dtype=np.float32),
        "h": np.ascontiguousarray(np.broadcast_to(h, (n,)), dtype=np.float32),
        "alpha_v": np.full(n, alpha_v, dtype=np.float32),
        "alpha_c": np.full(n, alpha_c, dtype=np.float32),
        "box": np.asarray(box, dtype=np.float64),
    }


def _lattice_f64(n, box=(1.0, 1.0, 1.0), origin=(0.0, 0.0, 0.0), shape=None):
    """Cell-centred simple cubic lattice, n per unit length along each axis."""
    shape = shape or (n, n, n)
    dx = 1.0 / n
    ii = [np.arange(s, dtype=np.float64) for s in shape]
    gx, gy, gz = np.meshgrid(*ii, indexing="ij")
    x = np.stack([gx.ravel(), gy.ravel(), gz.ravel()], axis=1)
    return (x + 0.5) * dx + np.asarray(origin)[None, :]


def lattice(n=16, h_factor=1.5 * ETA / H_STAR_LATTICE, vel_sigma=0.0, seed=0, u=1.5):
    """C1: uniform periodic lattice n^3 in the unit box (rho_0 = 1, P = 1 for u = 1.5).

    h0 = h_factor * H_STAR * dx; the default h_factor makes h0 = 1.5*eta*dx so that the
    h iteration has work to do.  vel_sigma > 0 draws seeded Gaussian
    velocities (variant A, exercises div v and curl v).
    """
    dx = 1.0 / n
    x = _lattice_f64(n)
    N = x.shape[0]
    rng = np.random.default_rng(seed)
    v = rng.normal(0.0, vel_sigma, size=(N, 3)) if vel_sigma > 0 else np.zeros((N, 3))
    return _pack(f"lattice{n}", _fixed_point(x, (1, 1, 1)), v, 1.0 / N, u,
                 h_factor * H_STAR_LATTICE * dx, (1.0, 1.0, 1.0))


def jittered_lattice(n=16, jitter=0.1, seed=1, vel_sigma=0.01, h_factor=1.0, u=1.5, u_sigma=0.0):
    """C1 variant B / C4 variant: lattice with uniform jitter +-jitter*dx per axis."""
    dx = 1.0 / n
    rng = np.random.default_rng(seed)
    x = _lattice_f64(n) + rng.uniform(-jitter, jitter, size=(n ** 3, 3)) * dx
    N = x.shape[0]
    v = rng.normal(0.0, vel_sigma, size=(N, 3)) if vel_sigma > 0 else np.zeros((N, 3))
    uu = u * np.exp(u_sigma * rng.standard_normal(N)) if u_sigma > 0 else np.full(N, u)
    return _pack(f"jitter{n}", _fixed_point(x, (1, 1, 1)), v, 1.0 / N, uu,
                 h_factor * H_STAR_LATTICE * dx, (1.0, 1.0, 1.0))


def poisson(N=4096, seed=2, vel_sigma=0.05, u=1.5, u_sigma=0.2, h_factor=1.0):
    """Uniform-random (Poisson) positions in the unit box: uneven neighbour counts."""
    rng = np.random.default_rng(seed)
    x = rng.uniform(0.0, 1.0, size=(N, 3))
    v = rng.normal(0.0, vel_sigma, size=(N, 3))
    uu = u * np.exp(u_sigma * rng.standard_normal(N))
    dx = N ** (-1.0 / 3.0)
    return _pack(f"poisson{N}", _fixed_point(x, (1, 1, 1)), v, 1.0 / N, uu,
                 h_factor * H_STAR_LATTICE * dx, (1.0, 1.0, 1.0))


def blob(N=4096, side=0.4, seed=31, vel_sigma=0.05, u=1.5, u_sigma=0.2, h_factor=1.0):
    """Uniform-random positions in a cube of `side` at the origin of the unit box, the rest
    empty: most cell blocks of the grid hold no particle (the loop kernels' block compaction)."""
    rng = np.random.default_rng(seed)
    x = rng.uniform(0.0, side, size=(N, 3)) + 0.05
    v = rng.normal(0.0, vel_sigma, size=(N, 3))
    uu = u * np.exp(u_sigma * rng.standard_normal(N))
    dx = side * N ** (-1.0 / 3.0)
    return _pack(f"blob{N}", _fixed_point(x, (1, 1, 1)), v, 1.0 / N, uu,
                 h_factor * H_STAR_LATTICE * dx, (1.0, 1.0, 1.0))


def sod(n=64, h_factor=1.0):
    """C2: 3-D Sod shock tube, two n^3 lattices with equal spacing 1/n in [0,2)x[0,1)^2.

    Left x in [0,1): m = 1/n^3 (rho = 1), P = 1 -> u = 1.5.
    Right x in [1,2): m = 0.125/n^3 (rho = 0.125), P = 0.1 -> u = 1.2.
    Periodic box, so there are two interfaces (x = 0 and x = 1).
    """
    dx = 1.0 / n
    left = _lattice_f64(n)
    right = _lattice_f64(n, origin=(1.0, 0.0, 0.0))
    x = np.concatenate([left, right])
    N1 = left.shape[0]
    m = np.concatenate([np.full(N1, 1.0 / N1), np.full(N1, 0.125 / N1)])
    u = np.concatenate([np.full(N1, 1.0 / ((GAMMA_EOS - 1.0) * 1.0)),
                        np.full(N1, 0.1 / ((GAMMA_EOS - 1.0) * 0.125))])
    box = (2.0, 1.0, 1.0)
    return _pack(f"sod{n}", _fixed_point(x, box), np.zeros_like(x), m, u,
                 h_factor * H_STAR_LATTICE * dx, box)


def sedov(n=128, R_s=0.25, P_out=1e-6):
    """C3: Sedov-like blast with strong h contrast.

    Lattice dx = 1/n centred on (1/2,1/2,1/2).  Inside R_s the radial remap
    r -> R_s (r/R_s)^{1/4} maps rho_0 to rho = 4 rho_0 (r/R_s)^9 (mass conserving).
    Inside: v = (r/R_s) r_hat, P = 0.3 + 0.7 (r/R_s)^3, u = P/((gamma-1) rho).
    Outside: v = 0, P = P_out.  h0 = H_STAR * (m/rho)^{1/3} from the prescribed density.
    """
    x = _lattice_f64(n)
    N = x.shape[0]
    c = np.array([0.5, 0.5, 0.5])
    d = x - c[None, :]
    r = np.linalg.norm(d, axis=1)
    inside = r < R_s
    rn = r.copy()
    rn[inside] = R_s * (r[inside] / R_s) ** 0.25
    with np.errstate(invalid="ignore", divide="ignore"):
        rhat = np.where(r[:, None] > 0, d / np.maximum(r, 1e-300)[:, None], 0.0)
    xn = c[None, :] + rhat * rn[:, None]
    rho = np.ones(N)
    rho[inside] = 4.0 * (rn[inside] / R_s) ** 9
    v = np.zeros((N, 3))
    v[inside] = (rn[inside] / R_s)[:, None] * rhat[inside]
    P = np.full(N, P_out)
    P[inside] = 0.3 + 0.7 * (rn[inside] / R_s) ** 3
    u = P / ((GAMMA_EOS - 1.0) * rho)
    m = 1.0 / N
    h = H_STAR_LATTICE * (m / rho) ** (1.0 / 3.0)
    return _pack(f"sedov{n}", _fixed_point(xn, (1, 1, 1)), v, m, u, h, (1.0, 1.0, 1.0))


def gresho_analytic(r):
    """PAPER.md Eq. 27 (v_theta) and Eq. 28 (p) of the Gresho-Chan vortex."""
    r = np.asarray(r, dtype=np.float64)
    vt = np.where(r < 0.2, 5.0 * r, np.where(r < 0.4, 2.0 - 5.0 * r, 0.0))
    with np.errstate(divide="ignore"):
        lr = np.log(np.maximum(r, 1e-300))
    p = np.where(r < 0.2, 5.0 + 12.5 * r * r,
                 np.where(r < 0.4, 9.0 - 4.0 * math.log(0.2) + 12.5 * r * r - 20.0 * r + 4.0 * lr,
                          3.0 + 4.0 * math.log(2.0)))
    return vt, p


def gresho(n=256, jitter=0.0, seed=3, h_factor=1.0):
    """C4: 3-D Gresho-Chan vortex, the paper's own workload.

    Periodic unit box, n^3 lattice, rho_0 = 1, gamma = 5/3, vortex axis parallel to z
    through (1/2, 1/2); v_theta from Eq. 27, p from Eq. 28, u = p/((gamma-1) rho_0).
    """
    dx = 1.0 / n
    x = _lattice_f64(n)
    if jitter > 0:
        rng = np.random.default_rng(seed)
        x = x + rng.uniform(-jitter, jitter, size=x.shape) * dx
    N = x.shape[0]
    dxy = x[:, :2] - 0.5
    r = np.sqrt(dxy[:, 0] ** 2 + dxy[:, 1] ** 2)
    vt, p = gresho_analytic(r)
    v = np.zeros((N, 3))
    with np.errstate(invalid="ignore", divide="ignore"):
        inv = np.where(r > 0, 1.0 / np.maximum(r, 1e-300), 0.0)
    v[:, 0] = -vt * dxy[:, 1] * inv
    v[:, 1] = vt * dxy[:, 0] * inv
    u = p / ((GAMMA_EOS - 1.0) * 1.0)
    return _pack(f"gresho{n}", _fixed_point(x, (1, 1, 1)), v, 1.0 / N, u,
                 h_factor * H_STAR_LATTICE * dx, (1.0, 1.0, 1.0))


def clustered(N=128 ** 3, seed=12345, f_halo=0.6, core=0.05, knn_h=True):
    """C5: cosmological-like clustered box, equal masses, u = 1.

    40 % uniform background + 60 % in NFW halos (c = 10, cored at core*r_s), halo sizes
    ~ M^-1.9 over [64, 0.002 N] particles, centres uniform, member velocities
    N(0, sigma_h^2) with sigma_h ~ M^(1/3).  r_vir from 200x the mean density.
    """
    rng = np.random.default_rng(seed)
    n_halo_total = int(f_halo * N)
    lo, hi = 64, max(65, int(0.002 * N))
    sizes = []
    tot = 0
    a = 1.9
    while tot < n_halo_total:
        # inverse-CDF sample of a power law p(M) ~ M^-a on [lo, hi]
        uu = rng.uniform()
        s = int((lo ** (1 - a) + uu * (hi ** (1 - a) - lo ** (1 - a))) ** (1.0 / (1 - a)))
        s = min(s, n_halo_total - tot)
        sizes.append(s)
        tot += s
    xs = [rng.uniform(0.0, 1.0, size=(N - n_halo_total, 3))]
    vs = [np.zeros((N - n_halo_total, 3))]
    c = 10.0
    for s in sizes:
        centre = rng.uniform(0.0, 1.0, size=3)
        r_vir = (3.0 * s / (4.0 * math.pi * 200.0 * N)) ** (1.0 / 3.0)
        r_s = r_vir / c
        # NFW enclosed-mass inverse sampling on a radial grid, cored at core*r_s
        rg = np.linspace(0.0, r_vir, 2048)
        y = np.maximum(rg, core * r_s) / r_s
        dens = 1.0 / (y * (1.0 + y) ** 2)
        cdf = np.cumsum(dens * rg ** 2)
        cdf /= cdf[-1]
        rr = np.interp(rng.uniform(size=s), cdf, rg)
        dirs = rng.normal(size=(s, 3))
        dirs /= np.linalg.norm(dirs, axis=1)[:, None]
        xs.append(centre[None, :] + dirs * rr[:, None])
        sig = 0.05 * (s / 64.0) ** (1.0 / 3.0)
        vs.append(rng.normal(0.0, sig, size=(s, 3)))
    x = np.concatenate(xs) % 1.0
    v = np.concatenate(vs)
    h = _h_from_knn(x, k=64) if knn_h else np.full(N, H_STAR_LATTICE * N ** (-1.0 / 3.0))
    return _pack(f"clustered{N}", _fixed_point(x, (1, 1, 1)), v, 1.0 / N, 1.0, h, (1.0, 1.0, 1.0))


def _h_from_knn(x, k=64):
    """Initial h from the local number density of the k nearest neighbours (periodic unit box):
    n = k / (4/3 pi d_k^3), h = eta n^(-1/3) (the closure's target, R1).  A starting guess only:
    the h iteration converges to the unique root from any start (R26)."""
    from scipy.spatial import cKDTree

    tree = cKDTree(x, boxsize=1.0)
    d, _ = tree.query(x, k=[k], workers=-1)
    n_loc = k / (4.0 / 3.0 * math.pi * d[:, 0] ** 3)
    return ETA * n_loc ** (-1.0 / 3.0)


def with_duplicates(p, frac=0.05, seed=5, vel_sigma=0.1, u_sigma=0.2):
    """Edge case S:203: append copies of a seeded `frac` of the particles at EXACTLY the same
    fixed-point position (coincident pairs, r_ij = 0 with j != i), with their own seeded
    velocities and internal energies and the original's mass and h."""
    rng = np.random.default_rng(seed)
    n = p["X"].shape[0]
    src = np.sort(rng.choice(n, max(1, int(frac * n)), replace=False))
    k = src.size
    q = dict(p)
    q["name"] = p["name"] + "_dup"
    q["X"] = np.ascontiguousarray(np.concatenate([p["X"], p["X"][src]]), dtype=np.uint32)
    q["v"] = np.ascontiguousarray(np.concatenate([p["v"], p["v"][src] + rng.normal(0.0, vel_sigma, (k, 3))]),
                                  dtype=np.float32)
    u2 = p["u"][src] * np.exp(rng.normal(0.0, u_sigma, k))
    q["u"] = np.ascontiguousarray(np.concatenate([p["u"], u2]), dtype=np.float32)
    for f in ("m", "h", "alpha_v", "alpha_c"):
        q[f] = np.ascontiguousarray(np.concatenate([p[f], p[f][src]]), dtype=np.float32)
    return q


def with_cold(p, frac=0.1, seed=6):
    """Edge case: internal energy u = 0 (so P = c_s = 0) for a seeded `frac` of the particles,
    next to particles with P > 0 (Eq. 20's pressure-weighted alpha_c,ij with one side at P = 0)."""
    rng = np.random.default_rng(seed)
    q = dict(p)
    q["name"] = p["name"] + "_cold"
    u = p["u"].copy()
    u[rng.random(u.size) < frac] = 0.0
    q["u"] = u
    return q


def by_name(name: str, **kw):
    """Named workloads used by tests and bench.py."""
    table = {
        "C1": lambda: lattice(16, **kw),
        "C1v": lambda: lattice(16, vel_sigma=0.01, **kw),
        "C1j": lambda: jittered_lattice(16, **kw),
        "C2": lambda: sod(64, **kw),
        "C3": lambda: sedov(128, **kw),
        "C4": lambda: gresho(256, **kw),
        "C5": lambda: clustered(512 ** 3, **kw),
    }
    return table[name]()
