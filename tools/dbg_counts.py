"""Debug: GPU neighbour counts vs oracle at fixed h on small cases (prints mismatch stats)."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import workloads as W
from parity_util import gpu_hydro, oracle_hydro

cases = {
    "lattice16": lambda: W.lattice(16, h_factor=1.0, vel_sigma=0.01, seed=21),
    "lattice16x1.5": lambda: W.lattice(16, h_factor=1.5, vel_sigma=0.01, seed=21),
    "jitter16": lambda: W.jittered_lattice(16, seed=22, vel_sigma=0.05, u_sigma=0.3),
    "poisson4096": lambda: W.poisson(4096, seed=23, vel_sigma=0.1, u_sigma=0.3),
    "gresho24": lambda: W.gresho(24),
}
for name, f in cases.items():
    p = f()
    try:
        g = gpu_hydro(p, fixed_h=True)
    except Exception as e:
        print(name, "GPU error", e)
        continue
    o = oracle_hydro(p, fixed_h=True)["density"]
    d = g["count"].astype(np.int64) - o["count"].astype(np.int64)
    cf = g["count_force"]
    print(f"{name}: n={len(d)} mismatched={np.count_nonzero(d)} min={d.min()} max={d.max()} "
          f"gpu_mean={g['count'].mean():.2f} oracle_mean={o['count'].mean():.2f} rho_relerr={np.max(np.abs(g['rho']/o['rho']-1)):.2e} "
          f"countf_mean={cf.mean():.2f}")
    if np.count_nonzero(d):
        idx = np.nonzero(d)[0][:10]
        print("   first bad:", idx, d[idx])
