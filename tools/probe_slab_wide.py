"""Probe: adaptive grid + wide particles on the slab path (loopback ranks on one GPU).
Runs one hydro pass of Sedov boxes at several sizes / rank counts and compares with the
single-context run at the same (fixed) h."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import workloads as W  # noqa: E402
from multirank_util import run_ranks  # noqa: E402
from parity_util import gpu_hydro  # noqa: E402


def prog(ctx):
    st = ctx.density()
    ctx.gradient(1e-3)
    dt = ctx.force()
    return {"dt": dt, "counters": ctx.counters()}


for n in [int(a) for a in sys.argv[1].split(",")]:
    p = W.sedov(n)
    one = gpu_hydro(p, dt_ghost=1e-3, fixed_h=True)
    for R in [int(a) for a in sys.argv[2].split(",")]:
        t0 = time.time()
        try:
            g, parts = run_ranks(p, R, prog, h_max_iter=0)
        except Exception as e:  # noqa: BLE001
            print(f"n={n} R={R}: ERROR {str(e)[:300]}", flush=True)
            continue
        ce = np.array_equal(g["count"], one["count"])
        cf = np.array_equal(g["count_force"], one["count_force"])
        nbad = int((g["count_force"] != one["count_force"]).sum())
        def rel(k):
            d = np.abs(g[k] - one[k]).reshape(len(g[k]), -1).max(1)
            s = np.abs(one[k]).reshape(len(g[k]), -1).max(1) + 1e-30
            return float((d / s).max())
        aerr = float((np.abs(g["a"] - one["a"]).max(1) / (np.abs(one["a"]).max() + 1e-30)).max())
        wide = [q["counters"]["wide_particles"] for q in parts]
        print(f"n={n} R={R}: counts {ce} force_counts {cf} (bad {nbad}) rho {rel('rho'):.2e} vsig {rel('v_sig'):.2e} "
              f"a/amax {aerr:.2e} du {rel('du'):.2e} wide {wide} single_wide {one['counters']['wide_particles']} "
              f"{time.time() - t0:.1f}s", flush=True)
