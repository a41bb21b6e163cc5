"""Debug: adaptive grid / wide particles on a small Sedov (counts vs oracle at fixed h)."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import workloads as W
from parity_util import oracle_hydro
from paper_2505_14538_b200 import Context

p = W.sedov(int(sys.argv[1]) if len(sys.argv) > 1 else 24)
ctx = Context(p, h_max_iter=0, h_tol=1e-6)
print("after create: wide", ctx.counters()["wide_particles"])
st = ctx.density()
print("after density: wide", ctx.counters()["wide_particles"], st)
cnt = ctx.get("count")
o = oracle_hydro(p, fixed_h=True)["density"]
d = cnt.astype(np.int64) - o["count"]
h = p["h"]
bad = np.nonzero(d)[0]
print("mismatch", len(bad), "of", len(d))
if len(bad):
    print("h of bad (rel to median):", np.round(h[bad[:20]] / np.median(h), 3))
    print("diff:", d[bad[:20]])
    print("h quantiles:", np.quantile(h, [0, .5, .9, .99, 1.0]) / np.median(h))
