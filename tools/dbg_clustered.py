"""Try the adaptive grid on a small C5-like clustered box: wide count, passes, time."""
import sys
import time
sys.path.insert(0, ".")
import numpy as np
import workloads as W
from paper_2505_14538_b200 import Context

N = int(sys.argv[1]) if len(sys.argv) > 1 else 64 ** 3
p = W.clustered(N)
h = p["h"]
print("N", N, "h range", float(h.min()), float(np.median(h)), float(h.max()))
t0 = time.time()
ctx = Context(p)
st = ctx.density(allow_unconverged=True)
ctx.gradient(1e-4)
dt = ctx.force()
ctx.synchronize()
print("ok: wide", ctx.counters()["wide_particles"], st, "dt", dt, "wall", round(time.time() - t0, 2))
ctx.set_timing(True)
for _ in range(3):
    ctx.kick_drift(0.5 * dt, dt)
    ctx.density(allow_unconverged=True)
    ctx.gradient(dt)
    dt = ctx.force()
    ctx.kick_drift(0.5 * dt, 0.0)
print({k: round(v[0] / 3, 3) for k, v in ctx.timings().items()}, "wide", ctx.counters()["wide_particles"])
