import sys; sys.path.insert(0, '.')
import workloads as W
from paper_2505_14538_b200 import Context
p = W.gresho(128)
ctx = Context(p)
ctx.set_timing(True)
st = ctx.density(); ctx.gradient(1e-4); dt = ctx.force()
for s in range(6):
    ctx.kick_drift(0.5 * dt, dt)
    st = ctx.density()
    ctx.gradient(dt); dtn = ctx.force(); ctx.kick_drift(0.5 * dt, 0.0); dt = dtn
    print(s, st, ctx.timings())
