import sys; sys.path.insert(0, "tests")
import numpy as np, workloads as W
from multirank_util import run_ranks
p = W.jittered_lattice(40, seed=64, vel_sigma=0.2, u_sigma=0.4)
def prog(ctx):
    st = ctx.density(); print("density ok", st, flush=True)
    ctx.gradient(1e-3); ctx.force()
run_ranks(p, 3, prog, h_tol=1e-5)
