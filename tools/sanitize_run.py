"""Small runs of every kernel path for compute-sanitizer (tools/sanitize.sh): the tile loops on a
jittered lattice, the adaptive grid with wide particles (Sedov), coincident particles, a KDK step
with a rebuild, the pipelined host I/O, and the two-rank slab path over the loopback transport (halo
put: the loop epilogues' peer stores into the other rank's ghost slots)."""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402
from paper_2505_14538_b200 import Context, LoopbackGroup  # noqa: E402
from paper_2505_14538_b200.binding import slab_mask  # noqa: E402


def hydro(p, steps=1, **kw):
    ctx = Context(p, **kw)
    ctx.density()
    ctx.gradient(1e-3)
    dt = ctx.force()
    for _ in range(steps):
        ctx.kick_drift(0.5 * dt, dt)
        ctx.density()
        ctx.gradient(dt)
        dt = ctx.force()
        ctx.kick_drift(0.5 * dt, 0.0)
    ctx.get("a")
    ctx.close()


def two_ranks(p):
    grp = LoopbackGroup(2)
    n = p["X"].shape[0]
    errs = []

    def run(r):
        try:
            mk = slab_mask(p["X"], r, 2)
            q = {k: (v[mk] if hasattr(v, "shape") and v.shape[:1] == (n,) else v) for k, v in p.items()}
            ctx = Context(q, rank=r, nranks=2, n_total=n, loopback=grp)
            ctx.density()
            ctx.gradient(1e-3)
            ctx.force()
            ctx.close()
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=run, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    grp.close()
    if errs:
        raise errs[0]


def pipelined(p):
    """The pipelined host I/O: staged uploads and asynchronous read-backs over two passes."""
    import numpy as np

    ctx = Context(p)
    a = np.zeros((p["X"].shape[0], 3), np.float32)
    ctx.stage_particles(p)
    for k in range(2):
        ctx.set_particles_staged()
        if k == 0:
            ctx.stage_particles(p)
        ctx.density()
        ctx.gradient(1e-3)
        ctx.force()
        ctx.get_async("a", a)
    ctx.synchronize()
    ctx.close()


hydro(W.jittered_lattice(12, seed=3, vel_sigma=0.05, u_sigma=0.2), steps=1)
pipelined(W.jittered_lattice(10, seed=9, vel_sigma=0.05, u_sigma=0.2))
hydro(W.sedov(20))
hydro(W.with_duplicates(W.poisson(1500, seed=5), 0.05))
two_ranks(W.jittered_lattice(16, seed=4, vel_sigma=0.05, u_sigma=0.2))
print("sanitize_run ok")
