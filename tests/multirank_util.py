"""Run the multi-rank (slab-decomposed) path on ONE GPU: R contexts of a loopback group,
one host thread each (include/sph.h "Several ranks").  The per-rank owned
fields are gathered back into the input order by particle id."""
from __future__ import annotations

import threading

import numpy as np

FIELDS = ("h", "rho", "drho_dh", "nhat", "dn_dh", "div", "curl", "count", "f", "P", "c", "B", "v_sig_grad", "lap_u",
          "alpha_v", "alpha_c", "a", "du", "v_sig", "count_force", "X", "v", "u")


def split(p, R):
    """Per-rank particle dicts (the rank's x-slab) with ids = input index."""
    from paper_2505_14538_b200 import slab_mask

    n = p["X"].shape[0]
    ids = np.arange(n, dtype=np.int64)
    out = []
    for r in range(R):
        mk = slab_mask(p["X"], r, R)
        sub = {k: (np.ascontiguousarray(v[mk]) if isinstance(v, np.ndarray) and v.shape[:1] == (n,) else v)
               for k, v in p.items()}
        sub["id"] = ids[mk]
        out.append(sub)
    return out


def gather(parts, n):
    """Owned-field dicts of the ranks -> full arrays in input order (each id exactly once)."""
    ids = np.concatenate([q["id"] for q in parts])
    assert ids.size == n and np.array_equal(np.sort(ids), np.arange(n)), "ids lost or duplicated across ranks"
    full = {}
    for k in parts[0]:
        if k == "id" or not isinstance(parts[0][k], np.ndarray) or parts[0][k].ndim == 0:
            continue
        cat = np.concatenate([q[k] for q in parts])
        arr = np.empty_like(cat)
        arr[ids] = cat
        full[k] = arr
    return full


def run_ranks(p, R, program, timeout=300.0, **cfg):
    """program(ctx) -> dict of extra results; runs on every rank of a loopback group."""
    from paper_2505_14538_b200 import Context, LoopbackGroup

    n = p["X"].shape[0]
    group = LoopbackGroup(R)
    subs = split(p, R)
    res = [None] * R
    errs = []

    def worker(r):
        try:
            ctx = Context(subs[r], rank=r, nranks=R, n_total=n, loopback=group, **cfg)
            extra = program(ctx) or {}
            out = {k: ctx.get(k) for k in FIELDS}
            out["id"] = ctx.get("id")
            out["n_local"] = ctx.n
            out.update(extra)
            res[r] = out
            ctx.close()
        except Exception as e:  # pragma: no cover - reported below
            errs.append((r, e))

    th = [threading.Thread(target=worker, args=(r,), daemon=True) for r in range(R)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout)
    if any(t.is_alive() for t in th):
        raise RuntimeError(f"multi-rank run hung (errors so far: {errs})")
    group.close()
    if errs:
        raise errs[0][1]
    return gather(res, n), res
