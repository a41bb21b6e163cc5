"""fp64 CPU oracle of the SPH hot path (density + h iteration, finalize, gradient,
gradient ghost, force, CFL dt, kick/drift).  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this package.  It shares no code with paper_2505_14538_b200 (the CUDA path)
and never imports it; both sides read inputs from `workloads` only.

The arithmetic lives in oracle.c (plain C, fp64, -ffp-contract=off); this module only
builds it with gcc and marshals numpy arrays through ctypes.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (fp64, OpenMP, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
               "-fno-fast-math", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


class Params(ctypes.Structure):
    """Physics parameters; defaults per DESIGN.md §3 readings."""
    _fields_ = [("gamma_k", ctypes.c_double), ("eta", ctypes.c_double), ("h_tol", ctypes.c_double),
                ("h_max_iter", ctypes.c_int32), ("gamma_eos", ctypes.c_double), ("beta", ctypes.c_double),
                ("alpha_v_max", ctypes.c_double), ("ell", ctypes.c_double), ("alpha_c_min", ctypes.c_double),
                ("alpha_c_max", ctypes.c_double), ("beta_c", ctypes.c_double), ("c_cfl", ctypes.c_double),
                ("fh_mode", ctypes.c_int32)]

    def __init__(self, **kw):
        d = dict(gamma_k=2.0, eta=1.2348, h_tol=1e-4, h_max_iter=32, gamma_eos=5.0 / 3.0, beta=3.0,
                 alpha_v_max=2.0, ell=0.05, alpha_c_min=0.0, alpha_c_max=1.0, beta_c=1.0, c_cfl=0.1,
                 fh_mode=0)
        d.update(kw)
        super().__init__(**d)


_P = ctypes.c_void_p
_D = ctypes.POINTER(ctypes.c_double)
_I64 = ctypes.POINTER(ctypes.c_int64)
_I32 = ctypes.POINTER(ctypes.c_int32)
_U8 = ctypes.POINTER(ctypes.c_uint8)
_U32 = ctypes.POINTER(ctypes.c_uint32)


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.orc_w.restype = ctypes.c_double
        L.orc_w.argtypes = [ctypes.c_double]
        L.orc_dw.restype = ctypes.c_double
        L.orc_dw.argtypes = [ctypes.c_double]
        L.orc_kernel.argtypes = [ctypes.c_double, ctypes.c_double, _D, _D, _D]
        L.orc_geom_create.restype = _P
        L.orc_geom_create.argtypes = [ctypes.c_int64, _D, _U32, ctypes.c_int, ctypes.c_double]
        L.orc_geom_destroy.argtypes = [_P]
        L.orc_neighbours.restype = ctypes.c_int64
        L.orc_neighbours.argtypes = [_P, ctypes.c_int64, ctypes.c_double, _I64, ctypes.c_int64]
        L.orc_density.restype = ctypes.c_int
        L.orc_density.argtypes = [_P, ctypes.POINTER(Params), _I64, ctypes.c_int64, _D, _D, _D, _D, _I64, _I32, _I64,
                                  _D, _D]
        L.orc_finalize.argtypes = [ctypes.POINTER(Params), _I64, ctypes.c_int64, _D, _D, _D, _D]
        L.orc_gradient.restype = ctypes.c_int
        L.orc_gradient.argtypes = [_P, ctypes.POINTER(Params), _I64, ctypes.c_int64, _D, _D, _D, _D, _D, _D, _U8, _D,
                                   _D, _D]
        L.orc_gradient_ghost.argtypes = [ctypes.POINTER(Params), _I64, ctypes.c_int64, ctypes.c_double, ctypes.c_int,
                                         _D, _D, _D, _D, _D, _D]
        L.orc_force.restype = ctypes.c_int
        L.orc_force.argtypes = [_P, ctypes.POINTER(Params), _I64, ctypes.c_int64, _D, _D, _D, _D, _U8,
                                ctypes.c_double, _D]
        L.orc_dt.restype = ctypes.c_double
        L.orc_dt.argtypes = [ctypes.POINTER(Params), _I64, ctypes.c_int64, _D, _D]
        L.orc_kick_drift.argtypes = [ctypes.c_int64, _D, ctypes.c_double, ctypes.c_double, _D, _D, _D, _D, _U32]
        L.orc_closure.argtypes = [_P, _U8, ctypes.c_double, _U8]
        L.orc_max_threads.restype = ctypes.c_int
        L.orc_set_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def _ptr(a, t):
    return a.ctypes.data_as(t)


def kernel(r, h):
    """(W, dW/dr, dW/dh) of the M4 kernel in fp64."""
    W, dr, dh = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    lib().orc_kernel(float(r), float(h), ctypes.byref(W), ctypes.byref(dr), ctypes.byref(dh))
    return W.value, dr.value, dh.value


def w(q):
    return lib().orc_w(float(q))


def dw(q):
    return lib().orc_dw(float(q))


def max_threads():
    return lib().orc_max_threads()


def set_threads(n):
    lib().orc_set_threads(int(n))


class Geometry:
    """Neighbour enumeration over a particle set: brute force (the definition) or a
    cell list with cell side >= min_side (pinned against brute force)."""

    def __init__(self, X, box, use_cells=False, min_side=None):
        self.X = np.ascontiguousarray(X, dtype=np.uint32)
        self.box = np.ascontiguousarray(box, dtype=np.float64)
        self.n = self.X.shape[0]
        if use_cells and min_side is None:
            raise ValueError("cell list needs min_side")
        self.h = lib().orc_geom_create(self.n, _ptr(self.box, _D), _ptr(self.X, _U32), int(bool(use_cells)),
                                       float(min_side or 1.0))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_geom_destroy(self.h)
            self.h = None

    def neighbours(self, i, R):
        out = np.empty(min(self.n, 1 << 20), dtype=np.int64)
        k = lib().orc_neighbours(self.h, int(i), float(R), _ptr(out, _I64), out.size)
        if k < 0:
            raise RuntimeError("neighbour buffer overflow")
        return out[:k].copy()

    def closure(self, mask, R):
        mask = np.ascontiguousarray(mask, dtype=np.uint8)
        out = np.empty_like(mask)
        lib().orc_closure(self.h, _ptr(mask, _U8), float(R), _ptr(out, _U8))
        return out.astype(bool)


def _idx(n, idx):
    if idx is None:
        return np.arange(n, dtype=np.int64)
    return np.ascontiguousarray(idx, dtype=np.int64)


@dataclass
class State:
    """fp64 working copy of a particle set (oracle side)."""
    X: np.ndarray
    box: np.ndarray
    v: np.ndarray
    m: np.ndarray
    u: np.ndarray
    h: np.ndarray
    alpha_v: np.ndarray
    alpha_c: np.ndarray
    div_prev: np.ndarray = field(default=None)

    @classmethod
    def from_particles(cls, p):
        n = p["X"].shape[0]
        return cls(X=p["X"].copy(), box=np.asarray(p["box"], dtype=np.float64),
                   v=p["v"].astype(np.float64).reshape(n, 3).copy(), m=p["m"].astype(np.float64),
                   u=p["u"].astype(np.float64), h=p["h"].astype(np.float64), alpha_v=p["alpha_v"].astype(np.float64),
                   alpha_c=p["alpha_c"].astype(np.float64), div_prev=np.zeros(n))


class Oracle:
    """Stage-by-stage oracle over one particle set.  mode = 'brute' (O(N^2) definition)
    or 'cells' (O(N) cell list, pinned against brute)."""

    def __init__(self, params: Params | None = None, mode="brute", cell_side=None):
        self.params = params or Params()
        self.mode = mode
        self.cell_side = cell_side

    def geometry(self, st: State, h_max=None):
        if self.mode == "brute":
            return Geometry(st.X, st.box, use_cells=False)
        side = self.cell_side or (self.params.gamma_k * float(h_max if h_max is not None else st.h.max()))
        return Geometry(st.X, st.box, use_cells=True, min_side=side)

    # -- density loop + h iteration --------------------------------------
    def density(self, st: State, idx=None, geom=None, fixed_h=False):
        n = st.X.shape[0]
        ii = _idx(n, idx)
        g = geom or self.geometry(st)
        prm = Params(**{f: getattr(self.params, f) for f, _ in Params._fields_})
        if fixed_h:
            prm.h_max_iter = 0
        h = st.h.copy()
        dens = np.full((n, 8), np.nan)
        count = np.full(n, -1, dtype=np.int64)
        iters = np.full(n, -2, dtype=np.int32)
        coinc = ctypes.c_int64(0)
        sdv = np.full(n, np.nan)
        sdt = np.full(n, np.nan)
        status = lib().orc_density(g.h, ctypes.byref(prm), _ptr(ii, _I64), ii.size, _ptr(h, _D),
                                   _ptr(np.ascontiguousarray(st.v), _D), _ptr(st.m, _D), _ptr(dens, _D),
                                   _ptr(count, _I64), _ptr(iters, _I32), ctypes.byref(coinc), _ptr(sdv, _D),
                                   _ptr(sdt, _D))
        return dict(status=status, h=h, rho=dens[:, 0], drho_dh=dens[:, 1], nhat=dens[:, 2], dn_dh=dens[:, 3],
                    div=dens[:, 4], curl=dens[:, 5:8], count=count, iters=iters, coincident=coinc.value,
                    scale_dv=sdv, scale_dv_tail=sdt, _dens=dens, idx=ii)

    def finalize(self, st: State, d, idx=None):
        n = st.X.shape[0]
        ii = _idx(n, idx)
        fin = np.full((n, 4), np.nan)
        lib().orc_finalize(ctypes.byref(self.params), _ptr(ii, _I64), ii.size, _ptr(d["h"], _D), _ptr(st.u, _D),
                           _ptr(d["_dens"], _D), _ptr(fin, _D))
        return dict(f=fin[:, 0], P=fin[:, 1], c=fin[:, 2], B=fin[:, 3])

    def gradient(self, st: State, h, rho, c, idx=None, valid=None, geom=None):
        n = st.X.shape[0]
        ii = _idx(n, idx)
        g = geom or self.geometry(st)
        grad = np.full((n, 2), np.nan)
        slap = np.full(n, np.nan)
        stl = np.full(n, np.nan)
        vm = None if valid is None else np.ascontiguousarray(valid, dtype=np.uint8)
        status = lib().orc_gradient(g.h, ctypes.byref(self.params), _ptr(ii, _I64), ii.size, _ptr(h, _D),
                                    _ptr(np.ascontiguousarray(st.v), _D), _ptr(st.m, _D), _ptr(st.u, _D),
                                    _ptr(np.ascontiguousarray(rho), _D), _ptr(np.ascontiguousarray(c), _D),
                                    None if vm is None else _ptr(vm, _U8), _ptr(grad, _D), _ptr(slap, _D),
                                    _ptr(stl, _D))
        return dict(status=status, v_sig=grad[:, 0], lap_u=grad[:, 1], scale_lap=slap, scale_lap_tail=stl,
                    _grad=grad)

    def gradient_ghost(self, st: State, h, c, div, grad, dt, first_step, idx=None):
        n = st.X.shape[0]
        ii = _idx(n, idx)
        state = np.ascontiguousarray(np.stack([st.alpha_v, st.alpha_c, st.div_prev], axis=1))
        lib().orc_gradient_ghost(ctypes.byref(self.params), _ptr(ii, _I64), ii.size, float(dt), int(bool(first_step)),
                                 _ptr(h, _D), _ptr(st.u, _D), _ptr(np.ascontiguousarray(c), _D),
                                 _ptr(np.ascontiguousarray(div), _D), _ptr(grad["_grad"], _D), _ptr(state, _D))
        return dict(alpha_v=state[:, 0].copy(), alpha_c=state[:, 1].copy(), div_prev=state[:, 2].copy())

    def force(self, st: State, h, f, P, c, B, rho, alpha_v, alpha_c, idx=None, valid=None, geom=None):
        n = st.X.shape[0]
        ii = _idx(n, idx)
        g = geom or self.geometry(st)
        pp = np.ascontiguousarray(np.stack([f, P, c, B, rho, st.u, alpha_v, alpha_c], axis=1))
        out = np.full((n, 11), np.nan)
        vm = None if valid is None else np.ascontiguousarray(valid, dtype=np.uint8)
        hm = float(np.nanmax(h if valid is None else np.where(valid, h, np.nan)))
        status = lib().orc_force(g.h, ctypes.byref(self.params), _ptr(ii, _I64), ii.size, _ptr(h, _D),
                                 _ptr(np.ascontiguousarray(st.v), _D), _ptr(st.m, _D), _ptr(pp, _D),
                                 None if vm is None else _ptr(vm, _U8), hm, _ptr(out, _D))
        return dict(status=status, a=out[:, 0:3], du=out[:, 3], v_sig=out[:, 4], scale_a=out[:, 5],
                    scale_u=out[:, 6], count=out[:, 7], scale_cond=out[:, 8],
                    scale_tail=out[:, 9], scale_v=out[:, 10])

    def dt(self, h, v_sig, idx=None):
        ii = _idx(h.shape[0], idx)
        return lib().orc_dt(ctypes.byref(self.params), _ptr(ii, _I64), ii.size, _ptr(np.ascontiguousarray(h), _D),
                            _ptr(np.ascontiguousarray(v_sig), _D))

    def kick_drift(self, st: State, a, du, dt_k, dt_d):
        n = st.X.shape[0]
        a = np.ascontiguousarray(a, dtype=np.float64)
        du = np.ascontiguousarray(du, dtype=np.float64)
        lib().orc_kick_drift(n, _ptr(st.box, _D), float(dt_k), float(dt_d), _ptr(a, _D), _ptr(du, _D),
                             _ptr(st.v, _D), _ptr(st.u, _D), _ptr(st.X, _U32))

    # -- one hydro pass: density (+h), finalize, gradient, ghost, force, dt -------
    def hydro(self, st: State, dt_ghost=0.0, first_step=True, fixed_h=False, sample=None, hop_radius=None):
        """Full hydro pass.  sample=None computes every particle; otherwise the outputs
        are exact for the sampled indices (their 2-hop neighbourhoods are computed
        upstream; hop_radius bounds the support radius of the final h, default
        1.5 gamma_k max(h0))."""
        n = st.X.shape[0]
        g = self.geometry(st, h_max=st.h.max() * (1.0 if fixed_h else 2.0))
        if sample is None:
            s0 = s1 = s2 = None
            valid = None
        else:
            R = hop_radius or 1.5 * self.params.gamma_k * float(st.h.max())
            m0 = np.zeros(n, dtype=np.uint8)
            m0[np.asarray(sample)] = 1
            m1 = g.closure(m0, R)
            # (a 1-hop set covering most of the box: computing everything is the cheaper superset)
            m2 = g.closure(m1, R) if m1.sum() < n // 2 else np.ones(n, dtype=bool)
            s0, s1, s2 = np.flatnonzero(m0), np.flatnonzero(m1), np.flatnonzero(m2)
            valid = m2
        d = self.density(st, idx=s2, geom=g, fixed_h=fixed_h)
        fin = self.finalize(st, d, idx=s2)
        gr = self.gradient(st, d["h"], d["rho"], fin["c"], idx=s1, valid=valid, geom=g)
        gh = self.gradient_ghost(st, d["h"], fin["c"], d["div"], gr, dt_ghost, first_step, idx=s1)
        v1 = None if sample is None else np.zeros(n, dtype=bool)
        if v1 is not None:
            v1[s1] = True
        fo = self.force(st, d["h"], fin["f"], fin["P"], fin["c"], fin["B"], d["rho"], gh["alpha_v"], gh["alpha_c"],
                        idx=s0, valid=v1, geom=g)
        dt = self.dt(d["h"], fo["v_sig"], idx=s0)
        return dict(density=d, finalize=fin, gradient=gr, ghost=gh, force=fo, dt=dt, sets=(s0, s1, s2))
