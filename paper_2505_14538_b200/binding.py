"""Thin ctypes binding of libsph (include/sph.h): argument marshalling only.

Every step of the SPH path runs in the CUDA kernels of libsph.so; there is no CPU
fallback.  If the library is missing this module raises on import of `lib()`.
Arrays may be numpy (host) or torch CUDA tensors (device pointers are passed through).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# (SPH_LIB names another in-tree build of the same library: A/B timing of kernel variants)
LIB_PATH = os.environ.get("SPH_LIB") or os.path.join(_HERE, "libsph.so")

SPH_OK, SPH_ERR_INVALID_ARG, SPH_ERR_CUDA, SPH_ERR_NCCL, SPH_ERR_OOM = 0, 1, 2, 3, 4
SPH_ERR_NOT_CONVERGED, SPH_ERR_H_EXCEEDS_CELL, SPH_ERR_NUMERIC, SPH_ERR_STATE = 5, 6, 7, 8
STATUS_NAMES = {0: "SPH_OK", 1: "SPH_ERR_INVALID_ARG", 2: "SPH_ERR_CUDA", 3: "SPH_ERR_NCCL", 4: "SPH_ERR_OOM",
                5: "SPH_ERR_NOT_CONVERGED", 6: "SPH_ERR_H_EXCEEDS_CELL", 7: "SPH_ERR_NUMERIC", 8: "SPH_ERR_STATE"}

# sph_field: name -> (enum, dtype, components)
FIELDS = {
    "X": (0, np.uint32, 3), "v": (1, np.float32, 3), "m": (2, np.float32, 1), "u": (3, np.float32, 1),
    "h": (4, np.float32, 1), "rho": (5, np.float32, 1), "drho_dh": (6, np.float32, 1), "nhat": (7, np.float32, 1),
    "dn_dh": (8, np.float32, 1), "div": (9, np.float32, 1), "curl": (10, np.float32, 3), "count": (11, np.int32, 1),
    "f": (12, np.float32, 1), "P": (13, np.float32, 1), "c": (14, np.float32, 1), "B": (15, np.float32, 1),
    "v_sig_grad": (16, np.float32, 1), "lap_u": (17, np.float32, 1), "alpha_v": (18, np.float32, 1),
    "alpha_c": (19, np.float32, 1), "div_prev": (20, np.float32, 1), "a": (21, np.float32, 3),
    "du": (22, np.float32, 1), "v_sig": (23, np.float32, 1), "count_force": (24, np.int32, 1),
    "id": (25, np.int64, 1), "iters": (26, np.int32, 1),
}


class SphError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class Config(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_uint32), ("n_total", ctypes.c_int64), ("box", ctypes.c_double * 3),
                ("gamma_k", ctypes.c_float), ("eta", ctypes.c_float), ("h_tol", ctypes.c_float),
                ("h_max_iter", ctypes.c_int32), ("cell_skin", ctypes.c_float), ("gamma_eos", ctypes.c_float),
                ("beta", ctypes.c_float), ("alpha_v_max", ctypes.c_float), ("ell", ctypes.c_float),
                ("alpha_c_min", ctypes.c_float), ("alpha_c_max", ctypes.c_float), ("beta_c", ctypes.c_float),
                ("c_cfl", ctypes.c_float), ("fh_mode", ctypes.c_int32), ("device", ctypes.c_int32),
                ("stream", ctypes.c_void_p), ("rank", ctypes.c_int32), ("nranks", ctypes.c_int32),
                ("tile_cells_z", ctypes.c_int32), ("predict_h", ctypes.c_int32), ("transport", ctypes.c_int32),
                ("nccl_uid", ctypes.c_void_p), ("loopback", ctypes.c_void_p), ("adaptive_h", ctypes.c_int32),
                ("decomp", ctypes.c_int32 * 3), ("halo_put", ctypes.c_int32),
                ("balance", ctypes.c_int32)]

SPH_TRANSPORT_NCCL, SPH_TRANSPORT_LOOPBACK = 0, 1


class ParticlesIn(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("on_device", ctypes.c_int32), ("X", ctypes.c_void_p), ("v", ctypes.c_void_p),
                ("m", ctypes.c_void_p), ("u", ctypes.c_void_p), ("h", ctypes.c_void_p), ("alpha_v", ctypes.c_void_p),
                ("alpha_c", ctypes.c_void_p), ("div_prev", ctypes.c_void_p), ("id", ctypes.c_void_p)]


class DensityStats(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("unconverged", ctypes.c_int32), ("rebuilds", ctypes.c_int32),
                ("max_rel_resid", ctypes.c_float), ("pairs_density", ctypes.c_int64),
                ("pairs_h_iter", ctypes.c_int64)]


PHASES = ["rebuild", "lists", "density", "gradient", "force", "kick_drift", "exchange"]


class Timings(ctypes.Structure):
    _fields_ = [("ms", ctypes.c_double * 8), ("count", ctypes.c_int64 * 8)]


class Counters(ctypes.Structure):
    _fields_ = [("pairs_density", ctypes.c_int64), ("pairs_gradient", ctypes.c_int64),
                ("pairs_force", ctypes.c_int64), ("pairs_h_iter", ctypes.c_int64), ("coincident", ctypes.c_int64),
                ("kernel_launches", ctypes.c_int64), ("wide_particles", ctypes.c_int64)]


EXPORTS = ["sph_abi_version", "sph_config_default", "sph_create", "sph_set_particles", "sph_rebuild_cells",
           "sph_density", "sph_gradient", "sph_force", "sph_kick_drift", "sph_get", "sph_get_counters",
           "sph_synchronize", "sph_last_error", "sph_destroy", "sph_local_count", "sph_nccl_unique_id",
           "sph_loopback_create", "sph_loopback_destroy", "sph_set_timing", "sph_get_timings",
           "sph_stage_particles", "sph_set_particles_staged", "sph_get_async"]

_lib = None


def lib():
    """Load libsph.so (fails loudly if it was not built: no fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2505_14538_b200.build` "
                              "(the SPH path has no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        L.sph_abi_version.restype = ctypes.c_int
        L.sph_config_default.argtypes = [ctypes.POINTER(Config)]
        L.sph_create.argtypes = [ctypes.POINTER(Config), ctypes.POINTER(ParticlesIn), ctypes.POINTER(P)]
        L.sph_set_particles.argtypes = [P, ctypes.POINTER(ParticlesIn)]
        L.sph_rebuild_cells.argtypes = [P]
        L.sph_density.argtypes = [P, ctypes.POINTER(DensityStats)]
        L.sph_gradient.argtypes = [P, ctypes.c_float]
        L.sph_force.argtypes = [P, ctypes.POINTER(ctypes.c_float)]
        L.sph_kick_drift.argtypes = [P, ctypes.c_float, ctypes.c_float]
        L.sph_get.argtypes = [P, ctypes.c_int, P, ctypes.c_int]
        L.sph_stage_particles.argtypes = [P, ctypes.POINTER(ParticlesIn)]
        L.sph_set_particles_staged.argtypes = [P]
        L.sph_get_async.argtypes = [P, ctypes.c_int, P]
        L.sph_get_counters.argtypes = [P, ctypes.POINTER(Counters)]
        L.sph_synchronize.argtypes = [P]
        L.sph_last_error.argtypes = [P]
        L.sph_last_error.restype = ctypes.c_char_p
        L.sph_destroy.argtypes = [P]
        L.sph_set_timing.argtypes = [P, ctypes.c_int]
        L.sph_get_timings.argtypes = [P, ctypes.POINTER(Timings), ctypes.c_int]
        L.sph_local_count.argtypes = [P]
        L.sph_local_count.restype = ctypes.c_int64
        L.sph_nccl_unique_id.argtypes = [P]
        L.sph_loopback_create.argtypes = [ctypes.c_int32, ctypes.POINTER(P)]
        L.sph_loopback_destroy.argtypes = [P]
        for name in EXPORTS:
            if name not in ("sph_abi_version", "sph_config_default", "sph_last_error", "sph_local_count"):
                getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def default_config(box=(1.0, 1.0, 1.0), keep=None, **kw) -> Config:
    c = Config()
    lib().sph_config_default(ctypes.byref(c))
    for a in range(3):
        c.box[a] = float(box[a])
    for k, v in kw.items():
        if k == "nccl_uid":
            buf = ctypes.create_string_buffer(bytes(v), 128)
            if keep is not None:
                keep.append(buf)
            c.nccl_uid = ctypes.cast(buf, ctypes.c_void_p)
        elif k == "loopback":
            c.loopback = v.handle if isinstance(v, LoopbackGroup) else v
            c.transport = SPH_TRANSPORT_LOOPBACK
        else:
            setattr(c, k, v)
    return c


def slab_lo(rank: int, nranks: int) -> int:
    """First fixed-point x of rank's slab: floor(rank 2^32 / nranks) (include/sph.h)."""
    return (rank << 32) // nranks


def slab_mask(X, rank: int, nranks: int):
    """Boolean mask of the particles (fixed-point X [n,3]) in rank's x-slab."""
    x = np.asarray(X)[:, 0].astype(np.int64)
    return (x >= slab_lo(rank, nranks)) & (x < slab_lo(rank + 1, nranks))


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 creates it, the other ranks receive it out of band)."""
    buf = ctypes.create_string_buffer(128)
    st = lib().sph_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p))
    if st != SPH_OK:
        raise SphError(st, "sph_nccl_unique_id failed (libnccl.so.2 not loadable?)")
    return buf.raw


class LoopbackGroup:
    """In-process group of ranks for the loopback transport (tests on one GPU)."""

    def __init__(self, nranks: int):
        h = ctypes.c_void_p()
        st = lib().sph_loopback_create(int(nranks), ctypes.byref(h))
        if st != SPH_OK:
            raise SphError(st, "sph_loopback_create failed")
        self.handle = h.value
        self.nranks = nranks

    def close(self):
        if self.handle:
            lib().sph_loopback_destroy(self.handle)
            self.handle = None


def _is_torch(a):
    return type(a).__module__.startswith("torch")


def _ptr(a, keep, dtype):
    if a is None:
        return None, False
    if _is_torch(a):
        assert a.is_contiguous()
        return a.data_ptr(), a.is_cuda
    arr = np.ascontiguousarray(a, dtype=dtype)
    keep.append(arr)
    return arr.ctypes.data, False


def particles_in(p, keep):
    """Build a sph_particles_in from a dict of numpy arrays or torch tensors."""
    pin = ParticlesIn()
    pin.n = int(p["X"].shape[0])
    dev = []
    for name, dt in (("X", np.uint32), ("v", np.float32), ("m", np.float32), ("u", np.float32), ("h", np.float32),
                     ("alpha_v", np.float32), ("alpha_c", np.float32), ("div_prev", np.float32), ("id", np.int64)):
        ptr, on_dev = _ptr(p.get(name), keep, dt)
        setattr(pin, name, ptr)
        if ptr is not None:
            dev.append(on_dev)
    if any(dev) and not all(dev):
        raise ValueError("particle arrays must be all host or all device")
    pin.on_device = int(bool(dev and dev[0]))
    return pin


class Context:
    """One libsph context (one device).  Methods mirror the C-ABI one to one."""

    def __init__(self, particles, box=None, **cfg):
        self._keep = []
        box = box if box is not None else particles.get("box", (1.0, 1.0, 1.0))
        self._cfg_keep = []
        self.cfg = default_config(box=box, keep=self._cfg_keep, **cfg)
        pin = particles_in(particles, self._keep)
        h = ctypes.c_void_p()
        st = lib().sph_create(ctypes.byref(self.cfg), ctypes.byref(pin), ctypes.byref(h))
        self._keep.clear()
        if st != SPH_OK:
            raise SphError(st, "sph_create failed")
        self.h = h

    @property
    def n(self) -> int:
        """Particles this context owns (all of them on one rank)."""
        return int(lib().sph_local_count(self.h))

    def _check(self, st, what, allow=()):
        if st != SPH_OK and st not in allow:
            raise SphError(st, f"{what}: {lib().sph_last_error(self.h).decode()}")
        return st

    def set_particles(self, particles):
        keep = []
        pin = particles_in(particles, keep)
        self._check(lib().sph_set_particles(self.h, ctypes.byref(pin)), "sph_set_particles")

    def stage_particles(self, particles):
        """sph_stage_particles: asynchronous upload of host arrays (keep them unchanged until
        the copy is done: the next set_particles_staged or synchronize)."""
        self._stage_keep = []
        pin = particles_in(particles, self._stage_keep)
        self._check(lib().sph_stage_particles(self.h, ctypes.byref(pin)), "sph_stage_particles")

    def set_particles_staged(self):
        self._check(lib().sph_set_particles_staged(self.h), "sph_set_particles_staged")

    def get_async(self, field, out):
        """sph_get_async into host memory (a numpy array or a pinned torch tensor of the field's
        shape), written by the next synchronize."""
        ptr = out.data_ptr() if _is_torch(out) else out.ctypes.data
        self._check(lib().sph_get_async(self.h, FIELDS[field][0], ptr), "sph_get_async")
        return out

    def rebuild_cells(self):
        self._check(lib().sph_rebuild_cells(self.h), "sph_rebuild_cells")

    def density(self, allow_unconverged=False):
        s = DensityStats()
        st = lib().sph_density(self.h, ctypes.byref(s))
        self._check(st, "sph_density", allow=(SPH_ERR_NOT_CONVERGED,) if allow_unconverged else ())
        return {f: getattr(s, f) for f, _ in DensityStats._fields_} | {"status": st}

    def gradient(self, dt):
        self._check(lib().sph_gradient(self.h, float(dt)), "sph_gradient")

    def force(self):
        dt = ctypes.c_float()
        self._check(lib().sph_force(self.h, ctypes.byref(dt)), "sph_force")
        return dt.value

    def kick_drift(self, dt_kick, dt_drift):
        self._check(lib().sph_kick_drift(self.h, float(dt_kick), float(dt_drift)), "sph_kick_drift")

    def get(self, field, out=None):
        """Field in the caller's original particle order (several ranks: the owned particles in
        local order, see "id"): numpy (host) or into a torch CUDA tensor."""
        enum, dt, comps = FIELDS[field]
        if out is not None and _is_torch(out):
            self._check(lib().sph_get(self.h, enum, out.data_ptr(), int(out.is_cuda)), "sph_get")
            return out
        arr = np.empty((self.n, comps) if comps > 1 else (self.n,), dtype=dt)
        self._check(lib().sph_get(self.h, enum, arr.ctypes.data, 0), "sph_get")
        return arr

    def counters(self):
        c = Counters()
        self._check(lib().sph_get_counters(self.h, ctypes.byref(c)), "sph_get_counters")
        return {f: getattr(c, f) for f, _ in Counters._fields_}

    def set_timing(self, on=True):
        self._check(lib().sph_set_timing(self.h, int(on)), "sph_set_timing")

    def timings(self, reset=True):
        """{phase: (summed device ms, launches)} since the last reset (synchronises)."""
        t = Timings()
        self._check(lib().sph_get_timings(self.h, ctypes.byref(t), int(reset)), "sph_get_timings")
        return {name: (t.ms[k], t.count[k]) for k, name in enumerate(PHASES)}

    def synchronize(self):
        self._check(lib().sph_synchronize(self.h), "sph_synchronize")

    def close(self):
        if getattr(self, "h", None):
            lib().sph_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
