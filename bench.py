#!/usr/bin/env python
"""Benchmark of the SPH hot path (arXiv 2505.14538) on B200: one KDK hydro step per
"step" = kick/drift -> cell rebuild (device radix sort) -> density + h iteration (+finalize)
-> gradient (+ghost) -> force (+CFL dt) -> closing kick, i.e. every SURVEY §8(a) row.

Metric (BASELINE.json): SPH pair interactions per second (density + gradient + force,
directed pairs) and the time per hydro step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C4] [--impl ours|reference]

Under torchrun (N > 1) the job is ONE simulation decomposed into x-slabs, one per GPU
(include/sph.h "Several ranks"), exchanging ghost planes, migrants and the global h_max / dt
over NCCL every step.  Default --scaling strong: the workload itself (BASELINE.json C4:
"256^3 on 1 B200, then 2/4/8 with halo exchange") split into N slabs.  --scaling weak: N
copies of the workload side by side along x in a box (N Lx, Ly, Lz), one per rank.
The timed region is bracketed by a barrier and torch.cuda.synchronize(), and the max over
ranks is reported.  Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

# Algorithmic FP32 work per pair (FMA = 2 flops), frozen here and in
# density 54 / directed pair, gradient 30 / directed pair, force 95 /
# UNORDERED pair.
FLOPS_DENSITY, FLOPS_GRADIENT, FLOPS_FORCE_UNORDERED = 54.0, 30.0, 95.0
# FP32 peak derived from unit counts and clock: 148 SM x 128 lanes x 2 x 1.965 GHz.
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12
# Algorithmic HBM bytes per particle of one launch (the records a loop
# must read once + the results it writes): density 32 + 36, gradient 48 + 8, force 64 + 20.
BYTES_PER_PARTICLE = {"density": 68.0, "gradient": 56.0, "force": 84.0}


def hbm_peak():
    """Measured copy bandwidth (MEASURED_PEAKS.json, driver-written), else the profiling guide's
    fallback (6.65 TB/s)."""
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None

WORKLOADS = {
    "C4": ("gresho256", lambda: W.gresho(256)),
    "C4j": ("gresho256_jitter0.1", lambda: W.gresho(256, jitter=0.1)),
    "C2": ("sod2x64", lambda: W.sod(64)),
    "C3": ("sedov128", lambda: W.sedov(128)),
    "C5s": ("clustered128", lambda: W.clustered(128 ** 3)),
    "C1": ("lattice16", lambda: W.lattice(16)),
    "G128": ("gresho128", lambda: W.gresho(128)),
    "G64": ("gresho64", lambda: W.gresho(64)),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="C4", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample", default="G64", choices=sorted(WORKLOADS))
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--tile-z", type=int, default=0, help="cells per CTA block along z (0 = auto)")
    ap.add_argument("--skin", type=float, default=None, help="cell_skin (default: the library's)")
    ap.add_argument("--spin", type=int, default=1, choices=[0, 1],
                    help="spin-wait host synchronisation (cuCtxSetFlags CU_CTX_SCHED_SPIN; default 1)")
    ap.add_argument("--balance", action="store_true",
                    help="several ranks: move the slab cuts toward equal particle counts at every rebuild")
    ap.add_argument("--halo-put", type=int, default=-1, choices=[-1, 0, 1],
                    help="X2/X3 halos by peer stores from the loop epilogues (1), NCCL send/recv (0), "
                         "or the library default (-1: send/recv over several NCCL ranks)")
    ap.add_argument("--cpu-baseline-all", default=None, metavar="OUT.json",
                    help="time the oracle on every config family (+ single-thread C1-C3) and exit")
    return ap.parse_args()


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.times = []
        self._stop = threading.Event()
        self._proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self._proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                           "--format=csv,noheader,nounits", "-lms",
                                           os.environ.get("SPH_CLOCKS_MS", "100")],
                                          stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self._proc = None
        return self

    def _read(self):
        for line in self._proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)
                self.times.append(time.monotonic())

    def wait_first(self, timeout=10.0):
        """Block until nvidia-smi's first sample: its start-up (NVML initialisation) holds driver
        locks that stall the host's CUDA calls, so it must be over before the timed region."""
        t = time.monotonic()
        while self._proc and not self.samples and time.monotonic() - t < timeout:
            time.sleep(0.01)

    def window(self, t0, t1):
        """Keep the samples taken in [t0, t1] (the timed region; else the first one after t0)."""
        keep = [s for s, t in zip(self.samples, self.times) if t0 <= t <= t1]
        if not keep:
            keep = [s for s, t in zip(self.samples, self.times) if t >= t0][:1] or self.samples[-1:]
        self.samples = keep

    def __exit__(self, *a):
        if self._proc:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except Exception:
                self._proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        util = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        loaded = [x for x, u in zip(sm, util) if u > 50] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4) if s[3 + k].lower() == "active"})
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        return {"sm_mhz": float(np.median(loaded)) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def rank_workload(key, rank, world, scaling="strong"):
    """Rank's share of the job.  strong: the particles of the workload inside rank's
    x-slab [floor(r 2^32 / N), floor((r+1) 2^32 / N)) (ids = global indices).  weak: copy
    `rank` of the workload, placed at x in [rank Lx, (rank + 1) Lx) of a box (world Lx, Ly,
    Lz): X' = floor((X + rank 2^32) / world), inside rank's slab up to one grid unit (which
    the library migrates)."""
    from paper_2505_14538_b200.binding import slab_mask

    name, gen = WORKLOADS[key]
    p = gen()
    if world == 1:
        return name, p
    n = p["X"].shape[0]
    if scaling == "strong":
        mk = slab_mask(p["X"], rank, world)
        q = {k: (np.ascontiguousarray(v[mk]) if isinstance(v, np.ndarray) and v.shape[:1] == (n,) else v)
             for k, v in p.items()}
        q["id"] = np.flatnonzero(mk).astype(np.int64)
        q["n_total"] = n
        return name, q
    q = dict(p)
    X = p["X"].astype(np.uint64)
    X[:, 0] = (X[:, 0] + (np.uint64(rank) << np.uint64(32))) // np.uint64(world)
    q["X"] = np.ascontiguousarray(X.astype(np.uint32))
    box = np.asarray(p["box"], dtype=np.float64).copy()
    box[0] *= world
    q["box"] = box
    q["n_total"] = n * world
    return f"{name}_x{world}", q


def share_uid(uid, rank, device=None):
    """Broadcast rank 0's 128-byte NCCL id to every rank over torch.distributed."""
    import torch
    import torch.distributed as dist

    t = torch.zeros(128, dtype=torch.uint8, device=device)
    if rank == 0:
        t.copy_(torch.frombuffer(bytearray(uid), dtype=torch.uint8))
    dist.broadcast(t, src=0)
    return bytes(t.cpu().numpy().tobytes())


def dist_init(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        import torch

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    return world, rank, local


def oracle_rate(sample_key, steps=1, threads=None):
    """The fp64 cell-list oracle, as it stands, on a bounded sample: one full hydro pass."""
    import oracle

    name, gen = WORKLOADS[sample_key]
    p = gen()
    if threads:
        oracle.set_threads(threads)
    # (the cell list is the oracle's acceleration structure, pinned against brute force: its side
    # only sets the speed; a typical support radius, not the largest, for strong h contrast)
    o = oracle.Oracle(oracle.Params(), mode="cells", cell_side=2.0 * float(np.percentile(p["h"], 75)))
    times, inter = [], 0
    for _ in range(steps):
        st = oracle.State.from_particles(p)
        t0 = time.perf_counter()
        r = o.hydro(st, dt_ghost=1e-4, first_step=True)
        times.append(time.perf_counter() - t0)
        inter = int(r["density"]["count"].sum()) * 2 + int(r["force"]["count"].sum())
    t = float(np.mean(times))
    npart = p["X"].shape[0]
    return {"value": inter / t, "unit": "interactions/s", "cores": oracle.max_threads(), "kind": "oracle",
            "particle_passes_per_s_per_core": npart / t / oracle.max_threads(),
            "sample": f"{name}: one full hydro pass (density+h, gradient, force) with the fp64 cell-list "
                      f"oracle, {npart} particles, {inter} interactions, {t:.2f} s/pass"}, t, inter, times


# bounded single-thread samples of the C1-C3 families (PAPER.md:506 quotes ~120k particle
# steps/s per core for SWIFT's CPU loops): the oracle on one core
SINGLE_THREAD_SAMPLES = {"C1": ("lattice16", lambda: W.lattice(16)), "C2": ("sod2x32", lambda: W.sod(32)),
                         "C3": ("sedov48", lambda: W.sedov(48))}


def oracle_single_thread(keys=("C1",)):
    import oracle

    nmax = oracle.max_threads()
    out = {}
    try:
        for k in keys:
            name, gen = SINGLE_THREAD_SAMPLES[k]
            WORKLOADS["_st"] = (name, gen)
            r = oracle_rate("_st", threads=1)[0]
            out[k] = {"value": r["value"], "unit": r["unit"], "cores": 1,
                      "particle_passes_per_s": r["particle_passes_per_s_per_core"], "sample": r["sample"]}
    finally:
        WORKLOADS.pop("_st", None)
        oracle.set_threads(nmax)
    return out


def cpu_baseline_all(out_path):
    """--cpu-baseline-all: the oracle on every config family (bounded samples, all host cores)
    and single-threaded on C1-C3, with the CPU model; written to out_path."""
    res = {"cpu_model": cpu_model(), "configs": {}, "single_thread": oracle_single_thread(("C1", "C2", "C3"))}
    # C1, C2 at full size; C4 (Gresho 256^3), C3 (Sedov 128^3) and C5s (clustered 128^3) as bounded
    # samples of their families (the oracle on the full C4 takes minutes)
    WORKLOADS["C3_64"] = ("sedov64", lambda: W.sedov(64))
    WORKLOADS["C5_64"] = ("clustered64", lambda: W.clustered(64 ** 3))
    for key in ("C1", "C2", "G64", "C3_64", "C5_64"):
        r = oracle_rate(key)[0]
        res["configs"][key] = r
        print(key, json.dumps(r), flush=True)
    json.dump(res, open(out_path, "w"), indent=1)
    print(json.dumps(res["single_thread"]), flush=True)


METRIC = "SPH pair interactions/sec (density+gradient+force) and time per hydro step"


def run_reference(args, world, rank):
    if rank != 0:
        return
    for _ in range(args.warmup):
        pass  # the oracle has no warm-up state; warm-up steps would only repeat the same pass
    base, t, inter, times = oracle_rate(args.cpu_sample, steps=args.steps)
    name, _ = WORKLOADS[args.workload]
    # the same metric and workload name as our arm; each step is a bounded sample of that
    # workload family (the oracle on the full workload would take hours), named in `sample`
    line = {"impl": "reference", "metric": METRIC,
            "value": base["value"], "unit": "interactions/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": name, "sample": WORKLOADS[args.cpu_sample][0],
                       "note": "fp64 oracle on host cores; each step one pass over the bounded sample"},
            "cpu_baseline": base,
            "e2e": {"value": base["value"], "unit": "interactions/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def spin_wait(torch):
    """Spin-wait host synchronisation for this process's CUDA context (cuCtxSetFlags
    CU_CTX_SCHED_SPIN): the hydro pass reads a few counters back per step and waits for each; a
    yielding wait lets the host thread be descheduled for up to milliseconds on a busy host."""
    import ctypes

    torch.cuda.synchronize()  # (the primary context is current)
    try:
        cu = ctypes.CDLL("libcuda.so.1")
        cu.cuCtxSetFlags.argtypes = [ctypes.c_uint]
        return cu.cuCtxSetFlags(1) == 0  # CU_CTX_SCHED_SPIN
    except (OSError, AttributeError):
        return False


def run_ours(args, world, rank, local):
    import torch

    from paper_2505_14538_b200 import Context, nccl_unique_id

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if args.spin:
        spin_wait(torch)
    name, p = rank_workload(args.workload, rank, world, args.scaling)
    n = p["X"].shape[0]
    n_total = int(p.get("n_total", n))
    stream = torch.cuda.Stream(device=dev)
    multi = {}
    if world > 1:
        uid = share_uid(nccl_unique_id() if rank == 0 else b"", rank, device=dev)
        multi = dict(rank=rank, nranks=world, n_total=n_total, nccl_uid=uid)
    if args.tile_z:
        multi["tile_cells_z"] = args.tile_z
    if args.skin is not None:
        multi["cell_skin"] = args.skin
    if world > 1 and args.halo_put >= 0:
        multi["halo_put"] = args.halo_put
    if world > 1 and args.balance:
        multi["balance"] = 1
    ctx = Context(p, stream=stream.cuda_stream, device=local, **multi)
    dt = 1e-4

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    def step(log=None):
        nonlocal dt
        ctx.kick_drift(0.5 * dt, dt)
        st = ctx.density()
        ctx.gradient(dt)
        dt_next = ctx.force()
        ctx.kick_drift(0.5 * dt, 0.0)
        c = ctx.counters()
        if log is not None:
            log.append((st, c))
        dt = float(min(dt_next, 2 * dt))
        return st, c

    # clock sampling starts before the warm-up (nvidia-smi's start-up stalls CUDA host calls)
    clk = Clocks(local).__enter__()
    clk.wait_first()
    # first density pass establishes a consistent state (h converged, a computed)
    ctx.density()
    ctx.gradient(dt)
    dt = min(ctx.force(), 1e-3)
    for _ in range(args.warmup):
        step()
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    torch.cuda.synchronize()
    launches0 = ctx.counters()["kernel_launches"]
    ctx.timings(reset=True)
    ctx.set_timing(True)
    log = []
    w0 = time.monotonic()
    t0 = ev()
    for _ in range(args.steps):
        step(log)
    t1 = ev()
    torch.cuda.synchronize()
    w1 = time.monotonic()
    clk.__exit__(None, None, None)
    clk.window(w0, w1)
    launches = ctx.counters()["kernel_launches"] - launches0
    ms = t0.elapsed_time(t1)
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    tm = ctx.timings(reset=True)  # per-kernel device time (CUDA events on the context stream)
    ctx.set_timing(False)
    inter = 0
    pd = pg = pf = ph_iter = 0
    iters = []
    regrids = []
    for st, c in log:
        pd += c["pairs_density"]
        pg += c["pairs_gradient"]
        pf += c["pairs_force"]
        ph_iter += c["pairs_h_iter"]
        iters.append(st["iterations"])
        regrids.append(st["rebuilds"])
    inter = pd + pg + pf
    K = args.steps
    ms_step = ms / K
    inter_all = inter
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([float(inter)], dtype=torch.float64, device=dev)
        dist.all_reduce(t)  # interactions of all ranks (units all ranks processed)
        inter_all = float(t.item())
    value = inter_all / (ms * 1e-3)
    # algorithmic FP32 work of the three loops; density counts every pass
    flops = {"density": FLOPS_DENSITY * ph_iter, "gradient": FLOPS_GRADIENT * pg,
             "force": FLOPS_FORCE_UNORDERED * pf / 2.0}
    kernels = {}
    for name_k, (kms, kn) in tm.items():
        if kn == 0:
            continue
        e = {"ms_per_step": kms / K, "launches_per_step": kn / K, "ms_per_launch": kms / kn, "share": kms / ms}
        if name_k in flops:
            e["tflops"] = flops[name_k] / (kms * 1e-3) / 1e12
        kernels[name_k] = e
    # roofline: the loop kernel (§8 rows a2/a5/a7) with the largest share of the step
    dom = max(("density", "gradient", "force"), key=lambda k: kernels.get(k, {}).get("ms_per_step", 0.0))
    traffic = None
    prof = os.path.join(ROOT, "profiles", "r02", "ncu_summary.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("dram_bytes_per_launch", {}).get(dom)
        except Exception:
            traffic = None
    roof = {"bound": "alu", "kernel": dom, "achieved": kernels[dom]["tflops"], "peak": FP32_PEAK_TFLOPS,
            "unit": "TFLOP/s", "frac": kernels[dom]["tflops"] / FP32_PEAK_TFLOPS, "traffic": traffic,
            "peak_source": "derived: 148 SM x 128 FP32 lanes x 2 x 1.965 GHz (DESIGN.md §7); "
                           "FFMA2 microbenchmark 74.2 TFLOP/s (profiles/r01/ubench2.jsonl)"}
    # the same kernel against the HBM roofline: algorithmic bytes (d.2) and the ncu DRAM bytes
    # of one launch over the live average launch time
    pk, pk_src = hbm_peak()
    t_launch = kernels[dom]["ms_per_launch"] * 1e-3
    alg_bytes = BYTES_PER_PARTICLE[dom] * n_total / max(world, 1)
    roof["hbm"] = {"algorithmic_bytes": alg_bytes, "algorithmic_gbs": alg_bytes / t_launch / 1e9,
                   "dram_gbs": (traffic / t_launch / 1e9) if traffic else None, "peak_gbs": pk,
                   "frac": (traffic / t_launch / 1e9 / pk) if traffic else None, "peak_source": pk_src}

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(ctx, p, torch, dev, stream, max(2, min(K, 10)), world)
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([float(launches)], dtype=torch.float64, device=dev)
        dist.all_reduce(t)
        launches = int(t.item())

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_rate(args.cpu_sample)[0]
        cpu["cpu_model"] = cpu_model()
        cpu["single_thread"] = oracle_single_thread(("C1",))
        cpu["all_configs"] = "profiles/r02/cpu_baseline.json (bench.py --cpu-baseline-all)"
    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value, "unit": "interactions/s", "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": name, "particles": n_total,
                       "parallelism": f"x-slabs{world} (NCCL halo exchange)" if world > 1 else "1gpu",
                       "step": "KDK: kick/drift, rebuild, density+h-iteration, gradient, force+dt, kick",
                       "l2": "inputs larger than L2 (n x ~300 B >> 126 MB)",
                       "interactions_per_step": inter_all / K, "density_passes_mean": float(np.mean(iters)),
                       "density_regrids_mean": float(np.mean(regrids))},
            "gpu_launches": int(launches),
            "kernels": kernels,
            "roofline": roof,
            "clocks": clk.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    ctx.close()


def run_e2e(ctx, p, torch, dev, stream, K, world):
    """Same metric through the public API with host buffers: every step uploads the
    particles from pinned host memory (sph_set_particles), runs density + gradient +
    force, and reads a and du/dt back to pinned host memory (sph_get)."""
    n = p["X"].shape[0]

    def pinned(a):
        t = torch.empty(a.shape, dtype={np.uint32: torch.int32, np.float32: torch.float32}[a.dtype.type],
                        pin_memory=True)
        t.numpy()[...] = a.view(np.int32) if a.dtype == np.uint32 else a
        return t

    host = {k: pinned(p[k]) for k in ("X", "v", "m", "u", "h", "alpha_v", "alpha_c")}
    hin = {k: (host[k].numpy().view(np.uint32) if k == "X" else host[k].numpy()) for k in host}
    cap = n + (n // 4 + 4096 if world > 1 else 0)  # owned count after migration (several ranks)
    a_out = torch.empty((cap, 3), dtype=torch.float32, pin_memory=True)
    du_out = torch.empty((cap,), dtype=torch.float32, pin_memory=True)
    h2d = sum(v.nbytes for v in hin.values())
    d2h = n * 16

    # pipelined through the public API: step k's inputs are uploaded (sph_stage_particles, on
    # the context's host-to-device copy stream) while step k-1 computes, and step k's a, du/dt
    # are read back (sph_get_async, device-to-host copy stream) while step k+1 computes; every
    # step pays its own copies, the timed region runs from the first upload to the last
    # read-back (sph_synchronize)
    def one(last):
        ctx.set_particles_staged()
        if not last:
            ctx.stage_particles(hin)
        ctx.density()
        ctx.gradient(1e-4)
        ctx.force()
        ctx.get_async("a", a_out)
        ctx.get_async("du", du_out)
        return ctx.counters()

    ctx.stage_particles(hin)
    one(True)
    ctx.synchronize()
    torch.cuda.synchronize()
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    t0 = time.perf_counter()
    inter = 0
    ctx.stage_particles(hin)
    for k in range(K):
        c = one(k == K - 1)
        inter += c["pairs_density"] + c["pairs_gradient"] + c["pairs_force"]
    ctx.synchronize()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    # (untimed) where an e2e step's device time goes: two more pipelined steps with the
    # library's per-launch events
    ctx.set_timing(True)
    ctx.timings(reset=True)
    ctx.stage_particles(hin)
    for k in range(2):
        one(k == 1)
    ctx.synchronize()
    phases = {name: round(ms / 2, 3) for name, (ms, cnt) in ctx.timings(reset=True).items() if cnt}
    ctx.set_timing(False)
    if world > 1:
        import torch.distributed as dist

        tm = torch.tensor([dt], dtype=torch.float64, device=dev)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        ts = torch.tensor([float(inter)], dtype=torch.float64, device=dev)
        dist.all_reduce(ts)
        dt, inter = float(tm.item()), float(ts.item())
    return {"value": inter / dt, "unit": "interactions/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": 1e3 * dt / K, "device_ms_per_step": phases,
            "note": "host-timed (perf_counter) over K pipelined steps through the C-ABI: each step uploads its "
                    "inputs from pinned host memory (sph_stage_particles, overlapping the previous step's "
                    "hydro pass) and reads a, du/dt back (sph_get_async, overlapping the next step); "
                    "hydro pass = rebuild + lists + density + gradient + force, no kick/drift"}


def main():
    args = parse()
    if args.cpu_baseline_all:
        cpu_baseline_all(args.cpu_baseline_all)
        return
    world, rank, local = dist_init(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
