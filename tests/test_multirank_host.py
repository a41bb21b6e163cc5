"""Host-side logic of the multi-GPU bench path on CPU (gloo, world_size 2): the weak-scaling
workload split (bench.rank_workload) and the NCCL-id broadcast (bench.share_uid).  The
device exchanges themselves are covered on one GPU by tests/test_gpu_multirank.py through
the loopback transport."""
import os
import socket
import sys

import numpy as np
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    uid = bytes(range(128)) if rank == 0 else b""
    got = bench.share_uid(uid, rank)
    name, p = bench.rank_workload("G64", rank, world, "weak")
    np.save(os.path.join(out, f"X{rank}.npy"), p["X"])
    _, q = bench.rank_workload("G64", rank, world, "strong")
    np.save(os.path.join(out, f"S{rank}.npy"), q["id"])
    with open(os.path.join(out, f"uid{rank}.bin"), "wb") as fh:
        fh.write(got)
    with open(os.path.join(out, f"box{rank}.txt"), "w") as fh:
        fh.write(" ".join(str(float(b)) for b in p["box"]) + " " + name)
    dist.barrier()
    dist.destroy_process_group()


def test_uid_broadcast_and_slab_split(tmp_path):
    from paper_2505_14538_b200.binding import slab_lo

    import bench

    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, start_method="spawn")
    for r in range(world):
        assert open(tmp_path / f"uid{r}.bin", "rb").read() == bytes(range(128))
    _, base = bench.rank_workload("G64", 0, 1)
    n = base["X"].shape[0]
    for r in range(world):
        X = np.load(tmp_path / f"X{r}.npy")
        box = open(tmp_path / f"box{r}.txt").read().split()
        assert float(box[0]) == 2.0 * float(base["box"][0]) and box[-1].endswith("_x2")
        assert X.shape[0] == n
        # y, z untouched; x compressed into rank r's slab (up to one grid unit)
        assert np.array_equal(X[:, 1:], base["X"][:, 1:])
        x = X[:, 0].astype(np.int64)
        lo, hi = slab_lo(r, world), slab_lo(r + 1, world)
        assert x.min() >= lo and x.max() <= hi
        expect = (base["X"][:, 0].astype(np.int64) + (r << 32)) // world
        assert np.array_equal(x, expect)
    # strong scaling: the ranks' slabs partition the workload, each particle in its slab
    ids = np.concatenate([np.load(tmp_path / f"S{r}.npy") for r in range(world)])
    assert np.array_equal(np.sort(ids), np.arange(n))
    for r in range(world):
        x = base["X"][np.load(tmp_path / f"S{r}.npy"), 0].astype(np.int64)
        assert x.min() >= slab_lo(r, world) and x.max() < slab_lo(r + 1, world)
