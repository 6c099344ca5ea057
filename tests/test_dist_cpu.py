"""World-size-2 `gloo` tests on CPU of the N > 1 host logic of bench.py: row-panel partition, per-rank
construction of every problem's H slab (any rank builds its panel bit-identically to the full
matrix's columns), and the max-over-ranks timing reduction. The device path of nranks > 1 runs in
tests/test_gpu_multirank.py (emulated ranks on one GPU)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cf, nprob, q):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import bench

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        n = cf["n"]
        row0, nloc = bench.rank_rows(n, world, rank)
        panels = bench.build_panels(cf, row0, nloc, nprob, lambda: np.empty((nloc, n), dtype=np.complex128))
        for ell, p in enumerate(panels):
            t = torch.from_numpy(np.ascontiguousarray(p).view(np.float64))
            gathered = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(gathered, t)
            if rank == 0:
                full = np.concatenate([g.numpy().view(np.complex128) for g in gathered], axis=0)  # (n x n)^T
                q.put(("panel", ell, full.tobytes()))
        ms = bench.max_over_ranks(10.0 + rank, dist, "cpu")
        if rank == 0:
            q.put(("max", ms))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_row_panels_and_timing_reduction(world):
    import gen as G
    from gen.configs import HNORM

    cf = dict(n=96, nd=80, nev=8, nex=4, cap=20, tol=1e-10, nprob=3, delta=1e-3, seed=31)
    nprob = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cf, nprob, q)) for r in range(world)]
    for p in procs:
        p.start()
    msgs = [q.get(timeout=120) for _ in range(nprob + 1)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # reference: the whole matrix of every problem built on one process
    w = G.wy(cf["n"], cf["nd"], cf["seed"])
    for m in msgs:
        if m[0] == "max":
            assert m[1] == 10.0 + world - 1
            continue
        _, ell, raw = m
        full_t = np.frombuffer(raw, dtype=np.complex128).reshape(cf["n"], cf["n"])  # rows = columns of H
        ref = w.full()
        for l in range(1, ell + 1):
            G.perturb(ref, cf["seed"], l, cf["delta"] * HNORM)
        assert np.array_equal(full_t.T, ref), ell
    with pytest.raises(ValueError):
        sys.path.insert(0, ROOT)
        import bench

        bench.rank_rows(13001, 8, 0)
