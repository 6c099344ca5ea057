"""Multi-GPU check of the NCCL path (run under torchrun, one process per GPU): the row-panel filter and a
c0-shaped solve with the library-owned NCCL communicator, in both exchange modes (pipelined allgather,
peer push over CUDA IPC), compared with the oracle / the exact spectrum. Prints one JSON line per case on
rank 0 and exits non-zero on a mismatch.
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 tools/nccl_check.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import gen as G  # noqa: E402
import oracle as O  # noqa: E402
import paper_1404_4161_b200 as chfsi  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    obj = [chfsi.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ok = True
    n, k = 1000 if world <= 8 else 1024, 37
    n = n - n % world
    nloc = n // world
    w = G.wy(n, int(0.9 * n), 77)
    H = w.full()
    rng = np.random.default_rng(5)
    deg = sorted(rng.integers(1, 21, k).tolist())
    Y0 = rng.standard_normal((n, k)) + 1j * rng.standard_normal((n, k))
    l1, a, b = w.lam[0] - 0.05, w.lam[k], 45.0
    c, e = (a + b) / 2, (b - a) / 2
    Yo, _ = O.chebyshev_filter(H, Y0, deg, l1, c, e) if rank == 0 else (None, None)
    for mode in (0, 1):
        ctx = chfsi.Context(local, nccl_id=obj[0], rank=rank, nranks=world)
        ctx.set_pipeline(8)
        ctx.reserve(n, nloc, 64)
        if mode == 1:
            ctx.set_exchange(1)
        Hp = chfsi.to_colmajor(np.asfortranarray(H[:, rank * nloc:(rank + 1) * nloc]))
        Yd = chfsi.to_colmajor(Y0[rank * nloc:(rank + 1) * nloc])
        ctx.filter(Hp, Yd, deg, l1, c, e, n=n, row0=rank * nloc)
        parts = [torch.empty_like(Yd.t().contiguous()) for _ in range(world)]
        dist.all_gather(parts, Yd.t().contiguous())
        if rank == 0:
            Y = np.concatenate([p.t().cpu().numpy() for p in parts], axis=0)
            err = float((np.linalg.norm(Y - Yo, axis=0) / np.linalg.norm(Yo, axis=0)).max())
            ok &= err <= 1e-11
            print(json.dumps({"case": "filter", "exchange": mode, "world": world, "n": n, "max_rel_err": err}),
                  flush=True)
        nev, nex = 24, 8
        X = chfsi.to_colmajor(G.start_basis(n, nev + nex, 9, rank * nloc, nloc))
        out = ctx.solve_sequence(lambda ell: Hp, 1, X, nev, nex, 1e-10, deg_cap=20, seed=9, n=n, row0=rank * nloc)
        err = float(np.max(np.abs(out["lam"][0] - w.lam[:nev]) / np.abs(w.lam[:nev])))
        ok &= out["status"] == 0 and err <= 1e-10
        if rank == 0:
            print(json.dumps({"case": "solve", "exchange": mode, "world": world, "status": out["status"],
                              "max_rel_eig_err": err}), flush=True)
        if mode == 0:  # NEXT-1 on row panels: reduce, back-transform (collectives over the same communicator)
            A, B, _ = G.generalized_pair(w, 2)
            cols = slice(rank * nloc, (rank + 1) * nloc)
            Ap = chfsi.to_colmajor(np.asfortranarray(A[:, cols]))
            Bp = chfsi.to_colmajor(np.asfortranarray(B[:, cols]))
            Ld = chfsi.colmajor(n, n)
            ctx.reduce_generalized_panel(Ap, Bp, Ld, n=n, row0=rank * nloc)
            At = Ap.t().contiguous()
            parts = [torch.empty_like(At) for _ in range(world)]
            dist.all_gather(parts, At)
            if rank == 0:
                Hg = np.concatenate([q.t().cpu().numpy() for q in parts], axis=1)
                Ho, _ = O.reduce_generalized(A, B)
                herr = float(np.abs(Hg - Ho).max())
                herm = bool(np.array_equal(Hg, Hg.conj().T))
                ok &= herr <= 1e-11 and herm
                print(json.dumps({"case": "reduce_generalized_panel", "world": world, "max_abs_err": herr,
                                  "exactly_hermitian": herm}), flush=True)
        ctx.close()
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
