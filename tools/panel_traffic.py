"""One filter call of the c2 block on P emulated ranks (push exchange): the K1 launch of a p = 8 rank
(n_loc = 1625 rows, full-height B operand) for an ncu DRAM-traffic capture (profiles/).
usage: python tools/panel_traffic.py [P]"""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import gen as G
    import paper_1404_4161_b200 as chfsi
    from gen.configs import CONFIGS

    P = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    cf = CONFIGS["c2"]
    n, k = cf["n"], cf["nev"] + cf["nex"]
    nloc = n // P
    w = G.wy(n, cf["nd"], cf["seed"])
    l1, a, b = w.lam[0] - 0.05, w.lam[k - 1], 41.0
    c, e = (a + b) / 2, (b - a) / 2
    lg = chfsi.LocalGroup(P)
    errs = []

    def work(r):
        try:
            s = torch.cuda.Stream(device=0)
            with torch.cuda.stream(s):
                Hp = chfsi.colmajor(n, nloc)
                Hp.copy_(torch.from_numpy(w.panel(r * nloc, nloc)))
                Y = chfsi.to_colmajor(G.start_basis(n, k, cf["seed"], r * nloc, nloc))
                ctx = chfsi.Context(0, stream=s, local_group=lg, rank=r)
                ctx.reserve(n, nloc, k)
                ctx.set_exchange(1)
                ctx.filter(Hp, Y, [2] * k, l1, c, e, n=n, row0=r * nloc)
                s.synchronize()
                ctx.close()
        except BaseException as ex:  # noqa: BLE001
            errs.append(ex)

    th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    lg.close()
    if errs:
        raise errs[0]
    print("ok", flush=True)


if __name__ == "__main__":
    main()
