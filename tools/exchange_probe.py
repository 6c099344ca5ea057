"""The p > 1 filter exchange on one GPU: P emulated ranks (a chfsi local group, one host
thread and stream per rank) filter the c2 block (n = 13000, k = 624) on 1-D row panels, with the
per-step exchange done by copy engines (cudaMemcpyAsync, the local group's default), by an SM copy
kernel standing in for NCCL's thread blocks (CHFSI_LG_COLL=kernel), or by the filter epilogue's peer
push; sm_reserve SMs are left out of K1's persistent grid. Prints one JSON line per configuration: the
filter call's device time (max over ranks, CUDA events) and, from the CHFSI_TIMELINE trace of one call,
how much of each exchange interval ran while a K1 launch of the same rank was executing.

usage: python tools/exchange_probe.py P [configs]   configs: comma list of coll:reserve:exchange, e.g.
       copy:0:allgather,kernel:0:allgather,kernel:8:allgather,copy:0:push
"""
import glob
import json
import os
import subprocess
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run_one(P, coll, reserve, exchange, tl_prefix):
    import numpy as np
    import torch

    import gen as G
    import paper_1404_4161_b200 as chfsi
    from gen.configs import CONFIGS

    cf = CONFIGS["c2"]
    n, k = cf["n"], cf["nev"] + cf["nex"]
    nloc = n // P
    w = G.wy(n, cf["nd"], cf["seed"])
    lam = w.lam
    l1, a, b = lam[0] - 0.05, lam[k - 1], 41.0
    c, e = (a + b) / 2, (b - a) / 2
    deg = sorted(int(8 + (12 * j) // k) for j in range(k))  # sorted degrees 8..19: a shrinking active block
    lg = chfsi.LocalGroup(P)
    times = [0.0] * P
    errs = []
    bar = threading.Barrier(P)

    def work(r):
        try:
            s = torch.cuda.Stream(device=0)
            with torch.cuda.stream(s):
                Hp = chfsi.colmajor(n, nloc)
                Hp.copy_(torch.from_numpy(w.panel(r * nloc, nloc)))
                Y0 = chfsi.to_colmajor(G.start_basis(n, k, cf["seed"], r * nloc, nloc))
                ctx = chfsi.Context(0, stream=s, local_group=lg, rank=r)
                ctx.reserve(n, nloc, k)
                ctx.set_pipeline(128, reserve)
                if exchange == "push":
                    ctx.set_exchange(1)
                Y = chfsi.colmajor(nloc, k)
                best = 1e30
                for it in range(4):  # call 1 warms up; the timeline records call 2 (CHFSI_TIMELINE_SKIP=1)
                    Y.copy_(Y0)
                    s.synchronize()
                    bar.wait()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(s)
                    ctx.filter(Hp, Y, deg, l1, c, e, n=n, row0=r * nloc)
                    e1.record(s)
                    s.synchronize()
                    bar.wait()
                    if it:
                        best = min(best, e0.elapsed_time(e1))
                times[r] = best
                ctx.close()
        except BaseException as ex:  # noqa: BLE001
            errs.append(ex)
            bar.abort()

    th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    lg.close()
    if errs:
        raise errs[0]
    flops = 8.0 * n * n * sum(deg)
    out = {"P": P, "coll": coll, "sm_reserve": reserve, "exchange": exchange, "filter_ms": max(times),
           "tflops_zgemm_conv": flops / max(times) / 1e9}
    # overlap from the timeline of the recorded call
    rows = []
    for f in glob.glob(tl_prefix + "_rank*.jsonl"):
        rows += [json.loads(l) for l in open(f)]
    if rows:
        ex_tot = ex_ov = 0.0
        for r in range(P):
            k1 = [(x["t0"], x["t1"]) for x in rows if x["rank"] == r and x["kind"] == "k1"]
            for x in rows:
                if x["rank"] != r or x["kind"] != "exchange":
                    continue
                d = x["t1"] - x["t0"]
                ov = sum(max(0.0, min(x["t1"], b1) - max(x["t0"], a1)) for a1, b1 in k1)
                ex_tot += d
                ex_ov += min(ov, d)
        out.update({"exchange_ms_sum": ex_tot, "exchange_overlapped_frac": ex_ov / ex_tot if ex_tot else None,
                    "timeline": os.path.basename(tl_prefix)})
    print(json.dumps(out), flush=True)


def main():
    P = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    cfgs = (sys.argv[2] if len(sys.argv) > 2 else
            "copy:0:allgather,kernel:0:allgather,kernel:8:allgather,kernel:16:allgather,copy:0:push").split(",")
    if os.environ.get("EXCHANGE_PROBE_CHILD"):
        coll, reserve, exchange = cfgs[0].split(":")
        run_one(P, coll, int(reserve), exchange, os.environ["CHFSI_TIMELINE"])
        return
    outdir = os.environ.get("EXCHANGE_PROBE_OUT", "/tmp")
    for cfg in cfgs:  # one process per configuration: the local group's collective mode is read at creation
        coll, reserve, exchange = cfg.split(":")
        prefix = os.path.join(outdir, f"tl_P{P}_{coll}_r{reserve}_{exchange}")
        for f in glob.glob(prefix + "_rank*.jsonl"):
            os.remove(f)
        env = dict(os.environ, EXCHANGE_PROBE_CHILD="1", CHFSI_TIMELINE=prefix, CHFSI_TIMELINE_SKIP="1",
                   CHFSI_LG_COLL=coll)
        subprocess.run([sys.executable, __file__, str(P), cfg], env=env, check=True)


if __name__ == "__main__":
    main()
