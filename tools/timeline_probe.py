"""GPU timeline of a short c2 sequence (3 problems) under torch.profiler (CUPTI kernel records): kernel
time by kind (K1 vs the rest) and the GPU idle gaps between kernels, grouped by the kernels around them --
where the non-filter time of an eigenproblem goes (the host round trips of the loop).
usage: python tools/timeline_probe.py [config] [nprob]"""
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile

    import gen as G
    import paper_1404_4161_b200 as chfsi
    from gen.configs import CONFIGS, DEG0, HNORM, LANCZOS_STEPS, MAX_LOOPS

    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    nprob = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    cf = CONFIGS[cfg]
    n, nev, nex = cf["n"], cf["nev"], cf["nex"]
    w = G.wy(n, cf["nd"], cf["seed"])
    H = w.full()
    Hs = [chfsi.to_colmajor(H)]
    for ell in range(1, nprob):
        G.perturb(H, cf["seed"], ell, cf["delta"] * HNORM)
        Hs.append(chfsi.to_colmajor(H))
    del H
    ctx = chfsi.Context(0)
    X0 = G.start_basis(n, nev + nex, cf["seed"])

    def run():
        Xd = chfsi.to_colmajor(X0)
        return ctx.solve_sequence(lambda ell: Hs[ell], nprob, Xd, nev, nex, cf["tol"], deg_cap=cf["cap"],
                                  deg0=DEG0, max_loops=MAX_LOOPS, lanczos_steps=LANCZOS_STEPS, seed=cf["seed"])

    run()  # warm-up (workspace, cuBLAS / cuSOLVER handles)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        out = run()
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA" and e.time_range.elapsed_us() > 0]
    ks = sorted(((e.time_range.start, e.time_range.end, e.name) for e in ev), key=lambda x: x[0])
    t0, t1 = ks[0][0], max(e for _, e, _ in ks)
    k1 = sum(e - s for s, e, nm in ks if "filter_step" in nm)
    other = collections.Counter()
    for s, e, nm in ks:
        if "filter_step" not in nm:
            other[nm[:60]] += e - s
    gaps = collections.Counter()
    gapn = collections.Counter()
    end = ks[0][1]
    prev = ks[0][2]
    idle = 0.0
    for s, e, nm in ks[1:]:
        if s > end:
            g = s - end
            idle += g
            key = ("K1" if "filter_step" in prev else prev[:40]) + " -> " + ("K1" if "filter_step" in nm else nm[:40])
            gaps[key] += g
            gapn[key] += 1
        if e > end:
            end, prev = e, nm
    span = t1 - t0
    print(json.dumps({"config": cfg, "nprob": nprob, "loops": [r["loops"] for r in out["reports"]],
                      "span_ms": span / 1e3, "k1_ms": k1 / 1e3, "other_kernels_ms": sum(other.values()) / 1e3,
                      "idle_ms": idle / 1e3}))
    for nm, t in other.most_common(15):
        print(json.dumps({"kernel": nm, "ms": t / 1e3}))
    for key, g in gaps.most_common(25):
        print(json.dumps({"gap": key, "ms": g / 1e3, "count": gapn[key], "avg_us": g / gapn[key]}))
    ctx.close()


if __name__ == "__main__":
    main()
