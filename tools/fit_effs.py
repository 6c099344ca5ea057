"""Fit the step model's per-variant efficiencies (filter_step.cu kVariantsZ3 / kVariantsReal) to width
tables (tools/width_table.py output): replicates step_cost / choose and searches the eff of every variant
but the reference one, minimising the summed measured time of the model's picks.
usage: fit_effs.py z3|real table.jsonl [table2.jsonl ...]"""
import json
import sys

WOFF = 0.75
# id: (bm, bnc, wnc, threads, eff)
Z3 = {"200": (128, 48, 16, 512, 1.0), "207": (64, 64, 16, 512, 0.88), "208": (128, 32, 8, 512, 0.83)}
REAL = {"104": (128, 64, 16, 512, 0.98), "132": (128, 32, 16, 384, 0.97), "133": (192, 64, 32, 512, 1.0),
        "135": (128, 48, 16, 512, 1.0)}


def cover(w):
    return 1.0 if w >= 12 else 0.85 if w >= 8 else 0.6 if w >= 4 else 0.4


def work_units(ncols, wnc, mma_cols):
    units = -(-ncols // wnc)
    rag = ncols % wnc
    half = (wnc // mma_cols) % 2 == 0 and rag != 0 and 2 * rag <= wnc
    return units - (0.5 if half else 0.0)


def step_cost(V, eff, nrows, ncols, speed, hbm, mma_cols):
    bm, bnc, wnc, threads, _ = V
    tm = -(-nrows // bm); units = -(-ncols // wnc); tn = -(-ncols // bnc); per = -(-units // tn)
    warps = threads // 32; wm = warps // (bnc // wnc)
    cv = cover(per * wm) / cover(warps)
    wu = work_units(ncols, wnc, mma_cols)
    fill = (wu / tn + WOFF) / (per + WOFF)
    cols = tn * per * wnc * (fill if wu != tn * per else 1.0)
    rows = tm * bm
    comp = rows * cols / (eff * cv * speed); mem = rows * hbm * (1 + 0.25 * (tn - 1))
    return max(comp, mem) + 0.1 * comp


def picks(rows, table, effs, speed, hbm):
    tot = 0.0; cnt = {}
    for r in rows:
        best = None
        for v in table:
            if v not in r:
                continue
            c = step_cost(table[v], effs[v], r["n"], r["k"], speed, hbm, 8)
            if best is None or c < bc * 0.999:
                best, bc = v, c
        tot += r[best]; cnt[best] = cnt.get(best, 0) + 1
    return tot, cnt


def main():
    kind = sys.argv[1]
    table, ref, speed, hbm = (Z3, "200", 45.5 / 34.9, 17.7) if kind == "z3" else (REAL, "135", 1.0, 20.0)
    rows = [json.loads(l) for f in sys.argv[2:] for l in open(f) if l.startswith("{")]
    best_possible = sum(min(r[v] for v in table if v in r) for r in rows)
    auto = sum(r["auto"] for r in rows)
    effs = {v: table[v][4] for v in table}
    t0, c0 = picks(rows, table, effs, speed, hbm)
    print("measured auto / best %.4f; model with current effs / best %.4f %s" % (auto / best_possible, t0 / best_possible, c0))
    grid = [round(0.60 + 0.005 * i, 3) for i in range(81)]
    bt = t0
    for _ in range(3):
        for v in table:
            if v == ref:
                continue
            for g in grid:
                e = dict(effs); e[v] = g
                t, _ = picks(rows, table, e, speed, hbm)
                if t < bt - 1e-9:
                    bt, effs = t, e
    t, c = picks(rows, table, effs, speed, hbm)
    print("fitted", effs, "model / best %.4f" % (t / best_possible), c)


main()
