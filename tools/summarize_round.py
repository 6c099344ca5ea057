"""Summaries of a tools/profile_round.sh run for profiles/: the full ncu capture of the c2 full-width K1
launch (key metrics + the source page's warp-stall samples by instruction) and the kernel-time shares of
the short bench's ncu launch list. usage: python tools/summarize_round.py <tag>  (reads gpurun_out/<tag>_*)"""
import collections
import csv
import gzip
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ['dram__bytes_read.sum', 'dram__bytes_write.sum', 'gpc__cycles_elapsed.max', 'gpu__time_duration.sum',
        'launch__block_size', 'launch__grid_size', 'launch__registers_per_thread', 'lts__t_sector_hit_rate.pct',
        'sm__cycles_active.avg', 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed',
        'sm__pipe_tensor_cycles_active.max.pct_of_peak_sustained_elapsed',
        'sm__pipe_tensor_cycles_active.min.pct_of_peak_sustained_elapsed',
        'sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active']


def ncu_csv(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"] + (["--print-source", "sass"] if page == "source" else []),
                         capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


def main():
    tag = sys.argv[1]
    g = os.path.join(ROOT, "gpurun_out")
    rep = os.path.join(g, f"{tag}_k1.ncu-rep")
    rows = ncu_csv(rep, "raw")
    h, u, v = rows[0], rows[1], rows[2]
    lines = [f"# {tag}: ncu --set full --clock-control none of the full-width c2 K1 launch (n = 13000, k_a = 624, 3M z200 128x48, "
             "12 consumer warps + a producer warpgroup = 512 threads, setmaxnreg 24/160, persistent grid 148)",
             "# command: ncu --set full --clock-control none --import-source on -k regex:filter_step -s 4 -c 1 "
             "python tools/filter_perf.py 13000 624 4 auto3"]
    for k in KEYS:
        i = h.index(k)
        lines.append(f"{k} [{u[i]}] {v[i]}")
    src = ncu_csv(rep, "source")[1:]
    hh, body = src[0], src[1:]
    iS, iW = hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)")
    tot, by = 0, collections.Counter()
    for r in body:
        try:
            s = int(r[iW])
        except (ValueError, IndexError):
            continue
        tot += s
        ops = [o for o in r[iS].split() if not o.startswith("@")]
        by[ops[0].split(".")[0] if ops else "?"] += s
    lines.append(f"# source page: {tot} warp stall samples; by instruction: " +
                 ", ".join(f"{k} {100 * c / tot:.1f}%" for k, c in by.most_common(8)))
    lines.append("# launch__registers_per_thread is the launch allocation (128); setmaxnreg moves producers to 24 and "
                 "consumers to 160 at run time")
    lines.append("# before the producer warpgroup (r02_ncu_k1_z3_prepw.txt): tensor pipe 94.53 % of peak elapsed, 18.11 ms")
    open(os.path.join(ROOT, "profiles", "r02_ncu_k1_z3.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    # launch shares
    rows = [r for r in csv.reader(open(os.path.join(g, f"{tag}_launches.csv"))) if len(r) > 5]
    h, body = rows[0], rows[1:]
    iN, iM, iV = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    c, n = collections.Counter(), 0
    for r in body:
        if r[iM] != "gpu__time_duration.sum":
            continue
        name = "K1 chfsi::filter_step_kernel (all variants)" if "filter_step_kernel" in r[iN] else r[iN]
        c[name] += float(r[iV].replace(",", "")) * 1e-9
        n += 1
    tot = sum(c.values())
    out = [f"# {tag}: kernel-time shares of a short c2 bench (3 warm-up + 1 timed problem), ncu launch list "
           "(cold-cache, serialised; shares, not absolutes)",
           "# command: ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --steps 1 "
           "--warmup 3 --no-e2e --no-cpu-baseline --no-sequence",
           f"# {n} launches, {tot:.3f} s of kernel time"]
    out += [f"{100 * t / tot:6.2f}%  {k}" for k, t in c.most_common(20)]
    open(os.path.join(ROOT, "profiles", "r02_launch_shares.txt"), "w").write("\n".join(out) + "\n")
    with open(os.path.join(g, f"{tag}_launches.csv"), "rb") as fi, gzip.open(os.path.join(ROOT, "profiles", "r02_launches.csv.gz"), "wb") as fo:
        fo.write(fi.read())
    print("\n".join(out[:6]))


main()
