"""bench.py -- ChFSI on a synthetic correlated sequence shaped like the paper's DFT workloads.

Metric (BASELINE.json): "Chebyshev-filter FP64 TFLOP/s & frac of peak; time per eigenproblem at
1/2/4/8 GPU". A step is one eigenproblem of the c2 sequence solved by the whole hot path (Lanczos,
filter loops, CholQR2, Rayleigh-Ritz, locking, degree optimisation): n = 13000 complex128,
nev = 520, nex = 104, degree cap 36, tol 1e-10, H^(l+1) = H^(l) + 5e-4 * 40 * G_l.

  value   = algorithmic filter flops (8 n^2 sum(deg), all filter calls of the K timed problems)
            / device time of the K timed problems (inputs resident in HBM), TFLOP/s
  e2e     = the same, each problem's H^(l) copied host(pinned) -> device inside the timed region and
            the eigenvalues / residuals read back per problem
  filter_kernel_tflops: the filter alone (its CUDA-event time inside the steps), same convention
  roofline / frac_of_peak: K1 (the filter kernel), FP64 tensor (DMMA) bound, peak = 37.07 TF measured
            on this pool (profiles/r01_fp64_peaks.txt; MEASURED_PEAKS.json has no FP64 entry), counted
            in the real tensor flops K1 executes: 6 per complex MAC with Gauss's 3M product (default,
            --zmul 3), 8 with the 4M embedding (--zmul 4)

`python bench.py --gpus N --steps K --warmup W`; N > 1 under torchrun (row-panel sharding, NCCL).
`--impl reference` times the CPU oracle (oracle/, plain C) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Chebyshev-filter FP64 TFLOP/s & frac of peak; time per eigenproblem at 1/2/4/8 GPU"
FP64_PEAK_TFLOPS = 37.07  # DMMA.8x8x4 register-only probe at 1965 MHz (tools/fp64_probe.cu)
HBM_PEAK_GBS = None


def load_peaks():
    global HBM_PEAK_GBS
    try:
        HBM_PEAK_GBS = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        HBM_PEAK_GBS = 6650.0  # B200_PROFILING.md fallback


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        time.sleep(0.1)
        sm = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 8 and r[2].replace(".", "").isdigit()]
        pw = [float(r[3]) for r in self.rows if len(r) >= 8 and r[3].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 8 for i in range(4) if r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(pw) if pw else None, "samples": len(sm), "reasons": reasons}


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ------------------------------------------------------------------------------------------------
# sharding helpers (also exercised by tests/test_dist_cpu.py with gloo on CPU)
def rank_rows(n: int, world: int, rank: int):
    """1-D row panels: rank owns global rows [row0, row0 + nloc) (n divisible by world)."""
    if n % world:
        raise ValueError(f"n = {n} is not divisible by {world} ranks")
    nloc = n // world
    return rank * nloc, nloc


def build_panels(cf, row0: int, nloc: int, nprob: int, alloc):
    """This rank's column slab H^(l)[:, row0:row0+nloc] of problems l = 0..nprob-1 of the sequence
    (H^(1) = Q Lambda Q^H, then H^(l+1) = H^(l) + delta*40*G_l), each written into alloc() -> an
    (nloc x n) C-contiguous array / pinned tensor (i.e. a column-major n x nloc slab)."""
    import gen as G
    from gen.configs import HNORM

    n = cf["n"]
    wy = G.wy(n, cf["nd"], cf["seed"])
    out = []
    for ell in range(nprob):
        buf = alloc()
        hv = (buf.numpy() if hasattr(buf, "numpy") else buf).T  # F-ordered (n x nloc) view
        if ell == 0:
            wy.panel(row0, nloc, out=hv)
        else:
            prev = out[-1]
            hv[...] = (prev.numpy() if hasattr(prev, "numpy") else prev).T
            G.perturb(hv, cf["seed"], ell, cf["delta"] * HNORM, c0=row0)
        out.append(buf)
    return out


def max_over_ranks(x: float, dist, device):
    """The bench's timing reduction: max of a per-rank scalar over all ranks."""
    if dist is None:
        return x
    import torch

    t = torch.tensor([x], device=device, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def oracle_filter_sample(cf, ncols: int, deg: int):
    """The oracle (plain C, OpenMP) filtering `ncols` columns of the c2 start block with H^(1) at a
    uniform degree: a bounded sample of the filter work of the same workload. Returns (TFLOP/s,
    seconds, threads)."""
    import numpy as np

    import gen as G
    import oracle as O

    n = cf["n"]
    w = G.wy(n, cf["nd"], cf["seed"])
    H = w.full()
    Y0 = G.start_basis(n, ncols, cf["seed"])
    lam = w.lam
    l1, a, b = lam[0] - 0.05, lam[cf["nev"] + cf["nex"] - 1], 48.0
    c, e = (a + b) / 2, (b - a) / 2
    t0 = time.perf_counter()
    Y, mv = O.chebyshev_filter(H, Y0, [deg] * ncols, l1, c, e)
    dt = time.perf_counter() - t0
    assert np.isfinite(Y).all()
    return 8.0 * n * n * mv / dt / 1e12, dt, int(os.environ.get("OMP_NUM_THREADS", host_cores()))


def run_reference(args, cf, rank, world):
    if rank != 0:
        return
    K, W = args.steps, args.warmup
    ncols, deg = 8, 8
    vals = []
    for i in range(W + K):
        v, dt, thr = oracle_filter_sample(cf, ncols, deg)
        if i >= W:
            vals.append((v, dt))
    value = sum(v for v, _ in vals) / len(vals)
    ms = 1e3 * sum(dt for _, dt in vals) / len(vals)
    sample = (f"oracle.chebyshev_filter (naive C, OpenMP) on {ncols} columns of the c2 start block, "
              f"H^(1) n={cf['n']}, uniform degree {deg} ({8.0 * cf['n'] ** 2 * ncols * deg:.3g} flop per step)")
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus,
           "steps": K, "warmup": W, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": "c2 (filter-only sample)", "n": cf["n"], "nev": cf["nev"], "nex": cf["nex"]},
           "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": thr, "kind": "oracle", "sample": sample},
           "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="chfsi", choices=["chfsi", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sequence", action="store_true",
                    help="skip the untimed whole-sequence pass (per-problem times incl. the random-start problem 1)")
    ap.add_argument("--exchange", default="push", choices=["allgather", "push"],
                    help="N > 1: per-step operand exchange -- the filter epilogue's peer push (default: the "
                         "exchange fused into K1, 8-16 %% faster than the pipelined allgather on emulated ranks, "
                         "profiles/r02_exchange_probe.jsonl) or the pipelined in-place allgather")
    ap.add_argument("--eig", default="refine", choices=["refine", "dense"],
                    help="Rayleigh-Ritz k x k eigensolve: Jacobi-type refinement with dense fallback, or dense only")
    ap.add_argument("--zmul", type=int, default=3, choices=[3, 4],
                    help="complex filter arithmetic: 3 = Gauss 3M (default), 4 = 4M real embedding")
    ap.add_argument("--emulate-ranks", type=int, default=1,
                    help="run the N > 1 path as P threads on GPU 0 (correctness of the sharded path; not a timing)")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    load_peaks()
    from gen.configs import CONFIGS, DEG0, HNORM, LANCZOS_STEPS, MAX_LOOPS

    cf = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, cf, rank, world)
        return

    if args.emulate_ranks > 1:
        run_emulated(args, cf)
        return
    if args.gpus != world and rank == 0:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE = {world}: launch N > 1 under torch.distributed.run; "
              f"measuring {world} GPU(s)", file=sys.stderr)
    import torch

    import paper_1404_4161_b200 as chfsi

    torch.cuda.set_device(local_rank)
    group = None
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        t = torch.zeros(1, device="cuda")
        dist.all_reduce(t)
        # the library owns its NCCL communicator: rank 0's ncclUniqueId is broadcast over torch.distributed
        obj = [chfsi.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        group = TorchGroup(dist, obj[0])
    rank_main(args, cf, rank, world, local_rank, group)
    if world > 1:
        dist.destroy_process_group()


class TorchGroup:
    """N > 1 ranks = processes under torchrun; the library's NCCL communicator from a broadcast id."""

    def __init__(self, dist, nccl_id):
        self.dist, self.nccl_id = dist, nccl_id

    def context(self, chfsi, local_rank, rank, world):
        return chfsi.Context(local_rank, nccl_id=self.nccl_id, rank=rank, nranks=world)

    def barrier(self):
        import torch

        torch.cuda.synchronize()
        self.dist.barrier()
        torch.cuda.synchronize()

    def max(self, x):
        return max_over_ranks(x, self.dist, "cuda")


class ThreadGroup:
    """--emulate-ranks P: P ranks as threads on GPU 0 (chfsi local group, one stream each). Runs the whole
    N > 1 code path of this script (row panels, packed operands, collectives, reductions) on one GPU;
    its timings are not multi-GPU timings (the ranks share one device)."""

    def __init__(self, P):
        import threading

        import paper_1404_4161_b200 as chfsi

        self.P = P
        self.lg = chfsi.LocalGroup(P)
        self.bar = threading.Barrier(P)
        self.vals = [0.0] * P

    def context(self, chfsi, local_rank, rank, world):
        import torch

        return chfsi.Context(0, stream=torch.cuda.current_stream(), local_group=self.lg, rank=rank)

    def barrier(self):
        import torch

        torch.cuda.current_stream().synchronize()
        self.bar.wait()

    def max(self, x):
        import threading

        rank = threading.current_thread().rank
        self.vals[rank] = x
        self.bar.wait()
        m = max(self.vals)
        self.bar.wait()
        return m


def run_emulated(args, cf):
    import threading

    import torch

    P = args.emulate_ranks
    group = ThreadGroup(P)
    errs = []

    def work(r):
        threading.current_thread().rank = r
        try:
            s = torch.cuda.Stream(device=0)
            with torch.cuda.stream(s):
                rank_main(args, cf, r, P, 0, group)
        except BaseException as ex:  # surfaced after join
            errs.append(ex)
            group.bar.abort()

    th = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]


def rank_main(args, cf, rank, world, local_rank, group):
    import numpy as np
    import torch

    import gen as G
    import paper_1404_4161_b200 as chfsi
    from gen.configs import DEG0, LANCZOS_STEPS, MAX_LOOPS

    n, nev, nex = cf["n"], cf["nev"], cf["nex"]
    k = nev + nex
    row0, nloc = rank_rows(n, world, rank)
    K, W = args.steps, args.warmup
    nprob = W + K
    # the configuration's own sequence (BASELINE.json: c2 = 10 problems) is also solved once, untimed by
    # the step clock, after the timed passes: its per-problem device times (problem 1 included) are reported
    nseq = 0 if args.no_sequence else cf["nprob"]
    nbuild = max(nprob, nseq)

    # ---- inputs: this rank's column slab of every H^(l) (pinned host + HBM), start basis rows ----
    t_gen = time.perf_counter()
    host_H = build_panels(cf, row0, nloc, nbuild,
                          lambda: torch.empty((nloc, n), dtype=torch.complex128, pin_memory=True))
    dev_H = []
    for hp in host_H:
        d = torch.empty((nloc, n), dtype=torch.complex128, device="cuda")
        d.copy_(hp)
        dev_H.append(d.t())
    X0 = G.start_basis(n, k, cf["seed"], row0, nloc)
    torch.cuda.current_stream().synchronize()
    t_gen = time.perf_counter() - t_gen

    ctx = group.context(chfsi, local_rank, rank, world) if group else chfsi.Context(local_rank)
    ctx.set_complex_mult(args.zmul)
    ctx.set_eigensolver(0 if args.eig == "refine" else 1)
    ctx.reserve(n, nloc, k)
    exchange = args.exchange if world > 1 else None
    if world > 1 and args.exchange == "push":
        try:
            ctx.set_exchange(1)  # collective: maps every rank's operand buffers
        except RuntimeError as ex:  # every rank gets the same verdict (the library agrees on it)
            ctx.set_exchange(0)
            exchange = "allgather (peer push unavailable: %s)" % ex
            if rank == 0:
                print("warning: " + exchange, file=sys.stderr)
    stream = torch.cuda.current_stream()

    def barrier():
        if group:
            group.barrier()
        else:
            torch.cuda.synchronize()

    def rmax(x):
        return group.max(x) if group else x

    def run_pass(e2e: bool):
        Xd = chfsi.to_colmajor(X0)
        # e2e: every timed problem's panel goes host (pinned) -> device inside the timed region, double
        # buffered on a copy stream so problem l+1's H2D overlaps problem l's solve (the copy engine
        # runs beside the kernels); the first timed copy is not overlapped
        stages = [chfsi.colmajor(n, nloc), chfsi.colmajor(n, nloc)] if e2e else None
        copy_stream = torch.cuda.Stream() if e2e else None
        copied = {}
        ev = {}
        sampler = ClockSampler(local_rank)
        launches = {}

        def issue_copy(ell):
            free = torch.cuda.Event()
            free.record(stream)  # the previous user of this buffer (problem ell - 2) is done
            copy_stream.wait_event(free)
            with torch.cuda.stream(copy_stream):
                stages[ell % 2].t().copy_(host_H[ell], non_blocking=True)
                copied[ell] = torch.cuda.Event()
                copied[ell].record(copy_stream)

        def get_h(ell):
            if ell == W:
                barrier()
                launches["start"] = ctx.kernel_launches
                if rank == 0:
                    sampler.start()
                ev["start"] = torch.cuda.Event(enable_timing=True)
                ev["start"].record(stream)
                if e2e:
                    issue_copy(W)
            if e2e and ell >= W:
                stream.wait_event(copied[ell])
                if ell + 1 < nprob:
                    issue_copy(ell + 1)
                return stages[ell % 2]
            return dev_H[ell]

        out = ctx.solve_sequence(get_h, nprob, Xd, nev, nex, cf["tol"], deg_cap=cf["cap"], deg0=DEG0,
                                 max_loops=MAX_LOOPS, lanczos_steps=LANCZOS_STEPS, seed=cf["seed"], n=n, row0=row0)
        if e2e:
            Xd.cpu()  # the final block read back (part of the last step)
        ev["end"] = torch.cuda.Event(enable_timing=True)
        ev["end"].record(stream)
        barrier()
        clocks = sampler.stop() if rank == 0 else None
        ms = rmax(ev["start"].elapsed_time(ev["end"]))
        launches["n"] = ctx.kernel_launches - launches["start"]
        return out, ms, clocks, launches["n"]

    out, ms, clocks, nlaunch = run_pass(False)
    reps = out["reports"][W:]
    flops = sum(r["filter_flops"] for r in reps)
    t_filter = rmax(sum(r["t_filter"] for r in reps))
    t_k1 = rmax(sum(r["t_filter_kernel"] for r in reps))
    k1_launches = sum(r["filter_launches"] for r in reps)
    value = flops / (ms * 1e-3) / 1e12
    # per-GPU kernel rates: every rank executes 1/world of the filter flops (its row panel) in its own
    # K1 launches (emulated ranks share one GPU: their kernel intervals overlap, so no per-GPU rate exists)
    gpus = 1 if args.emulate_ranks > 1 else world
    filt_tf = flops / gpus / t_filter / 1e12  # whole filter calls (incl. the Y -> state copy, finite check)
    k1_tf = flops / gpus / t_k1 / 1e12 if t_k1 > 0 else float("nan")  # inside the K1 launches only
    e2e = None
    if not args.no_e2e:
        out2, ms2, _, _ = run_pass(True)
        flops2 = sum(r["filter_flops"] for r in out2["reports"][W:])
        e2e = {"value": flops2 / (ms2 * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": ms2 / K,
               "h2d_bytes_per_step": 16 * n * nloc, "d2h_bytes_per_step": 16 * nev + (16 * nloc * k) // K,
               "note": "each problem's H panel copied from pinned host memory inside the timed region (double "
                       "buffered: problem l+1's copy overlaps problem l's solve); eigenvalues/residuals read "
                       "back per problem, the final block once"}

    # the configuration's whole sequence from the start basis (problem 1 = random start, then reuse)
    sequence = None
    if nseq:
        Xs = chfsi.to_colmajor(X0)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        ev0.record(stream)
        out3 = ctx.solve_sequence(lambda ell: dev_H[ell], nseq, Xs, nev, nex, cf["tol"], deg_cap=cf["cap"], deg0=DEG0,
                                  max_loops=MAX_LOOPS, lanczos_steps=LANCZOS_STEPS, seed=cf["seed"], n=n, row0=row0)
        ev1.record(stream)
        barrier()
        per = [rmax(r["t_total"]) for r in out3["reports"]]
        sequence = {"problems": nseq, "avg_s": rmax(ev0.elapsed_time(ev1)) / 1e3 / nseq,
                    "problem1_s": per[0], "later_avg_s": sum(per[1:]) / max(len(per) - 1, 1),
                    "per_problem_s": per, "loops": [r["loops"] for r in out3["reports"]],
                    "converged": all(r["converged"] == nev for r in out3["reports"]),
                    "max_resid_over_tol": float(np.max(out3["resid"])) / cf["tol"],
                    "note": ("the configuration's sequence solved once from the start basis after the timed passes "
                             "(device time, CUDA events): avg_s over all problems including the random-start problem 1")}
        del Xs

    # roofline of K1: FP64 DMMA-bound contraction; achieved from the filter calls' CUDA-event time. traffic:
    # DRAM bytes of one full-width launch of THIS configuration from an ncu --set full capture (null when
    # none was taken for it)
    traffic, traffic_info = None, None
    tp = os.path.join(ROOT, "profiles", "k1_traffic.json")
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp)).get(args.config if args.zmul == 3 else f"{args.config}_4m", {})
            traffic = tj.get("dram_bytes_per_launch")
            traffic_info = {k: tj.get(k) for k in ("launch", "algorithmic_bytes_per_launch", "source")} if tj else None
        except Exception:
            traffic = None
    # the tensor work K1 executes per complex multiply-add: 6 real flops (3M) or 8 (4M); `value` and
    # filter_kernel_tflops keep the paper's ZGEMM convention 8 n^2 sum(deg)
    tensor_per_zmac = 6.0 if args.zmul == 3 else 8.0
    k1_tensor_tf = k1_tf * tensor_per_zmac / 8.0
    roofline = {"bound": "tensor", "achieved": k1_tensor_tf, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": k1_tensor_tf / FP64_PEAK_TFLOPS, "traffic": traffic,
                "kernel": f"K1 filter_step_kernel ({args.zmul}M complex arithmetic, DMMA.8x8x4, TMA, persistent stream-K)",
                "launches": k1_launches, "avg_launch_ms": 1e3 * t_k1 / max(k1_launches, 1),
                "flops_per_launch": flops / gpus * tensor_per_zmac / 8.0 / max(k1_launches, 1),
                "achieved_def": (f"{tensor_per_zmac:g} n^2 sum(deg) (the real FP64 tensor flops of the {args.zmul}M "
                                 "complex product) over the timed problems / sum of CUDA-event times of the K1 launches"),
                "achieved_zgemm_equivalent": k1_tf, "traffic_launch": traffic_info,
                "peak_source": "measured FP64 DMMA peak (register-only DMMA loop, 1965 MHz), profiles/r01_fp64_peaks.txt"}

    if args.emulate_ranks > 1:  # P ranks on one GPU: the launches of different ranks overlap in time
        roofline = None
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # a bounded sample of the same workload (~10 s of the oracle on the box's host cores)
        ncols, deg = 48, 16
        v, dt, thr = oracle_filter_sample(cf, ncols, deg)
        cpu = {"value": v, "unit": "TFLOP/s", "cores": thr, "kind": "oracle",
               "sample": f"oracle.chebyshev_filter (naive C, OpenMP) on {ncols} columns of the {args.config} start "
                         f"block with H^(1), degree {deg}: {8.0 * n * n * ncols * deg:.3g} flop in {dt:.1f} s"}

    # correctness guard on the timed problems: all converged, residuals within tol (R8)
    conv = all(r["converged"] == nev for r in reps)
    res_max = float(np.max(out["resid"][W:]))
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": 1 if args.emulate_ranks > 1 else world,
            "steps": K, "warmup": W,
            "ms_per_step": ms / K, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: ChFSI sequence, one eigenproblem per step", "n": n,
                       "nev": nev, "nex": nex, "deg_cap": cf["cap"], "tol": cf["tol"], "delta": cf["delta"],
                       "problems": f"{W} warm-up + {K} timed of the correlated sequence",
                       "parallelism": (f"1-D row panels over {world} emulated ranks on one GPU" if args.emulate_ranks > 1
                                       else f"1-D row panels over {world} GPU(s)" if world > 1 else "single GPU"),
                       "exchange": exchange, "complex_mult": f"{args.zmul}M",
                       "eigensolver": args.eig,
                       "l2": "inputs larger than L2 (H panel per problem >> 126 MB)"},
            "time_per_eigenproblem_s": ms / K / 1e3,
            "filter_kernel_tflops": filt_tf if args.emulate_ranks == 1 else None,
            "frac_of_peak": filt_tf * tensor_per_zmac / 8.0 / FP64_PEAK_TFLOPS if args.emulate_ranks == 1 else None,
            "flop_convention": ("value / filter_kernel_tflops count 8 n^2 sum(deg) (ZGEMM convention); frac_of_peak "
                                f"and roofline count the {tensor_per_zmac:g} real tensor flops per complex MAC "
                                f"the {args.zmul}M kernel executes"),
            "filter_share_of_step": t_filter / (ms * 1e-3),
            "loops_per_problem": [r["loops"] for r in reps],
            "phase_s_per_problem": {ph: sum(r[f"t_{ph}"] for r in reps) / len(reps)
                                    for ph in ("lanczos", "filter", "qr", "rr", "eig", "opt", "total")},
            "eigensolves_per_problem": {"refined": [r["eig_refined"] for r in reps], "dense": [r["eig_dense"] for r in reps]},
            "matvecs_filter_per_problem": [r["matvecs_filter"] for r in reps],
            "converged": conv, "max_resid_over_tol": res_max / cf["tol"],
            "sequence": sequence,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks, "gpu_launches": nlaunch,
            "input_generation_s": t_gen,
        }
        if args.emulate_ranks > 1:
            line["emulated_ranks"] = world
        print(json.dumps(line), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
