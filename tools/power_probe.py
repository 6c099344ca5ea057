"""Is K1 power-capped at mid widths? Runs many filter calls at one width (n = 13000) for ~20 s while
sampling nvidia-smi (SM clock, power, throttle reasons) every 100 ms; prints per-call times and the
clock / power samples. usage: python tools/power_probe.py <k> [seconds]"""
import json
import os
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1404_4161_b200 as chfsi  # noqa: E402


def main():
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 110
    secs = float(sys.argv[2]) if len(sys.argv) > 2 else 20
    n, m = 13000, 8
    torch.manual_seed(0)
    H = chfsi.colmajor(n, n)
    H.copy_(torch.randn(n, n, dtype=torch.complex128, device="cuda") / (2 * n) ** 0.5)
    Y0 = chfsi.colmajor(n, k)
    Y0.copy_(torch.randn(n, k, dtype=torch.complex128, device="cuda"))
    Y = chfsi.colmajor(n, k)
    ctx = chfsi.Context(0)
    samples, stop = [], threading.Event()

    def sampler():
        while not stop.is_set():
            out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout.strip()
            samples.append((time.time(), out))
            time.sleep(0.1)

    th = threading.Thread(target=sampler)
    th.start()
    t0 = time.time()
    times = []
    while time.time() - t0 < secs:
        Y.copy_(Y0)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        ctx.filter(H, Y, [m] * k, -2.2, 0.6, 1.6)
        e1.record()
        torch.cuda.synchronize()
        times.append((time.time() - t0, e0.elapsed_time(e1)))
    stop.set()
    th.join()
    ctx.close()
    ideal = 6.0 * n * n * k * m / 37.07e12 * 1e3
    q = max(1, len(times) // 5)
    for i in range(0, len(times), q):
        chunk = times[i:i + q]
        print(json.dumps({"k": k, "t_s": round(chunk[0][0], 2), "ms": round(sum(c[1] for c in chunk) / len(chunk), 4),
                          "eff": round(ideal / (sum(c[1] for c in chunk) / len(chunk)), 4)}))
    clk = [float(s[1].split(",")[0]) for s in samples if s[1]]
    pw = [float(s[1].split(",")[1]) for s in samples if s[1]]
    rs = sorted({s[1].split(",")[2].strip() for s in samples if s[1]})
    print(json.dumps({"k": k, "clock_min": min(clk), "clock_median": sorted(clk)[len(clk) // 2], "power_max": max(pw),
                      "power_median": sorted(pw)[len(pw) // 2], "reasons": rs, "samples": len(clk)}))


main()
