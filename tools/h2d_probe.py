"""Host->device copy rate from pinned memory (the e2e leg's H upload): one copy vs chunks on several
streams, 2.7 GB (a c2 H panel). usage: python tools/h2d_probe.py"""
import json
import time

import torch


def main():
    nbytes = 13000 * 13000 * 16
    h = torch.empty(nbytes // 8, dtype=torch.float64, pin_memory=True)
    h.fill_(1.0)
    d = torch.empty_like(h, device="cuda")
    torch.cuda.synchronize()
    for nstreams in (1, 2, 4, 8):
        streams = [torch.cuda.Stream() for _ in range(nstreams)]
        best = 1e9
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            chunks_h = h.chunk(nstreams)
            chunks_d = d.chunk(nstreams)
            for s, ch, cd in zip(streams, chunks_h, chunks_d):
                with torch.cuda.stream(s):
                    cd.copy_(ch, non_blocking=True)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        print(json.dumps({"streams": nstreams, "GB": nbytes / 1e9, "s": best, "GB_per_s": nbytes / best / 1e9}), flush=True)
    # device -> host for reference
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(json.dumps({"d2h": True, "GB_per_s": nbytes / dt / 1e9}))


main()
