"""Host link (B200 <-> host memory) probe: pinned allocation cost and copy bandwidth.

    python tools/hostlink_probe.py [GiB]

Prints the host's memory / cores, how long pinning N GiB takes, and H2D, D2H and
concurrent bidirectional copy bandwidth of 1 GiB pinned blocks (CUDA events).
"""
import json
import os
import sys
import time

import torch

gib = int(sys.argv[1]) if len(sys.argv) > 1 else 8
out = {"cpus": os.cpu_count()}
with open("/proc/meminfo") as f:
    for line in f:
        k, v = line.split(":")
        if k in ("MemTotal", "MemAvailable", "Hugepagesize"):
            out[k] = v.strip()
t0 = time.perf_counter()
host = torch.empty(gib << 30, dtype=torch.uint8, pin_memory=True)
out["pin_seconds_%dGiB" % gib] = round(time.perf_counter() - t0, 3)
dev = torch.empty(gib << 30, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, nbytes, reps=3):
    best = 0.0
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = max(best, nbytes / (time.perf_counter() - t) / 1e9)
    return round(best, 1)


def h2d():
    dev.copy_(host, non_blocking=True)


def d2h():
    host.copy_(dev, non_blocking=True)


half = (gib << 30) // 2


def both():
    with torch.cuda.stream(s1):
        dev[:half].copy_(host[:half], non_blocking=True)
    with torch.cuda.stream(s2):
        host[half:].copy_(dev[half:], non_blocking=True)


out["h2d_GBps"] = timed(h2d, gib << 30)
out["d2h_GBps"] = timed(d2h, gib << 30)
out["bidir_total_GBps"] = timed(both, gib << 30)
print(json.dumps(out))
