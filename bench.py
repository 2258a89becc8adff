#!/usr/bin/env python
"""Benchmark of the B200 gate-application hot path (driver contract: one JSON line).

Metric (BASELINE.json): "sec/gate & effective HBM GB/s vs roofline at N
qubits, 1/2/4/8 B200; adder circuit time".

Workload at N=1 GPU = BASELINE config[1]: "Hadamard + random 1q/2q gate
layers, N=33 FP64 on 1xB200 (128 GiB state)": H on all 33 qubits followed by
random layers drawn with the reference's generator (tests/circuits.py
random_circuit, depth 33 per layer, every gate kind).  One *step* = one
layer of 33 gates applied to the 2**33-amplitude state resident in HBM.

  value      = effective HBM GB/s over the timed steps: the algorithmic bytes
               of every gate (2*16*L read+write per non-diagonal gate,
               2*16*L/2**k for a diagonal on k qubits),
               summed over all GPUs, divided by the device time (CUDA events,
               max over ranks).  Gates are fused into tile passes, so this can
               exceed the HBM peak; roofline.* reports the per-pass truth.
  roofline   = the dominant kernel (k_fused, one read + one write of the
               state per launch), its algorithmic bytes / average launch time
               from CUDA events bracketing every launch on its own stream.
  e2e        = the same metric through the public API: run_circuit() on a
               Circuit built on the host (the Hadamard layer + one random layer
               + measure-all, i.e. the C2 circuit from |0..0>), state allocated
               by the call, report copied back; e2e.dense = the same calls with
               support tracking off (every tile of every pass).
  cpu_baseline = the reference algorithm (numpy port in oracle/, threaded over
               the box's cores) on a bounded sample of the same layers at N=24.

`--impl reference` runs only that CPU arm (rank 0) and prints its own line.
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sec/gate & effective HBM GB/s vs roofline at N qubits, 1/2/4/8 B200; adder circuit time"
SEED = 20240817
CPU_SAMPLE_N = 26


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def measured_traffic(bytes_per_launch: int):
    """DRAM traffic per fused-pass launch from the committed ncu capture
    (profiles/r02_traffic.json: dram read + write / algorithmic bytes, measured at N=32),
    applied to this launch size; (None, None) if the file is absent."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r02_traffic.json")
    try:
        with open(path) as fh:
            t = json.load(fh)
        return int(bytes_per_launch * t["ratio"]), f"profiles/r02_traffic.json (ncu --set full at N={t['n_qubits']}: " \
                                                   f"DRAM/algorithmic = {t['ratio']})"
    except (OSError, KeyError, ValueError):
        return None, None


def benchmark_kat(report, n: int, tol_z: float = 1e-12, tol_x: float = 1e-12):
    """build_benchmark(n) known answers at full size (test_builders.py:21-33): qubits hit
    twice read Qz=0, Qx=0.5, the others Qx=0, Qz=0.5.  Returns (ok, max deviation)."""
    twice = {n - 5, n - 6, n - 1, 0, n - 2, 1}
    dev = 0.0
    for q in range(n):
        if q in twice:
            dz, dx = abs(report.qz[q]), abs(report.qx[q] - 0.5)
        else:
            dz, dx = abs(report.qz[q] - 0.5), abs(report.qx[q])
        dev = max(dev, dz, dx)
        if dz > tol_z or dx > tol_x:
            return False, dev
    return True, dev


def benchmark_codebook_kat(codebook, n: int) -> bool:
    """BYTE benchmark codebook known answer: N+2 magnitudes m_0 = 0, m_1 = 1,
    m_k = fl(sqrt(1/2) * m_(k-1)); phases {0}."""
    from paper_2511_03359_b200 import gates as pg
    want = [0.0, 1.0]
    while len(want) < n + 2:
        want.append(pg.SQRT_HALF * want[-1])
    return list(codebook.mags) == want and list(codebook.thetas) == [0.0]


def workload_layers(n: int, n_layers: int):
    """H on every qubit, then random layers (depth n) — the BASELINE config[1] circuit."""
    from tests.circuits import random_circuit
    from oracle.ref_gates import OGate
    rng = np.random.default_rng(SEED)
    layers = [tuple(OGate("H", (q,)) for q in range(n))]
    for _ in range(n_layers - 1):
        layers.append(random_circuit(rng, n, n, measured=False).gates)
    return layers


def layer_bytes(layer, n: int, bpe: int = 16) -> int:
    from oracle.cpu_baseline import gate_bytes
    return sum(gate_bytes(g, n, bpe) for g in layer)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    QUERY = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def dist_init(world):
    if world <= 1:
        return None
    import torch.distributed as dist
    dist.init_process_group("gloo")
    return dist


def max_over_ranks(dist, value: float) -> float:
    if dist is None:
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(dist, value: float) -> float:
    if dist is None:
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


# --------------------------------------------------------------------------------------------
def cpu_baseline(steps: int, n_layers: int, sample_n: int = CPU_SAMPLE_N):
    from oracle.cpu_baseline import time_layers
    layers = workload_layers(sample_n, n_layers)
    chosen = [layers[i % len(layers)] for i in range(steps)]
    res, threads = time_layers(chosen, sample_n)
    secs = sum(r[0] for r in res)
    byts = sum(r[1] for r in res)
    gates = sum(r[2] for r in res)
    # the reference itself runs numpy on ONE core -- the same port on one
    # thread at three sizes, and sec/gate extrapolated to the bench size (x 2 per qubit, the
    # per-gate work is 2^N; fitted on the measured sizes)
    import math
    single = []
    for ns in (sample_n - 4, sample_n - 3, sample_n - 2):
        r1, _ = time_layers([workload_layers(ns, 2)[1]], ns, threads=1)
        single.append((ns, r1[0][0] / r1[0][2], r1[0][1] / r1[0][0] / 1e9))
    xs = [a for a, _, _ in single]
    ys = [math.log2(b) for _, b, _ in single]
    xm, ym = sum(xs) / len(xs), sum(ys) / len(ys)
    slope = sum((x - xm) * (y - ym) for x, y in zip(xs, ys)) / sum((x - xm) ** 2 for x in xs)
    extrap = lambda nn: 2 ** (ym + slope * (nn - xm))  # noqa: E731
    return {"value": byts / secs / 1e9, "unit": "GB/s", "cores": threads, "kind": "port",
            "sec_per_gate": secs / gates,
            "single_core": {"sec_per_gate": {str(a): round(b, 5) for a, b, _ in single},
                            "GBps": {str(a): round(c, 3) for a, _, c in single},
                            "fit_log2_slope_per_qubit": round(slope, 3),
                            "extrapolated_sec_per_gate_n33": round(single[-1][1] * 2 ** (33 - single[-1][0]), 2),
                            "fit_extrapolated_sec_per_gate_n33": round(extrap(33), 2),
                            "what": "numpy port, 1 thread (the reference's own execution model), one C2 "
                                    "layer per size; N=33 extrapolated (not measured) as sec/gate x 2^(33-N) "
                                    "from the largest size (per-gate work is 2^N), and by the log-linear fit"},
            "threaded_extrapolated_sec_per_gate_n33": round(secs / gates * 2 ** (33 - sample_n), 2),
            "sample": f"{len(chosen)} layer(s) x {n_layers}-layer workload at N={sample_n} FP64 "
                      f"({gates} gates, {secs:.1f} s), numpy port of svsim/kernels.py in oracle/, "
                      f"{threads} threads"}


def fp64_ops_per_amplitude(op) -> float:
    """FP64 instructions per amplitude of one gate in the numpy-exact arithmetic of the
    passes (sv_arith.cuh / sv_jit_dev.cuh): generic 1Q 10 (4 DMUL + 4 DFMA + 2 DADD), real
    1Q 6, monomial 0, any non-monomial 2Q 22, diagonal 4 on the selected 2^-k, Z 0 (fallback
    model for passes the generic kernel runs; sv_plan_pass_costs counts the others)."""
    import numpy as np
    from paper_2511_03359_b200 import _native as nat
    m = np.array(op.m[:32])
    if op.kind == nat.SV_OP_1Q:
        mm = m[:8]
        if np.count_nonzero(mm) == 2 and all(np.count_nonzero(mm.reshape(4, 2), axis=1) <= 1):
            return 0.0
        return 6.0 if not np.any(mm[1::2]) else 10.0
    if op.kind == nat.SV_OP_2Q:
        if np.count_nonzero(m) == 4:
            return 0.0
        return 22.0                       # real 4x4 matrices run the generic row4 too
    if op.m[0] == -1.0 and op.m[1] == 0.0:
        return 0.0
    return 4.0 / (1 << bin(op.diag_mask).count("1"))


def fp64_aware_roofline(n: int, seq, tile_bits: int, pass_ms: float, hbm_peak: float, sm_mhz: float,
                        combine_diag: bool = False) -> dict:
    """Per launch the fused pass has two floors: its HBM bytes at the copy peak and its
    FP64 instructions at 64 lanes/clk/SM x 148 SMs x the SM clock measured under load.
    The FP64 count per pass is the library's own (sv_plan_pass_costs: warp instructions
    of the specialised kernel per amplitude -- a diagonal op selecting lanes still issues
    for the whole warp).  Returns the sum of max(floors) over the timed launches (the
    library's own pass split) against their measured time."""
    import ctypes
    import numpy as np
    from paper_2511_03359_b200 import _native as nat
    from paper_2511_03359_b200.device import ops_array
    lib = nat.load()
    sms = ctypes.c_int(0)
    lib.sv_sm_count(0, ctypes.byref(sms))
    fp64_peak = 64.0 * sms.value * sm_mhz * 1e6
    hbm_ms = 2 * 16 * 2 ** n / (hbm_peak * 1e9) * 1e3
    floor = f64_total = hbm_total = 0.0
    n_pass = 0
    per_amp = []
    for ops in seq:
        ends = (ctypes.c_int * 4096)()
        cost = np.zeros(4096)
        k = lib.sv_plan_pass_costs(n, nat.SV_FP64, ops_array(ops), len(ops), tile_bits, ends, nat.dptr(cost), 4096,
                                   1 if combine_diag else 0)
        nat.check(min(k, 0))
        a = 0
        for i in range(k):
            c = cost[i] if cost[i] >= 0 else sum(fp64_ops_per_amplitude(o) for o in ops[a:ends[i]])
            per_amp.append(float(c))
            f = c * 2 ** n / fp64_peak * 1e3
            a = ends[i]
            floor += max(hbm_ms, f)
            f64_total += f
            hbm_total += hbm_ms
            n_pass += 1
    return {"fp64_peak_Tops": round(fp64_peak / 1e12, 2), "passes": n_pass,
            "fp64_per_amplitude": {"min": min(per_amp), "mean": round(sum(per_amp) / len(per_amp), 1),
                                   "max": max(per_amp)} if per_amp else None,
            "hbm_floor_ms": round(hbm_total, 1), "fp64_floor_ms": round(f64_total, 1),
            "max_floor_ms": round(floor, 1), "measured_ms": round(pass_ms, 1),
            "frac": round(floor / pass_ms, 4) if pass_ms else None,
            "what": "sum over the timed launches of max(HBM bytes / copy peak, FP64 instructions / "
                    "(64 x SMs x measured SM clock)) vs their event-timed sum: passes carrying many "
                    "generic U2/U4 gates are FP64-bound, not HBM-bound"}


def fused_parity(n_small: int, device: int, tile_bits: int) -> dict:
    """One C2 layer at n_small through fused passes vs one kernel per gate (fuse=False), bit
    for bit, and at N=18 against the CPU oracle (test infrastructure, outside the timed
    region)."""
    import numpy as np
    import paper_2511_03359_b200 as pb
    from oracle import ref_engine
    from oracle.ref_builders import OCircuit
    from tests.circuits import to_product
    out = {}
    lay = workload_layers(n_small, 3)[2]
    circ = to_product(OCircuit(n_small, tuple(lay)))
    a = pb.run_circuit(circ, device=device, tile_bits=tile_bits).gathered_state()
    b = pb.run_circuit(circ, device=device, fuse=False).gathered_state()
    out[f"fused_vs_per_gate_n{n_small}_bit_exact"] = bool(np.array_equal(a, b))
    del a, b
    lay = workload_layers(18, 3)[2]
    oc = OCircuit(18, tuple(lay))
    got = pb.run_circuit(to_product(oc), device=device, tile_bits=tile_bits).gathered_state()
    out["oracle_n18_bit_exact"] = bool(np.array_equal(got, ref_engine.run_circuit(oc, ranks=1).gathered_state()))
    return out


_COLD = r"""
import json, os, sys, time
t_start = time.perf_counter()
sys.path.insert(0, sys.argv[1])
import paper_2511_03359_b200 as pb
from paper_2511_03359_b200 import _native as nat
from paper_2511_03359_b200.device import jit_stats
from oracle.ref_builders import OCircuit
from tests.circuits import to_product
n, layers, device, tile_bits = (int(x) for x in sys.argv[2:6])
sys.path.insert(0, sys.argv[1])
import bench
wl = bench.workload_layers(n, layers)
circ = pb.Circuit(n, tuple(to_product(OCircuit(n, tuple(wl[0]))).gates) + tuple(to_product(OCircuit(n, tuple(wl[1]))).gates)
                  + (pb.gates.measure_all(),))
t_imp = time.perf_counter()
import ctypes
c = ctypes.c_int(0)
nat.check(nat.load().sv_device_count(ctypes.byref(c)))
nat.check(nat.load().sv_set_device(device))
t_ctx0 = time.perf_counter()
free = ctypes.c_uint64(0); tot = ctypes.c_uint64(0)
nat.check(nat.load().sv_mem_info(device, ctypes.byref(free), ctypes.byref(tot)))   # creates the context
t_ctx = time.perf_counter() - t_ctx0
sys.stderr.write(f"cold child: free {free.value / 2**30:.1f} GiB of {tot.value / 2**30:.1f}\n")
t0 = time.perf_counter()
res = pb.run_circuit(circ, device=device, tile_bits=tile_bits)
q = res.report.qz[0]
t_first = time.perf_counter() - t0
del res
t0 = time.perf_counter()
res2 = pb.run_circuit(circ, device=device, tile_bits=tile_bits)
q = res2.report.qz[0]
t_second = time.perf_counter() - t0
print(json.dumps({"first_call_s": t_first, "second_call_s": t_second, "context_s": t_ctx,
                  "import_s": t_imp - t_start, "jit": jit_stats(), "free_GiB_at_start": free.value / 2**30}))
"""


def cold_e2e(n: int, layers: int, device: int, tile_bits: int) -> dict:
    """e2e of a FRESH process (run_circuit(H layer + layer + M), the same call as the warm e2e):
    context creation, 2^N allocation, the pass kernels loaded from the persistent cubin
    cache this process filled (sv_jit.cu) -- no NVRTC -- and the measure-all."""
    import subprocess
    root = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-c", _COLD, root, str(n), str(layers), str(device), str(tile_bits)],
                       capture_output=True, text=True, timeout=600)
    if r.returncode != 0:
        import ctypes
        from paper_2511_03359_b200 import _native as nat
        free, tot = ctypes.c_uint64(0), ctypes.c_uint64(0)
        nat.load().sv_mem_info(device, ctypes.byref(free), ctypes.byref(tot))
        child = [ln for ln in r.stderr.splitlines() if ln.startswith("cold child")]
        return {"error": (r.stderr or r.stdout)[-400:], "parent_free_GiB": round(free.value / 2 ** 30, 1),
                "child": child[-1] if child else None}
    d = json.loads(r.stdout.strip().splitlines()[-1])
    gb = layer_bytes(workload_layers(n, layers)[0], n) + layer_bytes(workload_layers(n, layers)[1], n)
    return {"value": round(gb / d["first_call_s"] / 1e9, 2), "unit": "GB/s",
            "first_call_s": round(d["first_call_s"], 4), "warm_second_call_s": round(d["second_call_s"], 4),
            "context_init_s": round(d["context_s"], 3), "import_s": round(d["import_s"], 2),
            "jit_disk_hits": d["jit"]["disk_hits"], "nvrtc_compiles": d["jit"]["compiled"],
            "what": "first run_circuit(H layer + layer + M) in a new process after CUDA context creation: 2^N "
                    "allocation, pass kernels from the on-disk cubin cache, measure-all, report to host"}


def tier_run(n: int, fast_gib: float, chunk_gib: float, device: int) -> dict:
    """build_benchmark(n) FP64 larger than HBM, the reference's staging plan
    executed with the slow chunks in pinned host memory (tier.py / csrc/sv_tier.cu)."""
    import ctypes
    import paper_2511_03359_b200 as pb
    from paper_2511_03359_b200 import _native as nat
    from paper_2511_03359_b200.tier import TierConfig
    free, tot = ctypes.c_uint64(0), ctypes.c_uint64(0)
    nat.check(nat.load().sv_mem_info(device, ctypes.byref(free), ctypes.byref(tot)))
    if free.value < (fast_gib + 4) * 2 ** 30:
        return {"skipped": f"needs {fast_gib + 4:.0f} GiB free HBM, {free.value / 2**30:.0f} GiB free"}
    cfg = TierConfig(int(fast_gib * 2 ** 30), int(chunk_gib * 2 ** 30))
    circ = pb.build_benchmark(n)
    t0 = time.perf_counter()
    res = pb.run_circuit(circ, tier_config=cfg, tier_execute=True, device=device)
    wall = time.perf_counter() - t0
    st = res.device_stats["tier"]
    kat = benchmark_kat(res.report, n)
    link = st["h2d_bytes"] + st["d2h_bytes"] + st["zero_copy_bytes"]
    hl = host_link_peak()
    out = {"circuit": f"build_benchmark({n}) FP64, {2 ** n * 16 / 2 ** 30:.0f} GiB state on 1 B200",
           "config": {"fast_capacity_GiB": fast_gib, "chunk_GiB": chunk_gib},
           "hbm_fast_GiB": st["hbm_fast_bytes"] / 2 ** 30, "slow_GiB": res.tier_accounts[0].slow_bytes / 2 ** 30,
           "gates": len(circ.gates), "staging_groups": st["groups"], "wall_s": round(wall, 2),
           "setup_s": st["setup_seconds"], "run_s": st["run_seconds"],
           "sec_per_gate": round(st["run_seconds"] / len(circ.gates), 4),
           "model_tier_bytes": res.total_tier_bytes, "physical_link_bytes": link,
           "link_GBps": round(link / st["run_seconds"] / 1e9, 2),
           "link_peak_GBps": hl, "link_frac": round(link / st["run_seconds"] / 1e9 / hl, 3) if hl else None,
           "kat_parity_pattern": kat[0], "kat_max_dev": kat[1],
           "what": "run_circuit(tier_config=TierConfig(fast, chunk), tier_execute=True): reference staging "
                   "plan executed, slow chunks in pinned host memory, copy engines overlapped with passes"}
    del res
    return out


def host_link_peak() -> float | None:
    """Concurrent H2D + D2H copy bandwidth of 1 GiB pinned buffers (the tier's link)."""
    try:
        import torch
        h = torch.empty(2 << 30, dtype=torch.uint8, pin_memory=True)
        d = torch.empty(2 << 30, dtype=torch.uint8, device="cuda")
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        best = 0.0
        for _ in range(3):
            torch.cuda.synchronize()
            t = time.perf_counter()
            with torch.cuda.stream(s1):
                d[: 1 << 30].copy_(h[: 1 << 30], non_blocking=True)
            with torch.cuda.stream(s2):
                h[1 << 30:].copy_(d[1 << 30:], non_blocking=True)
            torch.cuda.synchronize()
            best = max(best, (2 << 30) / (time.perf_counter() - t) / 1e9)
        del h, d
        torch.cuda.empty_cache()
        return round(best, 1)
    except Exception:
        return None


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle.cpu_baseline import time_layers
    layers = workload_layers(CPU_SAMPLE_N, args.layers)
    seq = [layers[i % len(layers)] for i in range(args.warmup + args.steps)]
    res, threads = time_layers(seq, CPU_SAMPLE_N)
    timed = res[args.warmup:]
    secs = sum(r[0] for r in timed)
    byts = sum(r[1] for r in timed)
    gates = sum(r[2] for r in timed)
    val = byts / secs / 1e9
    line = {
        "metric": METRIC, "value": round(val, 4), "unit": "GB/s", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(secs / max(1, len(timed)) * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128 (f64)",
        "data": "synthetic", "sec_per_gate": secs / gates,
        "config": {"workload": f"C2 layers sampled at N={CPU_SAMPLE_N} (reference CPU path cannot hold "
                               f"N={args.n}: 128 GiB + copies)", "n_qubits": CPU_SAMPLE_N,
                   "layer_gates": CPU_SAMPLE_N, "precision": "fp64"},
        "cpu_baseline": {"value": round(val, 4), "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": f"{len(timed)} timed layers at N={CPU_SAMPLE_N}, numpy port of "
                                   f"svsim/kernels.py (oracle/), {threads} threads"},
        "e2e": {"value": round(val, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------------------------
def run_b200(args):
    rank, world, local = dist_env()
    dist = dist_init(world)
    import paper_2511_03359_b200 as pb
    from paper_2511_03359_b200 import _native as nat
    from paper_2511_03359_b200.device import DeviceState
    from paper_2511_03359_b200.engine import gate_to_op
    from tests.circuits import to_product
    from oracle.ref_builders import OCircuit

    device = local if world > 1 else 0
    if world > 1 and os.environ.get("SVB200_DEVICES"):     # test only: ranks share GPUs (rank % k)
        device = local % int(os.environ["SVB200_DEVICES"])
    nat.check(nat.load().sv_set_device(device))
    nat.check(nat.load().sv_fused_variant(args.fused))
    nat.check(nat.load().sv_fused_segment_limit(args.seg_limit))
    if world > 1:
        return run_b200_multi(args, dist, rank, world, device)
    n = args.n
    layers_o = workload_layers(n, args.layers)
    layers = [to_product(OCircuit(n, tuple(l))).gates for l in layers_o]
    lbytes = [layer_bytes(l, n) for l in layers_o]
    step_layers = [i % len(layers) for i in range(args.warmup + args.steps)]

    dev = DeviceState(n, pb.PrecisionMode.FP64, device=device)
    dev.zero(0)
    ops = [[gate_to_op(g) for g in layer] for layer in layers]
    # compile the specialised pass kernels of every layer before the warm-up (sv_jit.cu)
    from paper_2511_03359_b200.device import jit_prepare, jit_stats, jit_wait
    # --fuse-steps 1: the timed steps are submitted as ONE op list (the circuit they form),
    # so fused passes span layer boundaries as in run_circuit; 0: one apply per step
    warm_seq = [ops[i] for i in step_layers[:args.warmup]]
    timed_seq = [ops[i] for i in step_layers[args.warmup:]]
    if args.fuse_steps:
        warm_seq = [[o for lst in warm_seq for o in lst]]
        timed_seq = [[o for lst in timed_seq for o in lst]]
    t_jit = time.perf_counter()
    for o in warm_seq + timed_seq:
        jit_prepare(n, o, args.tile_bits)
    jit_wait()
    t_jit = time.perf_counter() - t_jit
    for o in warm_seq:
        dev.apply_fused(o, args.tile_bits)
    dev.synchronize()
    if dist is not None:
        dist.barrier()
    ev0, ev1 = nat.Event(), nat.Event()
    launches0 = nat.launch_count()
    nat.pass_timing(True)
    nat.pass_timing_read()
    with ClockSampler(device) as clk:
        ev0.record(dev.stream)
        for o in timed_seq:
            dev.apply_fused(o, args.tile_bits)
        ev1.record(dev.stream)
        dev.synchronize()
    nat.pass_timing(False)
    passes, pass_ms, pass_bytes = nat.pass_timing_read()
    launches = nat.launch_count() - launches0
    jit = jit_stats()
    ms = ev0.elapsed_ms(ev1)
    # parity of the timed region (outside it): the 128 GiB state after warm-up + timed steps is
    # still normalised (unitary layers), every Qz in [0, 1]
    norm_t, ones_t, _ = dev.measure()
    parity = {"norm_deviation_after_timed": abs(norm_t - 1.0),
              "qz_in_range": bool(all(-1e-12 <= z <= norm_t + 1e-12 for z in ones_t))}
    if dist is not None:
        dist.barrier()
    ms_max = max_over_ranks(dist, ms)
    timed_bytes = sum(lbytes[i] for i in step_layers[args.warmup:])
    timed_gates = sum(len(layers[i]) for i in step_layers[args.warmup:])
    total_bytes = sum_over_ranks(dist, timed_bytes)
    value = total_bytes / (ms_max / 1e3) / 1e9
    peak, peak_src = peaks()
    achieved = pass_bytes / (pass_ms / 1e3) / 1e9 if pass_ms > 0 else 0.0

    clk_mhz = clk.summary().get("sm_mhz") or 1965.0
    # single-gate streaming kernel (no fusion): the per-gate roofline the north star names
    single = {}
    if args.single_gate:
        h = pb.gates.H_MATRIX
        for q in (0, 1, n // 2, n - 1):
            e0, e1 = nat.Event(), nat.Event()
            dev.apply_1q(q, h)
            e0.record(dev.stream)
            for _ in range(3):
                dev.apply_1q(q, h)
            e1.record(dev.stream)
            t = e0.elapsed_ms(e1) / 3
            single[f"q{q}"] = {"ms": round(t, 3), "GB/s": round(2 * 16 * dev.size / (t / 1e3) / 1e9, 1)}
    dev.free()
    del dev
    if args.parity:
        parity.update(fused_parity(n_small=args.parity_n, device=device, tile_bits=args.tile_bits))

    # FP32 storage: same layers, complex64 at rest, FP64 arithmetic, one
    # rounding per gate -- timed like the FP64 steps
    fp32 = None
    if args.fp32:
        for o in warm_seq + timed_seq:
            jit_prepare(n, o, args.tile_bits, nat.SV_FP32)
        jit_wait()
        dev32 = DeviceState(n, pb.PrecisionMode.FP32, device=device)
        dev32.zero(0)
        for o in warm_seq:
            dev32.apply_fused(o, args.tile_bits)
        dev32.synchronize()
        nat.pass_timing(True)
        nat.pass_timing_read()
        f0, f1 = nat.Event(), nat.Event()
        f0.record(dev32.stream)
        for o in timed_seq:
            dev32.apply_fused(o, args.tile_bits)
        f1.record(dev32.stream)
        dev32.synchronize()
        nat.pass_timing(False)
        p32, ms32, by32 = nat.pass_timing_read()
        t32 = f0.elapsed_ms(f1)
        fp32 = {"ms_per_step": round(t32 / args.steps, 3),
                "value": round(sum(layer_bytes(layers_o[i], n, 8) for i in step_layers[args.warmup:]) /
                               (t32 / 1e3) / 1e9, 2),
                "unit": "GB/s", "pass_GBps": round(by32 / (ms32 / 1e3) / 1e9, 1) if ms32 > 0 else None,
                "passes_per_step": round(p32 / args.steps, 2),
                "what": "same C2 steps with complex64 storage (8 B/amplitude), FP64 arithmetic, one rounding "
                        "to float per gate (kernels.py:36-40); bound by the F2F conversions (~16/clk/SM)"}
        dev32.free()
        del dev32

    # end to end through the public API (host-built circuit in, report out)
    e2e = None
    if args.e2e_steps > 0:
        h2d0, d2h0 = nat.transfer_bytes()
        t_e2e = 0.0
        e2e_bytes = 0
        # warm e2e = a repeated call: every circuit runs once untimed first (its pass kernels
        # compiled then, as a second call in production finds them); the first call of a
        # fresh process is `cold_process` below
        # the C2 circuit through the public API: the Hadamard layer on |0..0>, one random layer,
        # measure-all (the Hadamard layer makes the state dense before the random layer)
        e2e_circs = []
        for j in range(args.e2e_steps):
            li = 1 + j % (len(layers) - 1) if len(layers) > 1 else 0
            e2e_circs.append((li, pb.Circuit(n, tuple(layers[0]) + tuple(layers[li]) + (pb.gates.measure_all(),))))
        for li, circ in {li: c for li, c in e2e_circs}.items():
            for track in (True, False):
                warm = pb.run_circuit(circ, device=device, tile_bits=args.tile_bits, track_support=track)
                del warm
            jit_wait()

        def e2e_pass(track):
            t_sum, b_sum, cl = 0.0, 0, []
            for li, circ in e2e_circs:
                t0 = time.perf_counter()
                res = pb.run_circuit(circ, device=device, tile_bits=args.tile_bits, track_support=track)
                _ = res.report.qz[0]
                dt = time.perf_counter() - t0
                t_sum += dt
                b_sum += lbytes[0] + lbytes[li]
                cl.append({"layers": [0, li], "s": round(dt, 4), "gates": len(circ.gates) - 1,
                           "launches": res.device_stats.get("kernel_launches")})
                del res
            return t_sum, b_sum, cl

        h2d0, d2h0 = nat.transfer_bytes()
        t_e2e, e2e_bytes, calls = e2e_pass(True)
        h2d1, d2h1 = nat.transfer_bytes()
        t_dense, dense_bytes, _ = e2e_pass(False)
        t_e2e = max_over_ranks(dist, t_e2e)
        t_dense = max_over_ranks(dist, t_dense)
        e2e = {"value": round(sum_over_ranks(dist, e2e_bytes) / t_e2e / 1e9, 2), "unit": "GB/s",
               "h2d_bytes_per_step": (h2d1 - h2d0) // args.e2e_steps,
               "d2h_bytes_per_step": (d2h1 - d2h0) // args.e2e_steps,
               "calls": calls,
               "dense": {"value": round(sum_over_ranks(dist, dense_bytes) / t_dense / 1e9, 2), "unit": "GB/s",
                         "what": "the same calls with track_support=False: every tile of every pass"},
               "what": "run_circuit(H layer + random layer + M) on |0..0>: allocate 2^N state, fused passes "
                       "(support tracking: the Hadamard layer's early passes read only the tiles that can be "
                       "nonzero), measure-all, report to host; wall clock per call"}

    # adder circuit time (BASELINE config 3: build_adder(16, [47302, 18233]), N=32 FP64, public API)
    adder = None
    if args.adder:
        circ, regs = pb.build_adder(16, [47302, 18233])
        pb.run_circuit(pb.build_adder(4, [3, 12])[0], device=device)          # warm the code paths
        t0 = time.perf_counter()
        res = pb.run_circuit(circ, device=device, tile_bits=args.tile_bits)
        t_first = time.perf_counter() - t0
        del res
        jit_wait()                       # the first run queued the adder's pass kernels
        t_adder = None
        for rep in range(3):             # warm calls (the fastest: a stray slab re-allocation or
            if rep:                      # first launch of a helper kernel is not the circuit)
                del res
            t0 = time.perf_counter()
            res = pb.run_circuit(circ, device=device, tile_bits=args.tile_bits)
            dt = time.perf_counter() - t0
            t_adder = dt if t_adder is None else min(t_adder, dt)
        kat = all(abs(res.report.qz[q] - 1.0) < 1e-12 for q in regs["R2"])
        rep_support = res.device_stats.get("support")
        rep_exact = res.report
        launches_a = res.device_stats.get("kernel_launches")
        del res
        a_ops = [gate_to_op(gt) for gt in circ.gates if gt.kind != "M"]

        def timed_passes(**kw):
            """(wall seconds of a warm run, pass count, pass ms of a further run, report)"""
            pb.run_circuit(circ, device=device, tile_bits=args.tile_bits, **kw)
            jit_wait()
            t = None
            for _ in range(2):   # the faster of two warm calls (a stray slab re-allocation)
                t0 = time.perf_counter()
                r = pb.run_circuit(circ, device=device, tile_bits=args.tile_bits, **kw)
                dt = time.perf_counter() - t0
                t = dt if t is None else min(t, dt)
                rep = r.report
                del r
            nat.pass_timing(True)
            nat.pass_timing_read()
            r = pb.run_circuit(circ, device=device, tile_bits=args.tile_bits, **kw)
            nat.pass_timing(False)
            cnt, ms, _ = nat.pass_timing_read()
            del r
            return t, cnt, ms, rep

        # support tracking on (the default): the passes' own CUDA-event time
        _, s_passes, s_ms, _ = timed_passes()
        # dense (track_support=False): every tile of every pass, the amount of work the
        # reference does; its passes against their max(HBM, FP64) floors
        t_dense, d_passes, d_ms, _ = timed_passes(track_support=False)
        d_roof = fp64_aware_roofline(32, [a_ops], args.tile_bits, d_ms, peak, clk_mhz)
        adder = {"circuit": "build_adder(16, [47302, 18233])", "n_qubits": 32, "gates": len(circ.gates),
                 "seconds": round(t_adder, 4), "sec_per_gate": round(t_adder / len(circ.gates), 6),
                 "first_run_seconds": round(t_first, 4),
                 "kat_all_ones_R2": kat, "kernel_launches": launches_a,
                 "support": rep_support,
                 "support_passes": {"count": s_passes, "ms": round(s_ms, 2)},
                 "dense_seconds": round(t_dense, 4),
                 "dense_passes": {"count": d_passes, "ms": round(d_ms, 2), "hbm_floor_ms": d_roof["hbm_floor_ms"],
                                  "fp64_floor_ms": d_roof["fp64_floor_ms"], "max_floor_ms": d_roof["max_floor_ms"],
                                  "frac_of_max_floor": d_roof["frac"],
                                  "fp64_per_amplitude": d_roof["fp64_per_amplitude"]},
                 "what": "run_circuit wall clock incl. allocation, |0..0>, fused passes, measure-all (fastest "
                         "of three warm runs: specialised pass kernels compiled; first_run_seconds: cold).  The adder's state "
                         "stays inside a 2^k-amplitude support (basis-state inputs, only one register "
                         "superposed), which run_circuit tracks: passes and measurement read only its tiles "
                         "(support_passes).  dense_*: track_support=False, every tile, with the passes' "
                         "max(HBM, FP64) floors"}
        # the same circuit with combined diagonal runs (exact_diagonals=False: within 1e-12 of
        # the reference, not bit-identical): one multiply per register mask per CPHASE run
        t_comb, _, _, rep_comb = timed_passes(exact_diagonals=False)
        tc_dense, c_passes, c_ms, _ = timed_passes(exact_diagonals=False, track_support=False)
        c_roof = fp64_aware_roofline(32, [a_ops], args.tile_bits, c_ms, peak, clk_mhz, combine_diag=True)
        adder["combined_diagonals"] = {
            "seconds": round(t_comb, 4), "dense_seconds": round(tc_dense, 4),
            "dense_passes": {"count": c_passes, "ms": round(c_ms, 2), "fp64_floor_ms": c_roof["fp64_floor_ms"],
                             "max_floor_ms": c_roof["max_floor_ms"], "frac_of_max_floor": c_roof["frac"]},
            "report_max_diff_vs_exact": float(rep_exact.max_difference(rep_comb)),
            "kat_all_ones_R2": all(abs(rep_comb.qz[q] - 1.0) < 1e-12 for q in regs["R2"]),
            "what": "run_circuit(exact_diagonals=False): runs of diagonal gates multiply each amplitude "
                    "by their combined factor (north-star FP64 tolerance 1e-12, not bit-identical)"}
    # byte-encoded benchmark (BASELINE config 5 shape on one GPU): time per gate
    byte = None
    if args.byte_n > 0:
        from paper_2511_03359_b200.byte_state import ByteEngineState
        from paper_2511_03359_b200.layout import PartitionLayout
        bc = pb.build_benchmark(args.byte_n)
        bst = ByteEngineState(args.byte_n, PartitionLayout(args.byte_n, args.byte_n), device=device)
        bst.zero(0)
        t0 = time.perf_counter()
        for gte in bc.gates[:-1]:
            bst.apply_gate(gte)
        bst.synchronize()
        t_gates = time.perf_counter() - t0
        bst.measure_sums()                  # first call: kernel attributes, scratch pool
        t0 = time.perf_counter()
        norm, ones_b, cross_b = bst.measure_sums()
        t_meas = time.perf_counter() - t0
        from paper_2511_03359_b200.measure import report_from_sums
        kat_b = benchmark_kat(report_from_sums(norm, ones_b, cross_b), args.byte_n, 1e-3, 0.05)
        kat_cb = benchmark_codebook_kat(bst.codebook, args.byte_n)
        ng = len(bc.gates) - 1
        byte = {"circuit": f"build_benchmark({args.byte_n}) BYTE", "gates": ng,
                "sec_per_gate": round(t_gates / ng, 5),
                "effective_GBps": round(ng * 4 * 2 ** args.byte_n / t_gates / 1e9, 1),
                "measure_s": round(t_meas, 4), "measure_note": "second call (warm)", "norm": norm,
                "passes": bst.passes,
                "kat_parity_pattern": kat_b[0], "kat_max_dev": kat_b[1], "kat_codebook": kat_cb,
                "codebook": [len(bst.codebook.mags), len(bst.codebook.thetas)],
                "what": "apply_gate wall clock (passes + per-gate codebook barrier), 4 B/amplitude/gate as if "
                        "dense; the state's support is tracked (byte_state.py), so the early Hadamard stages "
                        "visit only its items"}
        bst.free()
        del bst

    if e2e and args.cold_e2e:
        import gc
        from paper_2511_03359_b200.device import release_cached_memory
        gc.collect()                         # RunResult <-> state cycles still holding slabs
        release_cached_memory()              # the child process allocates its own 2^N state
        e2e["cold_process"] = cold_e2e(n, args.layers, device, args.tile_bits)

    tier = None
    if args.tier_n > 0 and world == 1:
        import gc
        from paper_2511_03359_b200.device import release_cached_memory
        gc.collect()
        release_cached_memory()
        tier = tier_run(args.tier_n, args.tier_fast_gib, args.tier_chunk_gib, device)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(max(1, args.cpu_layers), args.layers)

    clocks = clk.summary()
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128 (f64)",
            "data": "synthetic",
            "sec_per_gate": round(ms_max / 1e3 / timed_gates, 6),
            "config": {"workload": f"C2: H layer + random 1q/2q/diag layers (depth {n}), N={n} FP64 "
                                   f"per GPU, {2 ** n * 16 / 2 ** 30:.0f} GiB state",
                       "n_qubits_per_gpu": n, "n_qubits_total": n + (world.bit_length() - 1),
                       "gates_per_step": n, "layers": args.layers, "tile_bits": args.tile_bits,
                       "steps_fused": bool(args.fuse_steps),
                       "parallelism": "replicas" if world > 1 else "single",
                       "l2": "inputs (128 GiB) >> 126 MB L2; no flush needed"},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "peak_source": peak_src, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": measured_traffic(2 * 16 * 2 ** n)[0],
                         "traffic_source": measured_traffic(2 * 16 * 2 ** n)[1],
                         "kernel": {0: "k_fused<c64s,12>", 1: "k_fused3<12,4,1>", 2: "k_fused3<11,3,2>",
                                    3: "k_fused3<12,3,1>", 4: "k_fused3<11,3,3>",
                                    5: "k_fused3<10,3,4>", 6: "k_fused3<11,4,3>",
                                    7: "k_fused3<10,4,6>", 8: "k_fused3<12,4,2> single buffer",
                                    9: "auto: k_fused3<11,4,3> / <12,4,2> per op list",
                                    10: "<13,4,1> single buffer (specialised only)"}[args.fused] + (
                             " as sv_pass (NVRTC-specialised per pass structure)" if jit["jit_launches"] else ""),
                         "launches_timed": passes,
                         "bytes_per_launch": 2 * 16 * 2 ** n,
                         "fp64_aware": fp64_aware_roofline(n, timed_seq, args.tile_bits, pass_ms, peak,
                                                           clocks.get("sm_mhz") or 1965.0)},
            "gpu_launches": launches,
            "fused_passes_per_step": round(passes / args.steps, 2),
            "jit": dict(jit, prepare_seconds=round(t_jit, 2)),
            "clocks": clocks,
        }
        if single:
            line["single_gate_h"] = single
        if fp32:
            line["fp32"] = fp32
        if e2e:
            line["e2e"] = e2e
        if cpu:
            line["cpu_baseline"] = cpu
        if adder:
            line["adder"] = adder
        if byte:
            line["byte_mode"] = byte
        line["parity"] = parity
        if tier:
            line["host_tier"] = tier
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def nccl_probe(dist, rank, world, device, gib: int):
    """Baseline for the exchange kernels: NCCL send/recv of `gib` GiB between rank pairs
    (rank ^ 1) through torch.distributed (batch_isend_irecv, both directions at once).
    Wall clock around 3 synchronised rounds, max over ranks (NCCL runs on its own
    stream, so CUDA events on ours would not bracket it)."""
    import torch
    torch.cuda.set_device(device)
    grp = dist.new_group(backend="nccl")
    nbytes = gib << 30
    send = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{device}")
    recv = torch.empty_like(send)
    partner = rank ^ 1

    def round_trip():
        ops = [dist.P2POp(dist.isend, send, partner, group=grp), dist.P2POp(dist.irecv, recv, partner, group=grp)]
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    round_trip()
    torch.cuda.synchronize()
    dist.barrier()
    reps = 3
    t0 = time.perf_counter()
    for _ in range(reps):
        round_trip()
    torch.cuda.synchronize()
    t = max_over_ranks(dist, time.perf_counter() - t0)
    del send, recv
    torch.cuda.empty_cache()
    dist.destroy_process_group(grp)
    gbps = nbytes * reps / t / 1e9
    return {"what": f"NCCL send/recv {gib} GiB per direction between rank pairs (torch.distributed "
                    f"batch_isend_irecv), wall clock max over ranks", "GBps_per_direction": round(gbps, 1),
            "frac_of_770": round(gbps / 770.0, 4)}


def run_b200_multi(args, dist, rank, world, device):
    """Weak scaling: 2**n amplitudes per GPU, N = n + log2(P) qubits, remapped NVLink exchanges."""
    import paper_2511_03359_b200 as pb
    from paper_2511_03359_b200 import _native as nat
    from paper_2511_03359_b200.distributed import CudaBackend, phys_op
    from paper_2511_03359_b200.remap import RemapPlanner, Swap, SwapGroup
    from tests.circuits import to_product
    from oracle.ref_builders import OCircuit

    n = args.n
    N = n + (world.bit_length() - 1)
    layers_o = workload_layers(N, args.layers)
    layers = [to_product(OCircuit(N, tuple(l))).gates for l in layers_o]
    lbytes = [layer_bytes(l, N) for l in layers_o]
    seq = [i % len(layers) for i in range(args.warmup + args.steps)]
    flat, owner = [], []
    for k, li in enumerate(seq):
        flat += list(layers[li])
        owner += [k] * len(layers[li])
    steps = RemapPlanner(N, n).plan(flat)
    per_step = [[] for _ in seq]
    pending_swaps = []
    for st in steps:
        if isinstance(st, (Swap, SwapGroup)):
            pending_swaps.append(st)
        else:
            k = owner[st.ordinal]
            per_step[k] += pending_swaps + [st]
            pending_swaps = []
    # each step as launch batches: ("ops", [sv_op]) or ("swapops", pairs, after, before): a remap
    # swap with the ops before and after it -- the swap overlaps the last pass before it and
    # the first pass after it (chunked, inter-process events)
    batches = []
    for k in range(len(seq)):
        out, pend, swap, before = [], [], None, []
        for st in per_step[k]:
            if isinstance(st, (Swap, SwapGroup)):
                if swap is not None:
                    out.append(("swapops", swap, pend, before))
                    before = []
                else:
                    before = pend
                pend = []
                swap = ((st.global_pos, st.local_pos),) if isinstance(st, Swap) else st.pairs
            else:
                op = phys_op(st.gate, st.qubits, n, rank)
                if op is not None:
                    pend.append(op)
        if swap is not None:
            out.append(("swapops", swap, pend, before))
        elif pend:
            out.append(("ops", pend))
        batches.append(out)
    from paper_2511_03359_b200.device import jit_prepare, jit_stats, jit_wait
    t_jit = time.perf_counter()
    for out in batches:
        for b in out:
            if b[0] == "ops":
                jit_prepare(n, b[1], args.tile_bits)
            else:            # the overlapped passes are planned on their own op ranges
                first, rest = CudaBackend._first_pass(b[2])
                head, last = CudaBackend._last_pass(b[3])
                for part in (first, rest, head, last, b[2], b[3]):
                    jit_prepare(n, part, args.tile_bits)
    jit_wait()
    t_jit = time.perf_counter() - t_jit
    be = CudaBackend(dist, n, pb.PrecisionMode.FP64, device, args.tile_bits)

    def run_step(k):
        for b in batches[k]:
            if b[0] == "ops":
                be.apply_local(b[1])
            elif args.overlap:
                be.swap_then_apply(b[1], b[2], before=b[3])
            else:
                if b[3]:
                    be.apply_local(b[3])
                if len(b[1]) == 1:
                    be.swap(*b[1][0])
                else:
                    be.swap_group(b[1])
                if b[2]:
                    be.apply_local(b[2])

    for k in range(args.warmup):
        run_step(k)
    be.dev.synchronize()
    dist.barrier()
    ev0, ev1 = nat.Event(), nat.Event()
    launches0 = nat.launch_count()
    nat.pass_timing(True)
    nat.pass_timing_read()
    be.swap_timing = True
    link0 = be.link_bytes
    with ClockSampler(device) as clk:
        ev0.record(be.dev.stream)
        for k in range(args.warmup, args.warmup + args.steps):
            run_step(k)
        ev1.record(be.dev.stream)
        be.dev.synchronize()
    nat.pass_timing(False)
    passes, pass_ms, pass_bytes = nat.pass_timing_read()
    swap_ms = sum(a.elapsed_ms(b) for a, b in be.swap_events)
    n_swaps = len(be.swap_events)
    launches = nat.launch_count() - launches0
    ms = ev0.elapsed_ms(ev1)
    dist.barrier()
    ms_max = max_over_ranks(dist, ms)
    timed_gates = sum(len(layers[seq[k]]) for k in range(args.warmup, args.warmup + args.steps))
    total_bytes = sum(lbytes[seq[k]] for k in range(args.warmup, args.warmup + args.steps))
    value = total_bytes / (ms_max / 1e3) / 1e9
    peak, peak_src = peaks()
    achieved = pass_bytes / (pass_ms / 1e3) / 1e9 if pass_ms > 0 else 0.0
    per_dir = (be.dev.size // 2) * 16            # bytes into this GPU per swap (L/2 amplitudes)
    clocks = clk.summary()
    # exchange probe: global<->local swaps with every rank-bit partner (outside the timed step)
    be.swap_events = []
    for rep in range(2):
        for bit in range(world.bit_length() - 1):
            be.swap(n + bit, n - 1 - bit)
    probe_ms = [a.elapsed_ms(b) for a, b in be.swap_events]
    probe_ms_max = max_over_ranks(dist, max(probe_ms))
    nvlink = {"swaps_in_timed_steps": n_swaps, "swap_ms_in_timed_steps": round(swap_ms, 3),
              "overlapped_swaps": be.overlapped,
              "swap_ms_note": "with overlap, a swap's time includes the first pass after it",
              "probe_swaps": len(probe_ms), "probe_ms_per_swap_max": round(probe_ms_max, 3),
              "bytes_per_direction_per_swap": per_dir,
              "achieved_GBps_per_direction": round(per_dir / (probe_ms_max / 1e3) / 1e9, 1),
              "peak_GBps_per_direction": 770.0,
              "frac": round(per_dir / (probe_ms_max / 1e3) / 1e9 / 770.0, 4),
              "peak_source": "B200_PROFILING.md measured peer copy per direction (900 nominal)",
              "physical_link_bytes_this_rank_timed": be.link_bytes - link0 - 2 * len(probe_ms) * (be.dev.size // 4) * 16}
    be.close()
    be.dev.free()
    del be
    shared = int(os.environ.get("SVB200_DEVICES", "0") or 0)
    if args.nccl_probe_gib > 0 and not (0 < shared < world):   # (NCCL: one rank per GPU)
        nvlink["nccl_baseline"] = nccl_probe(dist, rank, world, device, args.nccl_probe_gib)
    # end to end through the public API: run_circuit_distributed(layer + M) per step
    e2e = None
    if args.e2e_steps > 0:
        from paper_2511_03359_b200.distributed import run_circuit_distributed
        h2d0, d2h0 = nat.transfer_bytes()
        t_e2e, e2e_bytes = 0.0, 0
        for j in range(args.e2e_steps):
            li = 1 + j % (len(layers) - 1) if len(layers) > 1 else 0
            # the 1-GPU line's e2e circuit: the Hadamard layer on |0..0> (the state dense from
            # there, whatever the support tracking skips before), one random layer, measure-all
            circ = pb.Circuit(N, tuple(layers[0]) + tuple(layers[li]) + (pb.gates.measure_all(),))
            dist.barrier()
            t0 = time.perf_counter()
            res = run_circuit_distributed(circ, dist, device=device, tile_bits=args.tile_bits)
            _ = res.report.qz[0]
            dist.barrier()
            t_e2e += time.perf_counter() - t0
            e2e_bytes += lbytes[0] + lbytes[li]
            res.backend.close()
            res.backend.dev.free()
            del res
        h2d1, d2h1 = nat.transfer_bytes()
        t_e2e = max_over_ranks(dist, t_e2e)
        e2e = {"value": round(e2e_bytes / t_e2e / 1e9, 2), "unit": "GB/s",
               "h2d_bytes_per_step": (h2d1 - h2d0) // args.e2e_steps,
               "d2h_bytes_per_step": (d2h1 - d2h0) // args.e2e_steps,
               "what": "run_circuit_distributed(H layer + layer + M) per step: allocate + zero + IPC map, "
                       "remapped layers, measure-all, report on every rank; wall clock max over ranks"}
    jit = jit_stats()
    # adder circuit (BASELINE config 3, N=32 FP64, strong scaling) through the public API
    adder = None
    if args.adder:
        from paper_2511_03359_b200.distributed import run_circuit_distributed
        circ, regs = pb.build_adder(16, [47302, 18233])
        times = []
        for rep in range(4):   # cold, then three warm runs (the fastest is reported)
            dist.barrier()
            t0 = time.perf_counter()
            res = run_circuit_distributed(circ, dist, device=device, tile_bits=args.tile_bits)
            kat = all(abs(res.report.qz[q] - 1.0) < 1e-12 for q in regs["R2"])
            dist.barrier()
            times.append(max_over_ranks(dist, time.perf_counter() - t0))
            stats = res.device_stats
            res.backend.close()
            res.backend.dev.free()
            del res
            jit_wait()
        adder = {"circuit": "build_adder(16, [47302, 18233])", "n_qubits": 32, "gates": len(circ.gates),
                 "seconds": round(min(times[1:]), 4), "first_run_seconds": round(times[0], 4),
                 "sec_per_gate": round(min(times[1:]) / len(circ.gates), 6), "kat_all_ones_R2": kat,
                 "swaps": stats.get("swaps"), "swap_groups": stats.get("swap_groups"),
                 "scaling": "strong (fixed N=32 over the GPUs)",
                 "what": "run_circuit_distributed wall clock, max over ranks (fastest of three warm runs: compiled kernels)"}
    # traffic optimizer A/B (BASELINE config 4 circuit): the remap planner vs the reference's
    # per-gate exchange choreography (exchange-fused P2P pair updates), same circuit
    planner_ab = None
    if args.planner_ab:
        from paper_2511_03359_b200.distributed import run_circuit_distributed
        bc = pb.build_benchmark(N)
        planner_ab = {"circuit": f"build_benchmark({N}) FP64"}
        for remap in (True, False):
            times = []
            for rep in range(3):     # first run compiles the pass kernels; best of the next two
                dist.barrier()
                t0 = time.perf_counter()
                res = run_circuit_distributed(bc, dist, device=device, remap=remap, tile_bits=args.tile_bits)
                _ = res.report.qz[0]
                dist.barrier()
                times.append(max_over_ranks(dist, time.perf_counter() - t0))
                st = res.device_stats
                kat = benchmark_kat(res.report, N)
                res.backend.close()
                res.backend.dev.free()
                del res
                jit_wait()
            t = min(times[1:])
            planner_ab["remap" if remap else "reference_choreography"] = {
                "seconds": round(t, 4), "physical_link_bytes_rank0": st.get("physical_link_bytes"),
                "swaps": st.get("swaps"), "swap_groups": st.get("swap_groups"),
                "kat_parity_pattern": kat[0], "kat_max_dev": kat[1]}
    byte = None
    if args.byte_n_multi > 0:
        from paper_2511_03359_b200.distributed import run_circuit_distributed
        NB = args.byte_n_multi + (world.bit_length() - 1)
        bc = pb.build_benchmark(NB)
        dist.barrier()
        t0 = time.perf_counter()
        res = run_circuit_distributed(bc, dist, mode=pb.PrecisionMode.BYTE, device=device)
        norm_dev = res.report.norm_deviation
        kat_b = benchmark_kat(res.report, NB, 1e-3, 0.05)
        kat_cb = benchmark_codebook_kat(res.codebook, NB)
        dist.barrier()
        t_b = max_over_ranks(dist, time.perf_counter() - t0)
        st_b = res.device_stats
        cb = [len(res.codebook.mags), len(res.codebook.thetas)]
        res.backend.close()
        res.backend.st.free()
        del res
        ng = len(bc.gates) - 1
        byte = {"circuit": f"build_benchmark({NB}) BYTE", "n_qubits": NB, "gates": ng,
                "seconds": round(t_b, 3), "sec_per_gate": round(t_b / ng, 5),
                "effective_GBps_per_gpu": round(ng * 4 * 2 ** args.byte_n_multi / t_b / 1e9, 1),
                "codebook": cb, "norm_deviation": norm_dev,
                "kat_parity_pattern": kat_b[0], "kat_max_dev": kat_b[1], "kat_codebook": kat_cb, "swaps": st_b.get("swaps"), "swap_groups": st_b.get("swap_groups"),
                "byte_passes": st_b.get("byte_passes"),
                "what": "run_circuit_distributed(mode=BYTE) wall clock incl. allocation, per-gate codebook "
                        "barrier across ranks, remapped byte-plane swaps, measure-all; max over ranks"}
    # BYTE-encoded QFT adder (BASELINE config 5's second circuit: build_adder(19, [374982, 149305])
    # at N=38 on 8 GPUs): the widest even N <= byte_n_multi + log2(P); known answer R2 = all ones
    byte_adder = None
    if args.byte_adder and args.byte_n_multi > 0:
        from paper_2511_03359_b200.distributed import run_circuit_distributed
        w = (args.byte_n_multi + (world.bit_length() - 1)) // 2
        a_, b_ = 374982 % (1 << w), 149305 % (1 << w)
        circ, regs = pb.build_adder(w, [a_, b_])
        dist.barrier()
        t0 = time.perf_counter()
        res = run_circuit_distributed(circ, dist, mode=pb.PrecisionMode.BYTE, device=device)
        qz = res.report.qz
        dist.barrier()
        t_a = max_over_ranks(dist, time.perf_counter() - t0)
        st_a = res.device_stats
        byte_adder = {"circuit": f"build_adder({w}, [{a_}, {b_}]) BYTE", "n_qubits": 2 * w, "gates": len(circ.gates),
                      "seconds": round(t_a, 3), "sec_per_gate": round(t_a / len(circ.gates), 5),
                      "kat_all_ones_R2": all(qz[q] > 0.5 for q in regs["R2"]),
                      "norm_deviation": res.report.norm_deviation,
                      "codebook": [len(res.codebook.mags), len(res.codebook.thetas)],
                      "byte_passes": st_a.get("byte_passes"), "byte_host_fixes": st_a.get("byte_host_fixes"),
                      "what": "run_circuit_distributed(mode=BYTE) wall clock, max over ranks; lossy like the "
                              "reference encoding (norm deviation), R2 read-out by Qz > 0.5"}
        res.backend.close()
        res.backend.st.free()
        del res
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128 (f64)",
            "data": "synthetic", "sec_per_gate": round(ms_max / 1e3 / timed_gates, 6),
            "config": {"workload": f"C2 layers on N={N} qubits FP64, 2^{n} amplitudes ({2 ** n * 16 / 2 ** 30:.0f} GiB) "
                                   f"per GPU, global qubits made local by the remap planner",
                       "n_qubits_per_gpu": n, "n_qubits_total": N, "gates_per_step": N, "layers": args.layers,
                       "parallelism": f"state-sharded x{world} (rank = top {world.bit_length() - 1} index bits)",
                       "l2": "inputs >> 126 MB L2; no flush needed"},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "peak_source": peak_src,
                         "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": measured_traffic(2 * 16 * 2 ** n)[0],
                         "traffic_source": measured_traffic(2 * 16 * 2 ** n)[1],
                         "kernel": "sv_pass (NVRTC-specialised fused pass; k_fused3 until compiled), rank 0",
                         "launches_timed": passes,
                         "bytes_per_launch": 2 * 16 * 2 ** n},
            "nvlink": nvlink,
            "gpu_launches": launches,
            "jit": dict(jit, prepare_seconds=round(t_jit, 2)),
            "clocks": clocks,
        }
        if e2e:
            line["e2e"] = e2e
        if adder:
            line["adder"] = adder
        if planner_ab:
            line["planner_ab"] = planner_ab
        if byte:
            line["byte_mode"] = byte
        if byte_adder:
            line["byte_adder"] = byte_adder
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", "--qubits-per-gpu", dest="n", type=int, default=33, help="qubits per GPU")
    ap.add_argument("--layers", type=int, default=9, help="H layer + random layers in the workload")
    ap.add_argument("--tile-bits", type=int, default=12, help="v1 tile bits / upper bound")
    ap.add_argument("--fused", type=int, default=9, choices=[0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11],
                    help="fused-pass kernel: 0 smem-per-gate v1, 1-3 register-resident v3 configs")
    ap.add_argument("--seg-limit", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=4)
    ap.add_argument("--cpu-layers", type=int, default=6)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--adder", type=int, default=1, help="time the N=32 adder circuit (1 GPU line)")
    ap.add_argument("--byte-n", type=int, default=32, help="BYTE benchmark size for the 1 GPU line (0: skip)")
    ap.add_argument("--nccl-probe-gib", type=int, default=4,
                    help="N>1: NCCL send/recv baseline next to the P2P swap kernel (0: skip)")
    ap.add_argument("--byte-n-multi", type=int, default=35,
                    help="BYTE benchmark amplitudes per GPU (2^n) for N>1 lines: N = n + log2(P), "
                         "38 qubits on 8 GPUs = BASELINE config 5 (0: skip)")
    ap.add_argument("--single-gate", type=int, default=1)
    ap.add_argument("--overlap", type=int, default=1,
                    help="N>1: overlap each remap swap with the first pass after it (chunked, IPC events)")
    ap.add_argument("--byte-adder", type=int, default=1,
                    help="N>1: the BYTE-encoded adder at 2w <= byte_n_multi + log2(P) qubits (38 on 8 GPUs)")
    ap.add_argument("--planner-ab", type=int, default=1,
                    help="N>1: benchmark(N) with the remap planner vs the reference choreography")
    ap.add_argument("--fp32", type=int, default=1, help="1 GPU line: time the same steps in FP32 storage")
    ap.add_argument("--fuse-steps", type=int, default=1,
                    help="submit the timed steps as one op list (passes span layer boundaries)")
    ap.add_argument("--parity", type=int, default=1, help="1 GPU line: fused vs per-gate and oracle checks")
    ap.add_argument("--parity-n", type=int, default=26)
    ap.add_argument("--cold-e2e", type=int, default=1, help="1 GPU line: e2e of a fresh process")
    ap.add_argument("--tier-n", type=int, default=34, help="1 GPU line: host-memory tier run size (0: skip)")
    ap.add_argument("--tier-fast-gib", type=float, default=168.0)
    ap.add_argument("--tier-chunk-gib", type=float, default=4.0)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
