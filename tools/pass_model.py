"""Where the C2 step time goes: every fused pass of the bench layers, timed alone, next to
its three floors -- HBM (2 x 16 x 2^N bytes at the measured copy peak), FP64 (the pass's
FP64 instructions at 64 lanes/SM/clk) and shared memory (segment transposes at 128 B/clk/SM).

    python tools/pass_model.py [N] [cfg: 6 | 8 | 9=auto]

Pass split = the library's own planner (sv_plan_passes), per layer; cfg 9 replays the
auto choice per layer (config 8 when 2^12 tiles save a pass over 2^11).
FP64 instructions per amplitude (numpy-exact arithmetic, sv_arith.cuh): generic 1Q 10,
real 1Q (H) 6, monomial 0, generic 2Q 22, real 2Q 14, diagonal 4 x (active fraction),
Z 0.
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2511_03359_b200 as pb  # noqa: E402
from paper_2511_03359_b200 import _native as nat  # noqa: E402
from paper_2511_03359_b200.device import DeviceState, jit_prepare, jit_wait, ops_array  # noqa: E402
from paper_2511_03359_b200.engine import gate_to_op  # noqa: E402
from oracle.ref_builders import OCircuit  # noqa: E402
from tests.circuits import to_product  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 33
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 9
lib = nat.load()
peak = bench.peaks()[0]
sms = ctypes.c_int(0)
lib.sv_sm_count(0, ctypes.byref(sms))


def fp64_per_amp(op):
    m = np.array(op.m[:32])
    if op.kind == nat.SV_OP_1Q:
        mm = m[:8]
        nz = np.count_nonzero(mm.reshape(4, 2), axis=1)
        if all(c <= 1 for c in nz) and np.count_nonzero(mm) == 2:
            return 0.0
        return 6.0 if not np.any(mm[1::2]) else 10.0
    if op.kind == nat.SV_OP_2Q:
        mm = m[:32]
        if np.count_nonzero(mm) == 4:
            return 0.0
        return 14.0 if not np.any(mm[1::2]) else 22.0
    if op.m[0] == -1.0 and op.m[1] == 0.0:
        return 0.0
    return 4.0 / (1 << bin(op.diag_mask).count("1"))


TB = 13 if cfg == 10 else 12   # tile-bits cap handed to the library (config 10: 2^13 tiles)


def plan(ops):
    ends = (ctypes.c_int * 256)()
    k = lib.sv_plan_passes(n, nat.SV_FP64, ops_array(ops), len(ops), TB, ends, 256)
    nat.check(min(k, 0))
    out, a = [], 0
    for i in range(k):
        out.append((a, ends[i]))
        a = ends[i]
    return out


layers = [to_product(OCircuit(n, tuple(lo))).gates for lo in bench.workload_layers(n, 9)]
dev = DeviceState(n, pb.PrecisionMode.FP64)
dev.zero(0)
rows = []
clk = bench.ClockSampler(0)
with clk:
    for li, gates in enumerate(layers):
        ops = [gate_to_op(g) for g in gates]
        nat.check(lib.sv_fused_variant(cfg))
        passes = plan(ops)
        if cfg == 9:   # replay the auto choice for the sub-lists
            nat.check(lib.sv_fused_variant(6))
            p6 = len(plan(ops))
            nat.check(lib.sv_fused_variant(8))
            p8 = len(plan(ops))
            use = 8 if p8 < p6 else 6
        else:
            use = cfg
        nat.check(lib.sv_fused_variant(use))
        passes = plan(ops)
        for pi, (a, b) in enumerate(passes):
            sub = ops[a:b]
            jit_prepare(n, sub, TB)
            jit_wait()
            dev.apply_fused(sub, TB)
            dev.synchronize()
            nat.pass_timing(True)
            nat.pass_timing_read()
            for _ in range(3):
                dev.apply_fused(sub, TB)
            dev.synchronize()
            cnt, ms, by = nat.pass_timing_read()
            nat.pass_timing(False)
            ms /= max(cnt, 1)
            f64 = sum(fp64_per_amp(o) for o in sub)
            hbm_ms = 2 * 16 * 2 ** n / (peak * 1e9) * 1e3
            rows.append({"layer": li, "pass": pi, "cfg": use, "ops": b - a, "launches": cnt, "ms": round(ms, 2),
                         "hbm_floor_ms": round(hbm_ms, 2), "fp64_per_amp": f64,
                         "frac": round(hbm_ms / ms, 3)})
clocks = clk.summary()
for r in rows:
    print(json.dumps(r), flush=True)
tot = sum(r["ms"] for r in rows)
hb = sum(r["hbm_floor_ms"] for r in rows)
print(json.dumps({"passes": len(rows), "total_ms": round(tot, 1), "hbm_floor_ms": round(hb, 1),
                  "frac": round(hb / tot, 3), "clocks": clocks, "sms": sms.value}))
