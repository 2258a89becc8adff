"""Per-pass detail of the C2 bench layers: replays fused_impl's greedy pass split
(sv_capi.cu) in Python, runs every pass on its own and prints its op mix,
register segments and time (one row per pass)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_03359_b200 as pb
from paper_2511_03359_b200 import _native as nat
from paper_2511_03359_b200.device import DeviceState
from paper_2511_03359_b200.engine import gate_to_op
from tests.circuits import to_product
from oracle.ref_builders import OCircuit
import bench

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
only = tuple(int(x) for x in sys.argv[2].split(",")) if len(sys.argv) > 2 and sys.argv[2] != "all" else None   # "layer,pass"
K, RB = 11, 4


def split(ops):
    passes, cur, qm = [], [], 0
    low = (1 << 5) - 1
    for o in ops:
        need = 0
        if o.kind == nat.SV_OP_1Q:
            need = 1 << o.qa
        elif o.kind == nat.SV_OP_2Q:
            need = (1 << o.qa) | (1 << o.qb)
        if bin(qm | need | low).count("1") > K or len(cur) >= 128:
            passes.append(cur)
            cur, qm = [], 0
        cur.append(o)
        qm |= need
    passes.append(cur)
    return passes


def segments(ops):
    tq = set()
    for o in ops:
        if o.kind == nat.SV_OP_1Q:
            tq.add(o.qa)
        elif o.kind == nat.SV_OP_2Q:
            tq |= {o.qa, o.qb}
    segs, cur = 1, set()
    for o in ops:
        need = {o.qa} if o.kind == nat.SV_OP_1Q else ({o.qa, o.qb} if o.kind == nat.SV_OP_2Q else set())
        if len(cur | need) > RB:
            segs += 1
            cur = set()
        cur |= need
    return segs


if len(sys.argv) > 3 and sys.argv[3] == "adder":
    w = n // 2
    circ, _ = pb.build_adder(w, [47302 % (1 << w), 18233 % (1 << w)])
    layers_p = [tuple(g for g in circ.gates if g.kind != "M")]
else:
    layers_p = [to_product(OCircuit(n, tuple(lo))).gates for lo in bench.workload_layers(n, 4)]
nat.check(nat.load().sv_fused_variant(int(os.environ.get("SVB200_FUSED_CFG", "6"))))
dev = DeviceState(n, pb.PrecisionMode.FP64)
dev.zero(0)
for li, gates in enumerate(layers_p):
    for pi, ops in enumerate(split([gate_to_op(g) for g in gates])):
        if only is not None and (li, pi) != only:
            continue
        dev.apply_fused(ops)               # warm-up (compiles the specialised kernel in JIT mode 1)
        dev.synchronize()
        nat.load().sv_jit_wait()
        nat.pass_timing(True)
        nat.pass_timing_read()
        for rep in range(3):
            dev.apply_fused(ops)
        dev.synchronize()
        p, ms, by = nat.pass_timing_read()
        nat.pass_timing(False)
        kinds = {}
        for o in ops:
            key = {nat.SV_OP_1Q: "1q", nat.SV_OP_2Q: "2q"}.get(o.kind, "diag")
            kinds[key] = kinds.get(key, 0) + 1
        print(f"layer {li} pass {pi}: launches={p} ops={len(ops)} {kinds} segs={segments(ops)} "
              f"ms={ms / p:.2f} GB/s={by / (ms / 1e3) / 1e9:.0f}", flush=True)
    # gate kinds of the layer
    kc = {}
    for g in gates:
        kc[g.kind] = kc.get(g.kind, 0) + 1
    print(f"layer {li}: {kc}", flush=True)
