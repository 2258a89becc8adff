"""CPU-only: print / compile the specialised source of one fused pass of the C2 bench
layers (the library's own split) and summarise its SASS.

    python tools/jit_dump.py N LAYER PASS [cfg=8] [out_dir=/tmp/jitdump]

Writes <out>/pass.cu (the generated source), compiles it with nvcc for sm_100a against
the package headers and prints registers, spills and an opcode histogram (UBLKCP,
SYNCS, LDGSTS, LDS, STS, DFMA, ...).
"""
import collections
import ctypes
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2511_03359_b200 import _native as nat  # noqa: E402
from paper_2511_03359_b200.device import ops_array  # noqa: E402
from paper_2511_03359_b200.engine import gate_to_op  # noqa: E402
from oracle.ref_builders import OCircuit  # noqa: E402
from tests.circuits import to_product  # noqa: E402

n, li, pi = (int(x) for x in sys.argv[1:4])
cfg = int(sys.argv[4]) if len(sys.argv) > 4 else 8
out = sys.argv[5] if len(sys.argv) > 5 else "/tmp/jitdump"
os.makedirs(out, exist_ok=True)
lib = nat.load(require_device=False)
if li < 0:     # LAYER -1: build_adder(N // 2, ...) (BASELINE config 3 at N=32)
    import paper_2511_03359_b200 as pb
    circ = pb.build_adder(n // 2, [47302 % (1 << (n // 2)), 18233 % (1 << (n // 2))])[0]
    ops = [gate_to_op(g) for g in circ.gates if g.kind != "M"]
else:
    lay = bench.workload_layers(n, 9)[li]
    ops = [gate_to_op(g) for g in to_product(OCircuit(n, tuple(lay))).gates]
nat.check(lib.sv_fused_variant(cfg))
ends = (ctypes.c_int * 256)()
k = lib.sv_plan_passes(n, nat.SV_FP64, ops_array(ops), len(ops), 12, ends, 256)
ends = [ends[i] for i in range(k)]
print("passes:", len(ends), "ends:", ends)
a = 0 if pi == 0 else ends[pi - 1]
sub = ops[a:ends[pi]]
os.environ["SVB200_PROBE_CFG"] = str(cfg)
buf = ctypes.create_string_buffer(1 << 22)
rc = lib.sv_jit_probe(ops_array(sub), len(sub), n, buf, len(buf), None)
assert rc >= 1, lib.sv_last_error()
src = buf.value.decode()
path = os.path.join(out, "pass.cu")
with open(path, "w") as f:
    f.write(src)
inc = os.path.join(ROOT, "paper_2511_03359_b200", "csrc")
cubin = os.path.join(out, "pass.cubin")
r = subprocess.run(["nvcc", "-cubin", "-gencode", "arch=compute_100a,code=sm_100a", "-std=c++17", "-lineinfo",
                    "-Xptxas", "-v", "-I", inc, "-o", cubin, path], capture_output=True, text=True)
print(r.stderr.strip()[-600:])
if r.returncode:
    sys.exit(1)
sass = subprocess.run(["cuobjdump", "-sass", cubin], capture_output=True, text=True).stdout
ops_hist = collections.Counter()
for ln in sass.splitlines():
    m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", ln)
    if m:
        ops_hist[m.group(1)] += 1
with open(os.path.join(out, "pass.sass"), "w") as f:
    f.write(sass)
print(f"N={n} layer {li} pass {pi} cfg {cfg}: {len(sub)} ops, {sum(ops_hist.values())} SASS instructions")
keys = ["UBLKCP", "SYNCS", "LDGSTS", "LDS", "STS", "STG", "LDG", "LDC", "DFMA", "DMUL", "DADD", "BAR", "BRA"]
print({kk: ops_hist.get(kk, 0) for kk in keys})
print(ops_hist.most_common(25))
print("model FP64/amp:", sum(bench.fp64_ops_per_amplitude(o) for o in sub),
      "SASS FP64/amp:", (ops_hist["DFMA"] + ops_hist["DMUL"] + ops_hist["DADD"]) / 16)
print("kinds:", [({1: "1q", 2: "2q"}.get(o.kind, "diag"), bench.fp64_ops_per_amplitude(o)) for o in sub])
