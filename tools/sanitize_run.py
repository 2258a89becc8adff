"""Small workload for compute-sanitizer (racecheck / synccheck / memcheck / initcheck).

    compute-sanitizer --tool racecheck python tools/sanitize_run.py

Covers every kernel family of the hot path at N <= 16, each result checked
against the oracle so a sanitizer run is also a parity run:
  * specialised fused passes (NVRTC, compile-and-wait) in both tile
    configurations -- config 6 (2^11 double-buffered tiles) and config 8 (2^12
    single-buffer tiles whose next cp.async starts right after the last
    segment's register read, sv_jit.cu) -- plus the generic k_fused3;
  * FP32 storage passes, streaming 1q/2q/diagonal kernels;
  * k_measure3 (measure-all);
  * BYTE: k_byte_gate with its CAS-published shared-memory memo (<-1> and the
    <qa> 32-byte item variants), the diagonal code-table passes.
"""
import os
import sys

os.environ.setdefault("SVB200_JIT", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2511_03359_b200 as pb  # noqa: E402
from paper_2511_03359_b200 import _native as nat  # noqa: E402
from oracle import ref_engine  # noqa: E402
from oracle.ref_builders import adder, benchmark  # noqa: E402
from tests.circuits import random_circuit, to_product  # noqa: E402


def fp_case(name, circ, mode="fp64", ranks=1):
    pm = {"fp64": pb.PrecisionMode.FP64, "fp32": pb.PrecisionMode.FP32}[mode]
    got = pb.run_circuit(to_product(circ), ranks=ranks, mode=pm)
    want = ref_engine.run_circuit(circ, ranks=ranks, mode=mode)
    ok = np.array_equal(got.gathered_state(), want.gathered_state())
    print(f"{name} [{mode}] bit-exact={ok}", flush=True)
    return ok


def byte_case(name, circ, ranks=1):
    got = pb.run_circuit(to_product(circ), ranks=ranks, mode=pb.PrecisionMode.BYTE)
    want = ref_engine.run_circuit(circ, ranks=ranks, mode="be")
    mags = np.concatenate([s.mag_idx for s in got.states])
    phs = np.concatenate([s.phase_idx for s in got.states])
    ok = np.array_equal(mags, want.mag) and np.array_equal(phs, want.phase) and \
        got.codebook.dump() == want.codebook.dump()
    print(f"{name} [be] bytes bit-exact={ok}", flush=True)
    return ok


def main():
    lib = nat.load()
    ok = True
    for cfg in (6, 8, 3):       # 2^11 double-buffered, 2^12 single-buffered, generic 2^12
        nat.check(lib.sv_fused_variant(cfg))
        ok &= fp_case(f"random16 cfg{cfg}", random_circuit(np.random.default_rng(40 + cfg), 16, 60))
        ok &= fp_case(f"adder7 cfg{cfg}", adder(7, [100, 27])[0])
    nat.check(lib.sv_fused_variant(9))
    ok &= fp_case("random15", random_circuit(np.random.default_rng(3), 15, 50), "fp32")
    ok &= fp_case("bench14 ranks4", benchmark(14), ranks=4)
    ok &= byte_case("bench12", benchmark(12), ranks=2)
    ok &= byte_case("random10", random_circuit(np.random.default_rng(6), 10, 30))
    ok &= byte_case("adder5", adder(5, [20, 9])[0])
    # streaming kernels through the array API
    rng = np.random.default_rng(1)
    psi = (rng.standard_normal(1 << 14) + 1j * rng.standard_normal(1 << 14)).astype(np.complex128)
    from oracle import ref_kernels
    from paper_2511_03359_b200 import gates, kernels
    for q in (0, 3, 9, 13):
        a, b = psi.copy(), psi.copy()
        kernels.apply_single(a, q, gates.H_MATRIX)
        ref_kernels.gate1(b, q, gates.H_MATRIX)
        ok &= np.array_equal(a, b)
    print("streaming kernels bit-exact", ok, flush=True)
    print("SANITIZE_RUN", "OK" if ok else "MISMATCH", flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
