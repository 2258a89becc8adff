"""CPU oracle for the gate-application hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in plain numpy, the algorithm of the reference
package ``svsim`` (``/root/reference/pkg/src/svsim``) for the hot path the
B200 build replaces: strided 2x2 / 4x4 / diagonal gate kernels, the adaptive
two-byte polar codebook, partition layout + exchange planning + traffic
ledgers, the bulk-synchronous per-gate engine (FP64 / FP32 / BYTE, any power
of two in-process ranks), the all-qubit three-axis measurement, the static
relabel optimizer and the workload builders.  Every function cites the
reference file:line it follows.

Rules:
  * Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
    ``cpu_baseline`` / ``--impl reference`` leg may import this package, and
    only as the checker or the timed CPU baseline — never as the thing
    measured or shipped.  The product package ``paper_2511_03359_b200`` never
    imports it.
  * The restatement is pinned against golden vectors produced by the real
    reference in this container (``tests/golden/make_golden.py`` →
    ``tests/golden/*.npz``), see ``tests/test_oracle_golden.py``.
  * Arithmetic is numpy's, with the same operand order as the reference, so
    results are bit-identical to the reference on the same host.
"""
from . import ref_builders, ref_codec, ref_engine, ref_gates, ref_kernels, ref_layout, ref_optimize

__all__ = ["ref_builders", "ref_codec", "ref_engine", "ref_gates", "ref_kernels",
           "ref_layout", "ref_optimize"]
