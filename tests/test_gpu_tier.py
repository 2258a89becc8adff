"""GPU tests of run_circuit(tier_config=...) (svsim/tier.py on the B200).

Two levels:
  * the reference's numbers: for every golden case the reference ran
    (tests/golden/tier.json `run`), the product's run charges the same tier ledgers
    and high-water marks and ends in the same state (digest), resident in HBM;
  * the plan EXECUTED (tier_execute=True, csrc/sv_tier.cu): slow chunks in pinned
    host memory staged through HBM slots -- bit-identical states and reports, the
    same ledgers, and physical host-link bytes bounded by the model's.
"""
import json
import os

import numpy as np
import pytest

import paper_2511_03359_b200 as pb
from paper_2511_03359_b200.tier import TierConfig
from tests.circuits import exact_class_circuit, random_circuit, to_product
from tests.test_gpu_ladder import state_digest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
MODES = {"fp64": pb.PrecisionMode.FP64, "fp32": pb.PrecisionMode.FP32, "be": pb.PrecisionMode.BYTE}


def _golden_runs():
    """(case, circuit, execute): every golden run resident; executed physically too where
    the executor applies (FP storage, chunks of at least 32 amplitudes)."""
    from tests.golden.make_golden import tier_cases
    circs = {name: circ for name, circ, *_ in tier_cases()}
    with open(os.path.join(HERE, "golden", "tier.json")) as f:
        cases = [c for c in json.load(f)["cases"] if "run" in c]
    out = []
    for c in cases:
        out.append(pytest.param(c, circs[c["name"]], False, id=c["name"] + "-resident"))
        if c["mode"] != "be" and c["chunk_qubits"] >= 5:
            out.append(pytest.param(c, circs[c["name"]], True, id=c["name"] + "-executed"))
    return out


@pytest.mark.parametrize("case,circ,execute", _golden_runs())
def test_tiered_run_matches_reference(case, circ, execute):
    mode = MODES[case["mode"]]
    cfg = TierConfig(*case["config"])
    res = pb.run_circuit(to_product(circ), ranks=case["run"]["ranks"], mode=mode, tier_config=cfg,
                         tier_execute=execute)
    assert state_digest(res.gathered_state()) == case["run"]["state_sha256"]
    assert [led.snapshot() for led in res.ledgers] == case["run"]["ledgers"]
    assert [a.high_water_bytes for a in res.tier_accounts] == case["run"]["high_water"]
    assert res.device_stats["tier"]["executed"] is execute
    if execute:
        st = res.device_stats["tier"]
        chunk = 1 << case["chunk_qubits"]
        chunk_bytes = chunk * mode.bytes_per_element
        model = res.total_tier_bytes
        physical = st["h2d_bytes"] + st["d2h_bytes"] + st["slot_memsets"] * chunk_bytes
        assert physical <= model and (physical > 0) == (model > 0)


def _physical_cases():
    rng = lambda s: np.random.default_rng(900 + s)  # noqa: E731
    return [
        ("random14", random_circuit(rng(1), 14, 60), 1, "fp64", 8),
        ("random14_r4", random_circuit(rng(2), 14, 60), 4, "fp64", 7),
        ("exact13", exact_class_circuit(rng(3), 13, 50), 2, "fp64", 6),
        ("random13_fp32", random_circuit(rng(4), 13, 50), 1, "fp32", 6),
        ("bench15", pb.build_benchmark(15), 1, "fp64", 9),
        ("adder7", pb.build_adder(7, [100, 27])[0], 1, "fp64", 8),
    ]


@pytest.mark.parametrize("name,circ,ranks,mode,c", _physical_cases(), ids=lambda v: v if isinstance(v, str) else "")
def test_executed_plan_is_bit_identical_to_resident_run(name, circ, ranks, mode, c):
    """The physical two-tier run (pair / quad / pair2q chunk kernels, run-group passes per
    chunk, zero-copy cross terms) against the same circuit resident in HBM and the oracle."""
    from oracle import ref_engine
    circ = circ if isinstance(circ, pb.Circuit) else to_product(circ)
    m = MODES[mode]
    n_local = circ.n_qubits - (ranks.bit_length() - 1)
    chunk_bytes = (1 << c) * m.bytes_per_element
    state_bytes = (1 << n_local) * m.bytes_per_element
    cfg = TierConfig(state_bytes // 2, chunk_bytes)
    plain = pb.run_circuit(circ, ranks=ranks, mode=m)
    tiered = pb.run_circuit(circ, ranks=ranks, mode=m, tier_config=cfg, tier_execute=True)
    a, b = plain.gathered_state(), tiered.gathered_state()
    assert np.array_equal(a, b)
    assert plain.report.max_difference(tiered.report) < 1e-12
    assert [l.inter_rank_bytes_sent for l in plain.ledgers] == [l.inter_rank_bytes_sent for l in tiered.ledgers]
    assert tiered.total_tier_bytes > 0
    st = tiered.device_stats["tier"]
    assert st["d2h_bytes"] > 0 and st["hbm_fast_bytes"] > 0
    if name == "random14":
        from tests.circuits import random_circuit as rc
        want = ref_engine.run_circuit(rc(np.random.default_rng(901), 14, 60), ranks=1)
        assert np.array_equal(b, want.gathered_state())
