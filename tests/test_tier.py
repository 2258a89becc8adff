"""CPU tests of the two-tier staging model (paper_2511_03359_b200/tier.py) against the
REAL reference's outputs (tests/golden/tier.json, written by
`tests/golden/make_golden.py --tier` from svsim/tier.py): plan groups, chunk residency,
high-water marks, ledger counters, the naive per-gate baseline, validation messages."""
import json
import os

import pytest

import paper_2511_03359_b200 as pb
from paper_2511_03359_b200 import gates as g
from paper_2511_03359_b200.layout import TrafficLedger
from paper_2511_03359_b200.tier import (TierAccount, TierConfig, naive_staging_bytes, plan_passes,
                                        recommended_fast_bytes)
from tests.circuits import to_product

HERE = os.path.dirname(os.path.abspath(__file__))
MODES = {"fp64": pb.PrecisionMode.FP64, "fp32": pb.PrecisionMode.FP32, "be": pb.PrecisionMode.BYTE}


def _golden():
    with open(os.path.join(HERE, "golden", "tier.json")) as f:
        return json.load(f)


def _circuits():
    from tests.golden.make_golden import tier_cases
    return {name: circ for name, circ, *_ in tier_cases()}


@pytest.mark.parametrize("case", _golden()["cases"], ids=lambda c: c["name"])
def test_plan_and_account_match_reference(case):
    circ = to_product(_circuits()[case["name"]])
    cfg = TierConfig(*case["config"])
    mode = MODES[case["mode"]]
    plan = plan_passes(circ.gates, cfg, case["n_local"], mode)
    assert (plan.chunk_qubits, plan.n_chunks) == (case["chunk_qubits"], case["n_chunks"])
    got = [[grp.kind, list(grp.gate_indices), [list(m) for m in grp.chunk_groups]] for grp in plan.groups]
    assert got == case["groups"]
    assert len(plan.passes()) == case["n_passes"]
    led = TrafficLedger()
    acct = TierAccount(mode.bytes_per_element << case["n_local"], cfg, led)
    assert acct.fast_resident == case["fast_resident"]
    assert acct.static_fast_bytes == case["static_fast_bytes"] and acct.slow_bytes == case["slow_bytes"]
    for grp in plan.groups:
        acct.account(grp)
    assert acct.high_water_bytes == case["high_water_bytes"]
    assert (led.tier_bytes_moved, led.tier_transfer_count) == (case["tier_bytes"], case["tier_transfers"])
    assert naive_staging_bytes(circ.gates, cfg, case["n_local"], mode) == case["naive"]
    assert led.tier_bytes_moved <= case["naive"]


def test_validation_messages_match_reference():
    for args, msg in _golden()["errors"]:
        if args == "quad_tight":
            with pytest.raises(ValueError) as exc:
                plan_passes((g.u4(2, 3, g.CNOT_MATRIX),), TierConfig(2 * 64, 64), 6, pb.PrecisionMode.FP64)
        else:
            with pytest.raises(ValueError) as exc:
                TierConfig(*args)
        assert str(exc.value) == msg


def test_recommended_fast_bytes_matches_reference():
    for sb, cb, want in _golden()["recommended"]:
        assert recommended_fast_bytes(sb, cb) == want


def test_lookahead_window_splits_runs():
    plan = plan_passes(tuple(g.h(i % 2) for i in range(10)), TierConfig(4096, 256, lookahead_window=4), 8,
                       pb.PrecisionMode.FP64)
    assert [len(grp.gate_indices) for grp in plan.groups] == [4, 4, 2]


def test_run_circuit_charges_the_reference_tier_ledgers_without_a_device(monkeypatch):
    """The ledger side of run_circuit(tier_config=...) is pure host logic: the same
    staging plan and counters as the reference's run (golden `run` entries)."""
    from paper_2511_03359_b200.engine import tier_ledger_plan
    cases = [c for c in _golden()["cases"] if "run" in c]
    assert cases
    for case in cases:
        circ = to_product(_circuits()[case["name"]])
        P = case["run"]["ranks"]
        layout = pb.PartitionLayout(circ.n_qubits, case["n_local"])
        ledgers = [TrafficLedger() for _ in range(P)]
        plan, accounts = tier_ledger_plan(circ, layout, MODES[case["mode"]], TierConfig(*case["config"]), ledgers)
        for grp in plan.groups:
            for a in accounts:
                a.account(grp)
        want = case["run"]["ledgers"]
        assert [led.tier_bytes_moved for led in ledgers] == [w["tier_bytes_moved"] for w in want]
        assert [led.tier_transfer_count for led in ledgers] == [w["tier_transfer_count"] for w in want]
        assert [a.high_water_bytes for a in accounts] == case["run"]["high_water"]
