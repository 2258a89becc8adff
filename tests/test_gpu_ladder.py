"""SURVEY 8(c) parity ladder on the GPU: the product's run_circuit vs digests of the REAL
reference's run_circuit (tests/golden/ladder.json, written by
`tests/golden/make_golden.py --ladder` from /root/reference).

Per entry: SHA-256 of the gathered state (complex128, -0.0 folded: np.array_equal
semantics), of the BYTE planes and of the FP32 storage, the full ledgers (exact), the
codebook dump (exact) and the report within 1e-12.  C1 = build_benchmark(20) FP64 P=1.
"""
import json
import os

import numpy as np
import pytest

import paper_2511_03359_b200 as pb
from tests.circuits import ladder_cases, to_product

HERE = os.path.dirname(os.path.abspath(__file__))
MODES = {"fp64": pb.PrecisionMode.FP64, "fp32": pb.PrecisionMode.FP32, "be": pb.PrecisionMode.BYTE}


def _ladder():
    with open(os.path.join(HERE, "golden", "ladder.json")) as f:
        return json.load(f)


def _digest(a) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8).tobytes()).hexdigest()


def state_digest(state) -> str:
    return _digest(np.ascontiguousarray(np.asarray(state, dtype=np.complex128)).view(np.float64) + 0.0)


def _cases():
    circs = {name: (circ, mode) for name, circ, mode, _ in ladder_cases()}
    return [pytest.param(e, circs[e["name"]][0], id=f"{e['name']}-P{e['ranks']}") for e in _ladder()]


def test_ladder_covers_every_case():
    have = {(e["name"], e["ranks"]) for e in _ladder()}
    want = {(name, P) for name, _, _, ranks in ladder_cases() for P in ranks}
    assert have == want


def test_oracle_matches_ladder_c1():
    """The oracle itself against the reference's C1 digest (CPU, ~2 s)."""
    from oracle import ref_engine
    e = next(e for e in _ladder() if e["name"] == "C1_bench20")
    circ = next(c for n, c, _, _ in ladder_cases() if n == "C1_bench20")
    res = ref_engine.run_circuit(circ, ranks=1)
    assert state_digest(res.gathered_state()) == e["state_sha256"]
    assert res.ledgers == e["ledgers"]


@pytest.mark.gpu
@pytest.mark.parametrize("entry,circ", _cases())
def test_ladder_gpu(entry, circ):
    res = pb.run_circuit(to_product(circ), ranks=entry["ranks"], mode=MODES[entry["mode"]])
    assert state_digest(res.gathered_state()) == entry["state_sha256"], "state digest"
    assert [led.snapshot() for led in res.ledgers] == entry["ledgers"], "ledgers"
    qx, qy, qz = entry["report"]
    rep = res.report
    diff = max(np.max(np.abs(np.array(rep.qx) - qx)), np.max(np.abs(np.array(rep.qy) - qy)),
               np.max(np.abs(np.array(rep.qz) - qz)))
    assert diff < 1e-12, diff
    assert abs(rep.norm_deviation - entry["norm_deviation"]) < 1e-12
    if entry["mode"] == "be":
        mag = np.concatenate([s.mag_idx for s in res.states])
        ph = np.concatenate([s.phase_idx for s in res.states])
        h = __import__("hashlib").sha256()
        h.update(np.ascontiguousarray(mag).view(np.uint8).tobytes())
        h.update(np.ascontiguousarray(ph).view(np.uint8).tobytes())
        assert h.hexdigest() == entry["bytes_sha256"], "BYTE planes digest"
        assert res.codebook.dump() == entry["codebook_dump"], "codebook dump"
    if entry["mode"] == "fp32":
        psi = np.concatenate([s.psi for s in res.states])
        assert _digest(np.ascontiguousarray(psi).view(np.float32) + np.float32(0.0)) == entry["psi32_sha256"]
