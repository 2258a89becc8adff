"""Pin the CPU oracle against golden vectors produced by the real reference.

The fixtures under tests/golden/ were written by tests/golden/make_golden.py,
which runs /root/reference's svsim in the build container.  If the oracle
reproduces them bit for bit, it can stand in for the reference on the GPU
box (where /root/reference does not exist).
"""
import numpy as np
import pytest

from oracle import ref_codec, ref_engine, ref_kernels, ref_layout, ref_optimize
from oracle.ref_builders import adder, benchmark
from oracle.ref_gates import OGate, factor_of
from tests.circuits import unpack


def _same_bits(a, b):
    """array_equal plus identical bit patterns (signed zeros included)."""
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and a.tobytes() == b.tobytes()


def test_kernels_single(golden):
    g = golden("kernels.npz")
    for i in range(int(g["n_single"])):
        psi = g[f"s{i}_in"].copy()
        ref_kernels.gate1(psi, int(g[f"s{i}_q"]), g[f"s{i}_u"])
        assert _same_bits(psi, g[f"s{i}_out"]), i


def test_kernels_two(golden):
    g = golden("kernels.npz")
    for i in range(int(g["n_two"])):
        psi = g[f"t{i}_in"].copy()
        qa, qb = (int(x) for x in g[f"t{i}_q"])
        ref_kernels.gate2(psi, qa, qb, g[f"t{i}_u"])
        assert _same_bits(psi, g[f"t{i}_out"]), i


def test_kernels_diag_and_fp32(golden):
    g = golden("kernels.npz")
    for i in range(int(g["n_diag"])):
        psi = g[f"d{i}_in"].copy()
        ref_kernels.diag(psi, tuple(int(b) for b in g[f"d{i}_bits"]), complex(g[f"d{i}_f"]))
        assert _same_bits(psi, g[f"d{i}_out"]), i
    for i in range(int(g["n_fp32"])):
        psi = g[f"f{i}_in"].copy()
        ref_kernels.gate1(psi, int(g[f"f{i}_q"]), g[f"f{i}_u"])
        assert _same_bits(psi, g[f"f{i}_out"]), i
    for key in [k for k in g if k.startswith("pairs_")]:
        _, n, q = key.split("_")
        assert np.array_equal(ref_kernels.low_members(int(n), int(q)), g[key])


def test_gate_constants(golden):
    g = golden("kernels.npz")
    for k in (1, 2, 3, 4, -1, -2, -3, -4, 7, 16, 25):
        assert _same_bits(np.complex128(factor_of(OGate("PHASE", (0,), k))), g[f"factor_{k}"])


def test_codec_canonicalize_and_numpy_fingerprint(golden):
    g = golden("codec.npz")
    r, th, ux, uy = ref_codec.polar(g["canon_in"])
    for got, key in ((r, "canon_r"), (th, "canon_th"), (ux, "canon_ux"), (uy, "canon_uy")):
        assert _same_bits(got, g[key]), key
    # the numpy primitives the codec inherits behave as on the golden host
    assert _same_bits(np.abs(g["canon_in"]), g["abs_out"])
    assert _same_bits(np.angle(g["canon_in"]), g["angle_out"])
    a, b = g["canon_in"][:10000], g["canon_in"][10000:20000]
    assert _same_bits(a * b, g["mul_out"])


def test_codec_propose_merge_sequence(golden):
    g = golden("codec.npz")
    cb = ref_codec.RefCodebook()
    for s in range(int(g["n_seq"])):
        props = []
        for j in range(int(g[f"seq{s}_ranks"])):
            p = cb.propose(g[f"seq{s}_r{j}_in"])
            for got, key in zip(p, ("mags", "th", "ux", "uy")):
                assert _same_bits(got, g[f"seq{s}_r{j}_{key}"]), (s, j, key)
            props.append(p)
        cb.merge(props)
        assert _same_bits(cb.mags, g[f"seq{s}_mags"])
        assert _same_bits(cb.thetas, g[f"seq{s}_thetas"])
        assert _same_bits(cb.ux, g[f"seq{s}_ux"])
        assert _same_bits(cb.uy, g[f"seq{s}_uy"])
        assert [cb.mag_overflow, cb.phase_overflow] == list(g[f"seq{s}_flags"])
    assert cb.dump() == str(g["seq_dump"])
    mi, pi = cb.encode(g["enc_in"])
    assert _same_bits(mi, g["enc_mi"]) and _same_bits(pi, g["enc_pi"])
    assert _same_bits(cb.decode(mi, pi), g["enc_dec"])
    assert np.array_equal(np.array(cb.resolution()), g["resolution"])


def test_codec_saturated_table_encode(golden):
    g = golden("codec.npz")
    cb = ref_codec.RefCodebook()
    cb.mags, cb.thetas, cb.ux, cb.uy = g["sat_mags"], g["sat_thetas"], g["sat_ux"], g["sat_uy"]
    mi, pi = cb.encode(g["sat_in"])
    assert _same_bits(mi, g["sat_mi"]) and _same_bits(pi, g["sat_pi"])
    assert _same_bits(cb.decode(mi, pi), g["sat_dec"])


def _run_keys(golden):
    return [str(k) for k in golden("runs.npz")["run_keys"]]


def test_engine_runs_match_reference(golden):
    g = golden("runs.npz")
    fields = [str(f) for f in g["ledger_fields"]]
    circuits = {}
    for key in _run_keys(golden):
        name, mode, P = key.split("__")
        if name not in circuits:
            circuits[name] = unpack(g, f"{name}__circuit_")
        run = ref_engine.run_circuit(circuits[name], ranks=int(P), mode=mode)
        assert _same_bits(run.gathered_state(), g[key + "__state"]), key
        if mode == "be":
            assert _same_bits(run.mag, g[key + "__mag"]), key
            assert _same_bits(run.phase, g[key + "__phase"]), key
            assert run.codebook.dump() == str(g[key + "__cb_dump"]), key
            assert _same_bits(run.codebook.ux, g[key + "__cb_ux"]), key
            assert [run.codebook.mag_overflow, run.codebook.phase_overflow] == \
                list(g[key + "__cb_flags"]), key
        if mode == "fp32":
            assert _same_bits(run.psi, g[key + "__psi32"]), key
        got = np.array([[led[f] for f in fields] for led in run.ledgers], dtype=np.int64)
        assert np.array_equal(got, g[key + "__ledgers"]), key
        if key + "__report" in g:
            qx, qy, qz, dev = run.report
            assert np.array_equal(np.array([qx, qy, qz]), g[key + "__report"]), key
            assert dev == float(g[key + "__normdev"]), key


def test_planner_plans_and_memory(golden):
    p = golden("planner.json")
    for e in p["plans"]:
        gate = OGate(e["kind"], tuple(e["qubits"]))
        kind, masks, count, bpe = ref_layout.plan(e["n"], e["local"], gate, e["mode"])
        assert (kind, list(masks), count, bpe) == (e["plan_kind"], e["masks"], e["count"], e["bpe"]), e
    for e in p["memory"]:
        assert ref_layout.memory_bytes(e["n"], e["mode"]) == e["bytes"]


def _workload(name):
    import numpy as _np
    if name == "adder16":
        return adder(16, [47302, 18233])[0]
    if name == "adder19":
        return adder(19, [374982, 149305])[0]
    if name == "adder25":
        return adder(25, [21346502, 12207929])[0]
    if name.startswith("bench"):
        return benchmark(int(name[5:]))
    return None


def test_planner_optimize_labels(golden):
    p = golden("planner.json")
    for e in p["optimize"]:
        circ = _workload(e["name"])
        if circ is None:
            c = e["circuit"]
            d = {k: np.array(v) for k, v in c.items()}
            d["mats"] = np.zeros((len(c["kinds"]), 4, 4), dtype=np.complex128)
            circ = unpack(d)
        perm = ref_optimize.optimize_labels(circ, e["local"])
        assert list(perm) == e["perm"], e["name"]
        assert ref_optimize.predicted_bytes(circ, e["local"]) == e["identity_bytes"]
        assert ref_optimize.predicted_bytes(ref_optimize.relabel(circ, perm), e["local"]) == \
            e["optimized_bytes"]
        for mode in ("fp32", "be"):
            assert ref_optimize.predicted_bytes(circ, e["local"], mode) == e[f"identity_bytes_{mode}"]


def test_rank_order_never_matters_for_oracle(rng):
    from tests.circuits import random_circuit
    circ = random_circuit(rng, 7, 15)
    runs = [ref_engine.run_circuit(circ, ranks=P) for P in (1, 2, 4)]
    for r in runs[1:]:
        assert np.max(np.abs(r.gathered_state() - runs[0].gathered_state())) < 1e-12
