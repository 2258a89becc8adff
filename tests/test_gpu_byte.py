"""GPU parity tests for the adaptive byte encoding (BYTE mode).

Bar (BASELINE.json north star): bit-exact encoded byte streams and codebooks
versus the reference — checked against the reference's own runs (golden
fixtures) and against the CPU oracle at larger sizes.
"""
import numpy as np
import pytest

import paper_2511_03359_b200 as pb
from paper_2511_03359_b200 import gates as g
from oracle import ref_codec, ref_engine
from tests.circuits import exact_class_circuit, random_circuit, to_product, unpack

pytestmark = pytest.mark.gpu
BE = pb.PrecisionMode.BYTE


def _bytes(res):
    return (np.concatenate([s.mag_idx for s in res.states]),
            np.concatenate([s.phase_idx for s in res.states]))


def test_engine_byte_runs_match_reference_goldens(golden):
    d = golden("runs.npz")
    fields = [str(f) for f in d["ledger_fields"]]
    checked = 0
    circuits = {}
    for key in (str(k) for k in d["run_keys"]):
        name, mode, P = key.split("__")
        if mode != "be":
            continue
        if name not in circuits:
            circuits[name] = to_product(unpack(d, f"{name}__circuit_"))
        res = pb.run_circuit(circuits[name], ranks=int(P), mode=BE)
        mag, ph = _bytes(res)
        assert np.array_equal(mag, d[key + "__mag"]), key
        assert np.array_equal(ph, d[key + "__phase"]), key
        assert res.codebook.dump() == str(d[key + "__cb_dump"]), key
        assert np.array_equal(res.codebook.ux, d[key + "__cb_ux"]), key
        assert np.array_equal(res.codebook.uy, d[key + "__cb_uy"]), key
        assert [res.codebook.mag_overflow, res.codebook.phase_overflow] == list(d[key + "__cb_flags"]), key
        assert np.array_equal(res.gathered_state(), d[key + "__state"]), key
        got = np.array([[led.snapshot()[f] for f in fields] for led in res.ledgers])
        assert np.array_equal(got, d[key + "__ledgers"]), key
        if key + "__report" in d:
            diff = np.max(np.abs(np.array([res.report.qx, res.report.qy, res.report.qz]) - d[key + "__report"]))
            assert diff < 1e-12, (key, diff)
        checked += 1
    assert checked >= 30


@pytest.mark.parametrize("n,depth,spread,ranks", [(16, 80, 3, 1), (18, 100, 4, 4), (17, 60, 2, 8)])
def test_byte_support_tracking_sparse_circuits(n, depth, spread, ranks):
    """BYTE states keep a monotone support (byte_state.py sup_free; monomials and
    non-monomials free their qubits): sparse circuits give byte planes, codebook and report
    identical to the oracle, with the passes and the measurement restricted to the support."""
    from tests.circuits import sparse_circuit
    circ = sparse_circuit(np.random.default_rng(2000 + n + depth), n, depth, spread)
    want = ref_engine.run_circuit(circ, ranks=ranks, mode="be")
    got = pb.run_circuit(to_product(circ), ranks=ranks, mode=BE)
    mag, ph = _bytes(got)
    assert np.array_equal(mag, want.mag) and np.array_equal(ph, want.phase)
    assert got.codebook.dump() == want.codebook.dump()
    qx, qy, qz, _ = want.report
    diff = np.max(np.abs(np.array([got.report.qx, got.report.qy, got.report.qz]) - np.array([qx, qy, qz])))
    assert diff < 1e-12, diff


@pytest.mark.parametrize("n,ranks", [(14, 1), (16, 4), (18, 8)])
def test_byte_benchmark_matches_oracle(n, ranks):
    circ = to_product(__import__("oracle.ref_builders", fromlist=["benchmark"]).benchmark(n))
    want = ref_engine.run_circuit(__import__("oracle.ref_builders", fromlist=["benchmark"]).benchmark(n),
                                  ranks=ranks, mode="be")
    got = pb.run_circuit(circ, ranks=ranks, mode=BE)
    mag, ph = _bytes(got)
    assert np.array_equal(mag, want.mag) and np.array_equal(ph, want.phase)
    assert got.codebook.dump() == want.codebook.dump()
    # the recurrence m_k = fl(sqrt(1/2) * m_{k-1}) and phases {0}: no overflow
    assert not got.codebook.overflowed and len(got.codebook.thetas) == 1


def test_byte_random_and_adder_match_oracle(rng):
    from oracle.ref_builders import adder
    cases = [(random_circuit(rng, 12, 40), 2), (exact_class_circuit(rng, 14, 50), 4), (adder(6, [45, 18])[0], 1)]
    for circ, ranks in cases:
        want = ref_engine.run_circuit(circ, ranks=ranks, mode="be")
        got = pb.run_circuit(to_product(circ), ranks=ranks, mode=BE)
        mag, ph = _bytes(got)
        assert got.codebook.dump() == want.codebook.dump()
        assert np.array_equal(mag, want.mag) and np.array_equal(ph, want.phase)
        qx, qy, qz, dev = want.report
        assert got.report.max_difference(pb.ExpectationReport(qx, qy, qz)) < 1e-12


@pytest.mark.parametrize("ranks", [1, 8])
def test_byte_diagonal_table_passes_match_oracle(ranks):
    """Diagonal gates in BYTE mode run through the 65536-entry code table (scan of the
    selected amplitudes, in-place write; sv_byte.cu k_byte_diag_*): the CPHASE-heavy QFT
    adder at N=14, one rank and 8 reference ranks (tagged per-producer proposals)."""
    from oracle.ref_builders import adder
    circ = adder(7, [101, 77])[0]
    want = ref_engine.run_circuit(circ, ranks=ranks, mode="be")
    got = pb.run_circuit(to_product(circ), ranks=ranks, mode=BE)
    mag, ph = _bytes(got)
    assert got.codebook.dump() == want.codebook.dump()
    assert np.array_equal(mag, want.mag) and np.array_equal(ph, want.phase)
    assert got.report.max_difference(pb.ExpectationReport(*want.report[:3])) < 1e-12


def test_codebook_api_matches_reference(golden):
    c = golden("codec.npz")
    cb = pb.Codebook()
    for s in range(int(c["n_seq"])):
        props = []
        for j in range(int(c[f"seq{s}_ranks"])):
            p = cb.propose(c[f"seq{s}_r{j}_in"])
            assert np.array_equal(p.mags, c[f"seq{s}_r{j}_mags"]), (s, j)
            assert np.array_equal(p.thetas, c[f"seq{s}_r{j}_th"]), (s, j)
            assert np.array_equal(p.ux, c[f"seq{s}_r{j}_ux"]), (s, j)
            props.append(p)
        cb.merge(props)
        assert np.array_equal(cb.mags, c[f"seq{s}_mags"])
        assert np.array_equal(cb.thetas, c[f"seq{s}_thetas"])
    assert cb.dump() == str(c["seq_dump"])
    mi, pi = cb.encode(c["enc_in"])
    assert np.array_equal(mi, c["enc_mi"]) and np.array_equal(pi, c["enc_pi"])
    assert np.array_equal(cb.decode(mi, pi), c["enc_dec"])
    cb2 = pb.Codebook(c["sat_mags"].copy(), c["sat_thetas"].copy(), c["sat_ux"].copy(), c["sat_uy"].copy(),
                      True, True)
    mi, pi = cb2.encode(c["sat_in"])
    assert np.array_equal(mi, c["sat_mi"]) and np.array_equal(pi, c["sat_pi"])
    assert np.array_equal(cb2.decode(mi, pi), c["sat_dec"])


def test_codec_edge_cases():
    cb = pb.Codebook()
    mi, pi = cb.encode(np.array([0j]))
    assert mi[0] == 0 and pi[0] == 0 and cb.decode(mi, pi)[0] == 0
    vals = np.array([np.sqrt(0.5), -np.sqrt(0.5), 0.5j, -0.25j, 1.0, 0.0])
    cb.merge([cb.propose(vals)])
    assert np.array_equal(cb.decode(*cb.encode(vals)), vals)
    cb = pb.Codebook()
    cb.merge([cb.propose(np.array([0.25 + 0j, 0.75 + 0j]))])
    assert cb.encode(np.array([0.5 + 0j]))[0][0] == 2           # tie -> smaller index
    st = pb.LocalState.zero_state(5, BE, True)
    assert st.mag_idx[0] == 1 and st.storage_nbytes * 8 == pb.LocalState.zero_state(5, pb.PrecisionMode.FP64,
                                                                                   True).storage_nbytes


def test_byte_rank_invariant_codebooks(rng):
    circ = to_product(exact_class_circuit(rng, 10, 30))
    dumps = {pb.run_circuit(circ, ranks=r, mode=BE).codebook.dump() for r in (1, 2, 4, 8)}
    assert len(dumps) == 1


def test_numerics_fingerprint_on_the_box_host(golden):
    """SURVEY App. A on the GPU box's own host: the numpy primitives the BYTE host merge
    (codec.py finalize_proposal / host_encode) and the oracle inherit must behave as on the
    host that wrote the goldens -- complex abs, angle (SVML atan2) and complex multiply."""
    c = golden("codec.npz")
    v = c["canon_in"]
    assert np.array_equal(np.abs(v).view(np.uint64), c["abs_out"].view(np.uint64))
    assert np.array_equal(np.angle(v).view(np.uint64), c["angle_out"].view(np.uint64))
    a, b = v[:10000], v[10000:20000]
    assert np.array_equal((a * b).view(np.uint64), c["mul_out"].view(np.uint64))
    r, th, ux, uy = pb.codec.canonicalize(v)
    for got, key in ((r, "canon_r"), (th, "canon_th"), (ux, "canon_ux"), (uy, "canon_uy")):
        assert np.array_equal(np.asarray(got).view(np.uint64), c[key].view(np.uint64)), key


def test_phase_candidate_grouping_with_clustered_angles():
    """The device keeps one phase candidate per distinct GPU theta (sv_byte.cu CtaSets);
    the reference proposes per distinct numpy theta (codec.py:137-152).  Values whose
    angles differ by a few ulps -- where CUDA and numpy atan2 may round apart -- must
    still give the reference's proposals and encodings: clusters of 1-3 ulp angle steps
    around 200 angles (including the axes and 2 pi wrap), several magnitudes each."""
    rng = np.random.default_rng(77)
    base = np.concatenate([rng.uniform(-np.pi, np.pi, 200), [0.0, np.pi / 2, np.pi, -np.pi / 2, 1e-13, -1e-13]])
    vals = []
    for th in base:
        t = th
        for _ in range(6):
            t = np.nextafter(t, 10.0) if rng.integers(2) else np.nextafter(np.nextafter(t, 10.0), 10.0)
            r = rng.uniform(0.05, 1.0)
            vals.append(r * np.exp(1j * t))
    vals = np.array(vals)
    cb = pb.Codebook()
    ref = ref_codec.RefCodebook()
    p = cb.propose(vals)
    q = ref.propose(vals)
    for got, want in zip((p.mags, p.thetas, p.ux, p.uy), q):
        assert np.array_equal(got, want)
    cb.merge([p])
    ref.merge([q])
    assert cb.dump() == ref.dump()
    probe = vals[rng.permutation(vals.size)] * np.exp(1j * 1e-15)
    mi, pi = cb.encode(probe)
    rmi, rpi = ref.encode(probe)
    assert np.array_equal(mi, rmi) and np.array_equal(pi, rpi)
