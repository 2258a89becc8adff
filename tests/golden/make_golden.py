"""Generate golden vectors by running the REAL reference package.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It alias-loads ``/root/reference/pkg/src/svsim`` as ``ref_svsim`` (read-only,
nothing is copied into this repo) and writes small compressed fixtures next to
this script:

  kernels.npz  — apply_single / apply_two / apply_diagonal / FP32 rounding /
                 pair_indices on seeded random states        (kernels.py)
  codec.npz    — canonicalize, propose+merge, encode/decode, resolution,
                 numpy abs/angle fingerprints                (codec.py)
  runs.npz     — run_circuit over benchmark / adder / random / exact-class
                 circuits x {fp64, fp32, be} x ranks {1,2,4,8}: gathered
                 states, storage bytes, ledgers, reports, codebooks
  planner.json — plan_exchange, memory_bytes, predicted_exchange_bytes and
                 optimize_labels at the BASELINE configs (N up to 38)
  tier.json    — tier.py: plan_passes groups, TierAccount residency /
                 high-water / counters, naive_staging_bytes,
                 recommended_fast_bytes, validation errors, and
                 run_circuit(tier_config=...) ledgers + state digests
                 (`python tests/golden/make_golden.py --tier`)
  ladder.json  — the SURVEY 8(c) parity ladder at sizes too large for npz
                 fixtures: C1 = build_benchmark(20) FP64 P=1, benchmark 22/24
                 and adder(11) FP64 at P in {1, 8}, FP32 benchmark(22), BYTE
                 benchmark 20/22 and adder(10) at P=8.  Stored as SHA-256
                 digests of the state (complex128, -0.0 folded to +0.0) and of
                 the BYTE planes, plus the full ledgers, report and codebook
                 dump (`python tests/golden/make_golden.py --ladder`)

The fixtures are what pins the oracle (tests/test_oracle_golden.py) and what
the GPU parity tests compare against on the B200 box.
"""
from __future__ import annotations

import importlib.util
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from tests.circuits import (SEED, exact_class_circuit, haar_unitary, ladder_cases, pack,  # noqa: E402
                            random_circuit, to_reference)
from oracle.ref_builders import OCircuit, adder, benchmark  # noqa: E402
from oracle.ref_gates import OGate  # noqa: E402

REF_SRC = "/root/reference/pkg/src/svsim"


def load_reference():
    spec = importlib.util.spec_from_file_location(
        "ref_svsim", os.path.join(REF_SRC, "__init__.py"),
        submodule_search_locations=[REF_SRC])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["ref_svsim"] = mod
    spec.loader.exec_module(mod)
    return mod


def random_state(rng, n):
    psi = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    return (psi / np.linalg.norm(psi)).astype(np.complex128)


def make_kernels(ref):
    K = ref.kernels
    rng = np.random.default_rng(SEED)
    out = {}
    i = 0
    for n in (6, 9, 11):
        for q in range(n):
            psi = random_state(rng, n)
            u = haar_unitary(rng, 2)
            res = psi.copy()
            K.apply_single(res, q, u)
            out[f"s{i}_in"], out[f"s{i}_u"], out[f"s{i}_out"] = psi, u, res
            out[f"s{i}_q"] = np.int64(q)
            i += 1
    out["n_single"] = np.int64(i)
    i = 0
    for n, pairs in ((5, [(0, 1), (1, 0), (4, 2), (2, 4), (0, 4)]),
                     (9, [(0, 8), (8, 0), (3, 7), (7, 3), (5, 6), (1, 2)])):
        for qa, qb in pairs:
            psi = random_state(rng, n)
            u = haar_unitary(rng, 4)
            res = psi.copy()
            K.apply_two(res, qa, qb, u)
            out[f"t{i}_in"], out[f"t{i}_u"], out[f"t{i}_out"] = psi, u, res
            out[f"t{i}_q"] = np.array([qa, qb], dtype=np.int64)
            i += 1
    out["n_two"] = np.int64(i)
    i = 0
    for n, bits, gate in ((8, (), ref.gates.z(0)), (8, (3,), ref.gates.phase(3, 2)),
                          (8, (0, 7), ref.gates.cphase(0, 7, 1)),
                          (10, (2, 9), ref.gates.cphase(2, 9, -3)),
                          (10, (5,), ref.gates.phase(5, -4)), (10, (), ref.gates.phase(0, 4))):
        psi = random_state(rng, n)
        f = ref.gates.diagonal_factor(gate)
        res = psi.copy()
        K.apply_diagonal(res, bits, f)
        out[f"d{i}_in"], out[f"d{i}_out"] = psi, res
        out[f"d{i}_bits"] = np.array(bits, dtype=np.int64)
        out[f"d{i}_f"] = np.complex128(f)
        i += 1
    out["n_diag"] = np.int64(i)
    i = 0
    for n in (6, 9):
        for q in (0, 2, n - 1):
            psi32 = random_state(rng, n).astype(np.complex64)
            u = haar_unitary(rng, 2)
            res = psi32.copy()
            K.apply_single(res, q, u)
            out[f"f{i}_in"], out[f"f{i}_u"], out[f"f{i}_out"] = psi32, u, res
            out[f"f{i}_q"] = np.int64(q)
            i += 1
    out["n_fp32"] = np.int64(i)
    for n, q in ((6, 0), (6, 3), (8, 5), (12, 11)):
        out[f"pairs_{n}_{q}"] = K.pair_indices(n, q)
    # the gate constants, bit for bit
    for k in (1, 2, 3, 4, -1, -2, -3, -4, 7, 16, 25):
        out[f"factor_{k}"] = np.complex128(ref.gates.diagonal_factor(ref.gates.phase(0, k)))
    out["H"] = ref.gates.H_MATRIX
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **out)


def make_codec(ref):
    C = ref.codec
    rng = np.random.default_rng(SEED + 1)
    out = {}
    specials = np.array([0j, complex(-0.0, 0.0), complex(0.0, -0.0), 1 + 0j, -1 + 0j, 1j, -1j,
                         complex(0.5, -0.0), complex(-0.5, -0.0), complex(-0.5, 0.0),
                         complex(0.6, -0.8), complex(1e-300, 1e-300), complex(5e-324, 0),
                         complex(1.0, -1e-13), complex(1.0, -1e-12), complex(1.0, -2e-12),
                         complex(3.0, 4.0), complex(-3.0, -4.0), complex(1e200, 1e200)])
    vals = np.concatenate([specials,
                           rng.normal(size=20000) + 1j * rng.normal(size=20000),
                           np.exp(1j * rng.uniform(-np.pi, np.pi, 5000)) * rng.uniform(0, 1, 5000)])
    r, th, ux, uy = C.canonicalize(vals)
    out.update(canon_in=vals, canon_r=r, canon_th=th, canon_ux=ux, canon_uy=uy)
    # numpy primitives the codec inherits (fingerprint of this host)
    out["abs_out"] = np.abs(vals)
    out["angle_out"] = np.angle(vals)
    a, b = vals[:10000], vals[10000:20000]
    out["mul_out"] = a * b

    # propose / merge sequences, per-rank proposals, overflow
    cb = C.Codebook()
    steps = []
    for s in range(6):
        n_ranks = [1, 2, 4, 3, 8, 2][s]
        per_rank = []
        for _ in range(n_ranks):
            m = int(rng.integers(1, 80))
            v = (rng.uniform(0, 1, m) * np.exp(1j * rng.choice(np.linspace(0, 2 * np.pi, 40), m)))
            v = np.round(v, int(rng.integers(2, 6)))
            per_rank.append(v)
        props = [cb.propose(v) for v in per_rank]
        for j, (v, p) in enumerate(zip(per_rank, props)):
            out[f"seq{s}_r{j}_in"] = v
            out[f"seq{s}_r{j}_mags"] = p.mags
            out[f"seq{s}_r{j}_th"] = p.thetas
            out[f"seq{s}_r{j}_ux"] = p.ux
            out[f"seq{s}_r{j}_uy"] = p.uy
        cb.merge(props)
        out[f"seq{s}_ranks"] = np.int64(n_ranks)
        out[f"seq{s}_mags"] = cb.mags.copy()
        out[f"seq{s}_thetas"] = cb.thetas.copy()
        out[f"seq{s}_ux"] = cb.ux.copy()
        out[f"seq{s}_uy"] = cb.uy.copy()
        out[f"seq{s}_flags"] = np.array([cb.mag_overflow, cb.phase_overflow])
        steps.append(n_ranks)
    out["n_seq"] = np.int64(len(steps))
    out["seq_dump"] = np.array(cb.dump())
    probe = rng.normal(size=4000) + 1j * rng.normal(size=4000)
    probe = np.concatenate([probe, np.array([0j, 0.5 + 0j, -0.25j])])
    mi, pi = cb.encode(probe)
    out.update(enc_in=probe, enc_mi=mi, enc_pi=pi, enc_dec=cb.decode(mi, pi))
    out["resolution"] = np.array(cb.resolution())
    # a saturated generic table (both overflow flags set) and its encodings
    cb2 = C.Codebook()
    cb2.merge([cb2.propose(rng.normal(size=400) + 1j * rng.normal(size=400))])
    probe2 = rng.normal(size=20000) + 1j * rng.normal(size=20000)
    mi2, pi2 = cb2.encode(probe2)
    out.update(sat_mags=cb2.mags, sat_thetas=cb2.thetas, sat_ux=cb2.ux, sat_uy=cb2.uy,
               sat_in=probe2, sat_mi=mi2, sat_pi=pi2, sat_dec=cb2.decode(mi2, pi2),
               sat_flags=np.array([cb2.mag_overflow, cb2.phase_overflow]))
    np.savez_compressed(os.path.join(HERE, "codec.npz"), **out)


def run_cases():
    rng = lambda s: np.random.default_rng(SEED + 100 + s)  # noqa: E731
    cases = [
        ("bench8", benchmark(8), ("fp64", "fp32", "be"), (1, 2, 4, 8)),
        ("bench10", benchmark(10), ("fp64", "fp32", "be"), (1, 2, 4, 8)),
        ("bench12", benchmark(12), ("fp64", "be"), (1, 8)),
        ("rand6", random_circuit(rng(1), 6, 12), ("fp64", "fp32", "be"), (1, 2, 4)),
        ("rand7", random_circuit(rng(2), 7, 20), ("fp64", "fp32", "be"), (1, 2, 4, 8)),
        ("rand8", random_circuit(rng(3), 8, 25), ("fp64", "fp32", "be"), (1, 4, 8)),
        ("rand9", random_circuit(rng(4), 9, 40), ("fp64", "be"), (1, 2, 8)),
        ("exact8", exact_class_circuit(rng(5), 8, 20), ("fp64", "be"), (1, 2, 4, 8)),
        ("exact10", exact_class_circuit(rng(6), 10, 40), ("fp64", "be"), (1, 8)),
        ("adder3", adder(3, [2, 5])[0], ("fp64", "fp32", "be"), (1, 2, 4)),
        ("adder5", adder(5, [11, 19])[0], ("fp64", "be"), (1, 4, 8)),
        ("adder3x3", adder(3, [1, 5, 6])[0], ("fp64", "be"), (1, 8)),
        ("adder7", adder(7, [77, 50])[0], ("fp64", "be"), (1, 8)),
        ("adder8", adder(8, [172, 83])[0], ("fp64", "be"), (1, 4)),
        ("bench16", benchmark(16), ("be",), (1, 8)),
        ("diag6", OCircuit(6, (OGate("H", (0,)), OGate("H", (5,)), OGate("H", (3,)),
                               OGate("Z", (5,)), OGate("CPHASE", (4, 5), 2),
                               OGate("PHASE", (3,), 1), OGate("CPHASE", (0, 5), 3),
                               OGate("PHASE", (5,), -3), OGate("M"))),
         ("fp64", "fp32", "be"), (1, 2, 4, 8)),
        ("quad6", OCircuit(6, (OGate("H", (0,)), OGate("H", (4,)), OGate("U4", (4, 5), 0,
                                                                          haar_unitary(rng(7), 4)),
                               OGate("CNOT", (5, 1)), OGate("CNOT", (2, 4)),
                               OGate("U4", (5, 4), 0, haar_unitary(rng(8), 4)), OGate("M"))),
         ("fp64", "fp32", "be"), (1, 2, 4, 8)),
    ]
    return cases


def make_runs(ref):
    modes = {"fp64": ref.PrecisionMode.FP64, "fp32": ref.PrecisionMode.FP32,
             "be": ref.PrecisionMode.BYTE}
    out = {}
    names = []
    for name, circ, mode_list, rank_list in run_cases():
        out[f"{name}__circuit_" + "n_qubits"] = np.int64(circ.n_qubits)
        for k, v in pack(circ).items():
            out[f"{name}__circuit_{k}"] = v
        rc = to_reference(circ, ref)
        for mode in mode_list:
            for P in rank_list:
                if circ.n_qubits - (P.bit_length() - 1) < 2:
                    continue
                key = f"{name}__{mode}__{P}"
                res = ref.run_circuit(rc, ranks=P, mode=modes[mode])
                out[key + "__state"] = res.gathered_state()
                if mode == "be":
                    out[key + "__mag"] = np.concatenate([s.mag_idx for s in res.states])
                    out[key + "__phase"] = np.concatenate([s.phase_idx for s in res.states])
                    cb = res.codebook
                    out[key + "__cb_mags"] = cb.mags
                    out[key + "__cb_thetas"] = cb.thetas
                    out[key + "__cb_ux"] = cb.ux
                    out[key + "__cb_uy"] = cb.uy
                    out[key + "__cb_flags"] = np.array([cb.mag_overflow, cb.phase_overflow])
                    out[key + "__cb_dump"] = np.array(cb.dump())
                elif mode == "fp32":
                    out[key + "__psi32"] = np.concatenate([s.psi for s in res.states])
                fields = list(res.ledgers[0].snapshot().keys())
                out[key + "__ledgers"] = np.array(
                    [[l.snapshot()[f] for f in fields] for l in res.ledgers], dtype=np.int64)
                rep = res.report
                if rep is not None:
                    out[key + "__report"] = np.array([rep.qx, rep.qy, rep.qz])
                    out[key + "__normdev"] = np.float64(rep.norm_deviation)
                names.append(key)
                print("ran", key, flush=True)
    out["ledger_fields"] = np.array(fields)
    out["run_keys"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "runs.npz"), **out)


def make_planner(ref):
    P = ref.PrecisionMode
    g = ref.gates
    res = {"plans": [], "memory": [], "optimize": [], "predicted": []}
    gate_set = [g.h(0), g.h(35), g.h(39), g.z(39), g.cphase(38, 39, 3), g.phase(33, 2),
                g.cnot(2, 36), g.cnot(36, 2), g.u4(7, 9, ref.gates.CNOT_MATRIX),
                g.u4(33, 34, ref.gates.CNOT_MATRIX), g.u4(35, 33, ref.gates.CNOT_MATRIX),
                g.x(32), g.y(34), g.measure_all()]
    for (n, loc) in ((40, 32), (36, 33), (38, 35), (40, 39), (36, 36)):
        for gate in gate_set:
            if any(q >= n for q in gate.qubits):
                continue
            for mode in ("fp64", "fp32", "be"):
                p = ref.plan_exchange(ref.PartitionLayout(n, loc), gate,
                                      {"fp64": P.FP64, "fp32": P.FP32, "be": P.BYTE}[mode])
                res["plans"].append(dict(n=n, local=loc, kind=gate.kind, qubits=list(gate.qubits),
                                         mode=mode, plan_kind=p.kind, masks=list(p.masks),
                                         count=p.element_count, bpe=p.bytes_per_element))
    for n in (1, 20, 32, 33, 36, 38, 50):
        for mode in ("fp64", "fp32", "be"):
            res["memory"].append(dict(n=n, mode=mode, bytes=ref.memory_bytes(
                n, {"fp64": P.FP64, "fp32": P.FP32, "be": P.BYTE}[mode])))
    workloads = [
        ("adder16", ref.build_adder(16, [47302, 18233])[0], (29, 30, 31, 32)),
        ("adder19", ref.build_adder(19, [374982, 149305])[0], (35, 36, 37, 38)),
        ("bench33", ref.build_benchmark(33), (30, 31, 32, 33)),
        ("bench36", ref.build_benchmark(36), (33,)),
        ("bench38", ref.build_benchmark(38), (35,)),
        ("adder25", ref.build_adder(25, [21346502, 12207929])[0], (42, 45)),
    ]
    srcs = ref.relabel(ref.build_adder(3, [2, 5])[0], (3, 4, 5, 0, 1, 2))
    workloads.append(("adder3_srchigh", srcs, (4,)))
    rng = np.random.default_rng(SEED + 7)
    for t in range(6):
        n = int(rng.integers(5, 10))
        workloads.append((f"rand_opt{t}", to_reference(random_circuit(rng, n, 14), ref), (n - 2, n - 1)))
    for name, circ, locals_ in workloads:
        for loc in locals_:
            layout = ref.PartitionLayout(circ.n_qubits, loc)
            perm = ref.optimize_labels(circ, layout)
            entry = dict(name=name, local=loc, perm=list(perm),
                         identity_bytes=ref.predicted_exchange_bytes(circ, layout),
                         optimized_bytes=ref.predicted_exchange_bytes(ref.relabel(circ, perm), layout))
            for mode in ("fp32", "be"):
                entry[f"identity_bytes_{mode}"] = ref.predicted_exchange_bytes(
                    circ, layout, {"fp32": P.FP32, "be": P.BYTE}[mode])
            if name.startswith("rand") or name.endswith("srchigh"):
                entry["circuit"] = {k: (v.tolist() if hasattr(v, "tolist") else v)
                                    for k, v in pack(circ).items() if k != "mats"}
            res["optimize"].append(entry)
    with open(os.path.join(HERE, "planner.json"), "w") as f:
        json.dump(res, f, indent=1, default=lambda o: o.item() if hasattr(o, "item") else str(o))


def state_digest(state) -> str:
    """SHA-256 of a gathered state as complex128 with negative zeros folded (np.array_equal
    semantics: X / CNOT as moves may flip the sign of an exact zero)."""
    import hashlib
    a = np.ascontiguousarray(np.asarray(state, dtype=np.complex128)).view(np.float64) + 0.0
    return hashlib.sha256(a.tobytes()).hexdigest()


def bytes_digest(*planes) -> str:
    import hashlib
    h = hashlib.sha256()
    for p in planes:
        h.update(np.ascontiguousarray(p).view(np.uint8).tobytes())
    return h.hexdigest()


def make_ladder(ref):
    import time
    modes = {"fp64": ref.PrecisionMode.FP64, "fp32": ref.PrecisionMode.FP32, "be": ref.PrecisionMode.BYTE}
    out = []
    for name, circ, mode, ranks in ladder_cases():
        rc = to_reference(circ, ref)
        for P in ranks:
            t0 = time.perf_counter()
            res = ref.run_circuit(rc, ranks=P, mode=modes[mode])
            dt = time.perf_counter() - t0
            ent = dict(name=name, mode=mode, ranks=P, n_qubits=circ.n_qubits, gates=len(circ.gates),
                       state_sha256=state_digest(res.gathered_state()), ref_seconds=round(dt, 2),
                       ledgers=[l.snapshot() for l in res.ledgers])
            rep = res.report
            ent["report"] = [list(map(float, rep.qx)), list(map(float, rep.qy)), list(map(float, rep.qz))]
            ent["norm_deviation"] = float(rep.norm_deviation)
            if mode == "be":
                mag = np.concatenate([s_.mag_idx for s_ in res.states])
                ph = np.concatenate([s_.phase_idx for s_ in res.states])
                ent["bytes_sha256"] = bytes_digest(mag, ph)
                ent["codebook_dump"] = res.codebook.dump()
                ent["codebook_flags"] = [bool(res.codebook.mag_overflow), bool(res.codebook.phase_overflow)]
            if mode == "fp32":
                psi = np.concatenate([s_.psi for s_ in res.states])
                ent["psi32_sha256"] = bytes_digest(np.ascontiguousarray(psi).view(np.float32) + np.float32(0.0))
            out.append(ent)
            print("ladder", name, mode, P, f"{dt:.1f}s", flush=True)
            with open(os.path.join(HERE, "ladder.json"), "w") as f:
                json.dump(out, f, indent=0, default=lambda o: o.item() if hasattr(o, "item") else str(o))


def tier_cases():
    """(name, circuit, n_local, mode, TierConfig args) for the tier goldens."""
    from tests.circuits import random_circuit as rc
    r = lambda s: np.random.default_rng(SEED + 300 + s)  # noqa: E731
    B = lambda n, m: (1 << n) * {"fp64": 16, "fp32": 8, "be": 2}[m]  # noqa: E731
    return [
        ("rand10_q4_c64", rc(r(1), 10, 24), 10, "fp64", (B(10, "fp64") // 4, B(10, "fp64") // 64, 64)),
        ("rand10_q4_c16", rc(r(2), 10, 30), 10, "fp64", (B(10, "fp64") // 4, B(10, "fp64") // 16, 64)),
        ("rand9_w4", rc(r(3), 9, 40), 9, "fp64", (B(9, "fp64") // 4, B(9, "fp64") // 32, 4)),
        ("rand9_fp32", rc(r(4), 9, 30), 9, "fp32", (B(9, "fp32") // 3, B(9, "fp32") // 32, 64)),
        ("rand9_be", rc(r(5), 9, 30), 9, "be", (B(9, "be") // 4, B(9, "be") // 16, 64)),
        ("bench12_c8", benchmark(12), 12, "fp64", (B(12, "fp64") // 2, B(12, "fp64") // 8, 64)),
        ("bench12_resident", benchmark(12), 12, "fp64", (B(12, "fp64"), B(12, "fp64") // 2, 64)),
        ("adder6", adder(6, [40, 21])[0], 12, "fp64", (B(12, "fp64") // 4, B(12, "fp64") // 32, 64)),
        ("exact9_r4", exact_class_circuit(r(6), 9, 20), 7, "fp64", (B(7, "fp64") // 4, B(7, "fp64") // 32, 64)),
        ("rand8_r2", rc(r(7), 8, 30), 7, "fp64", (B(7, "fp64") // 4, B(7, "fp64") // 16, 64)),
        ("bench34_cfg", benchmark(34), 34, "fp64", (160 << 30, 4 << 30, 64)),
        ("bench34_c8", benchmark(34), 34, "fp64", (160 << 30, 8 << 30, 64)),
        ("adder17_cfg", adder(17, [3, 5])[0], 34, "fp64", (160 << 30, 4 << 30, 64)),
    ]


def make_tier(ref):
    T = ref.tier
    modes = {"fp64": ref.PrecisionMode.FP64, "fp32": ref.PrecisionMode.FP32, "be": ref.PrecisionMode.BYTE}
    out = {"cases": [], "errors": [], "recommended": []}
    for name, circ, n_local, mode, (fast, chunk, window) in tier_cases():
        cfg = T.TierConfig(fast, chunk, window)
        rc_ = to_reference(circ, ref)
        plan = T.plan_passes(rc_.gates, cfg, n_local, modes[mode])
        led = ref.TrafficLedger()
        state_bytes = (1 << n_local) * modes[mode].bytes_per_element
        acct = T.TierAccount(state_bytes, cfg, led)
        for grp in plan.groups:
            acct.account(grp)
        ent = dict(name=name, n_local=n_local, mode=mode, config=[fast, chunk, window],
                   chunk_qubits=plan.chunk_qubits, n_chunks=plan.n_chunks,
                   groups=[[grp.kind, list(grp.gate_indices), [list(m) for m in grp.chunk_groups]]
                           for grp in plan.groups],
                   fast_resident=[bool(x) for x in acct.fast_resident],
                   static_fast_bytes=acct.static_fast_bytes, high_water_bytes=acct.high_water_bytes,
                   slow_bytes=acct.slow_bytes, tier_bytes=led.tier_bytes_moved,
                   tier_transfers=led.tier_transfer_count,
                   naive=T.naive_staging_bytes(rc_.gates, cfg, n_local, modes[mode]),
                   n_passes=len(plan.passes()))
        if circ.n_qubits <= 12:
            P = 1 << (circ.n_qubits - n_local)
            res = ref.run_circuit(rc_, ranks=P, mode=modes[mode], tier_config=cfg)
            ent["run"] = dict(ranks=P, state_sha256=state_digest(res.gathered_state()),
                              ledgers=[l.snapshot() for l in res.ledgers],
                              high_water=[a.high_water_bytes for a in res.tier_accounts])
        out["cases"].append(ent)
        print("tier", name, flush=True)
    for args in ((1024, 100), (1024, 1024), (4096, 256, 0)):
        try:
            T.TierConfig(*args)
            out["errors"].append([list(args), None])
        except ValueError as exc:
            out["errors"].append([list(args), str(exc)])
    try:
        T.plan_passes((ref.gates.u4(2, 3, ref.gates.CNOT_MATRIX),), T.TierConfig(2 * 64, 64), 6,
                      ref.PrecisionMode.FP64)
        out["errors"].append(["quad_tight", None])
    except ValueError as exc:
        out["errors"].append(["quad_tight", str(exc)])
    for sb, cb in ((1280 * 1024, 1024), (256 << 30, 4 << 30), (1 << 20, 1 << 12), (12345678, 4096)):
        out["recommended"].append([sb, cb, T.recommended_fast_bytes(sb, cb)])
    with open(os.path.join(HERE, "tier.json"), "w") as f:
        json.dump(out, f, indent=0)


def main():
    ref = load_reference()
    if "--tier" in sys.argv:
        make_tier(ref)
        return
    if "--ladder" in sys.argv:
        make_ladder(ref)
        return
    make_kernels(ref)
    make_codec(ref)
    make_planner(ref)
    make_runs(ref)
    make_tier(ref)
    make_ladder(ref)


if __name__ == "__main__":
    main()
