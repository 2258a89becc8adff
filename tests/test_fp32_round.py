"""FP32 storage rounds every gate's FP64 result to float (kernels.py:36-40,
test_kernels.py:163-170).  The specialised passes can do that rounding on the FP64 pipe
with a Veltkamp split (sv_jit_dev.cuh r32_split) instead of two F2F conversions: these
tests pin it to the float conversion bit for bit -- every tie / carry / exponent-edge
pattern plus random values, the algorithm on the CPU (numpy, round-to-nearest-even FP64
like the device) and the device function itself on the GPU."""
import numpy as np
import pytest

C = np.float64(2 ** 29 + 1)


def edge_patterns() -> np.ndarray:
    """Doubles around every rounding decision: low 29 bits just below / at / above the tie,
    kept mantissa ending in 0 / 1 / all ones (carry into the exponent), every float
    exponent edge (subnormal boundary, overflow), both signs, zeros, infinities, NaN,
    double subnormals."""
    out = []
    exps = list(range(1023 - 150, 1023 - 118)) + list(range(1010, 1030)) + list(range(1023 + 115, 1023 + 131))
    his = [0, 1, 2, 3, 5, (1 << 23) - 1, (1 << 23) - 2, (1 << 22), (1 << 22) + 1, 0x2AAAAA, 0x555555]
    lows = [0, 1, 2, (1 << 28) - 2, (1 << 28) - 1, 1 << 28, (1 << 28) + 1, (1 << 29) - 1, 0x0F0F0F0]
    for e in exps:
        for hm in his:
            for lo in lows:
                for s in (0, 1):
                    out.append((s << 63) | (e << 52) | (hm << 29) | lo)
    out += [0, 1 << 63, 1, (1 << 63) | 1, 0x000FFFFFFFFFFFFF, 0x7FF0000000000000, 0xFFF0000000000000,
            0x7FF8000000000000]
    return np.array(out, dtype=np.uint64).view(np.float64)


def random_values(n: int, seed: int = 7) -> np.ndarray:
    rng = np.random.default_rng(seed)
    e = rng.integers(1023 - 140, 1023 + 4, n).astype(np.uint64)
    m = rng.integers(0, 1 << 52, n, dtype=np.uint64)
    s = rng.integers(0, 2, n).astype(np.uint64)
    return ((s << np.uint64(63)) | (e << np.uint64(52)) | m).view(np.float64)


def split_numpy(x: np.ndarray) -> np.ndarray:
    """r32_split restated: Veltkamp in the normal float range, the float conversion
    elsewhere, zeros as they are."""
    with np.errstate(over="ignore", invalid="ignore"):
        g = C * x
        v = g + (x - g)
        conv = x.astype(np.float32).astype(np.float64)
    e = (x.view(np.uint64) >> np.uint64(52)) & np.uint64(0x7FF)
    fast = (e >= 897) & (e <= 1149)
    return np.where(fast, v, np.where(x == 0.0, x, conv))


def int_numpy(x: np.ndarray) -> np.ndarray:
    """r32_int restated: add half a float ulp (ties to even) to the bits, clear 29 bits."""
    b = x.view(np.uint64)
    e = (b >> np.uint64(52)) & np.uint64(0x7FF)
    r = ((b + np.uint64(0x0FFFFFFF) + ((b >> np.uint64(29)) & np.uint64(1))) & ~np.uint64(0x1FFFFFFF)).view(np.float64)
    with np.errstate(over="ignore", invalid="ignore"):
        conv = x.astype(np.float32).astype(np.float64)
    fast = (e >= 897) & (e <= 1149)
    return np.where(fast, r, np.where(x == 0.0, x, conv))


def _same(a, b):
    return np.array_equal(a.view(np.uint64), b.view(np.uint64)) or np.array_equal(a, b, equal_nan=True)


def test_split_equals_float_rounding_cpu():
    for x in (edge_patterns(), random_values(2_000_000)):
        with np.errstate(over="ignore"):
            want = x.astype(np.float32).astype(np.float64)
        for got in (split_numpy(x), int_numpy(x)):
            assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), \
                np.nonzero(got.view(np.uint64) != want.view(np.uint64))[0][:5]


@pytest.mark.gpu
def test_split_equals_float_rounding_on_device():
    from paper_2511_03359_b200 import _native as nat
    lib = nat.load()
    for x in (edge_patterns(), random_values(8_000_000, seed=11)):
        x = np.ascontiguousarray(x)
        with np.errstate(over="ignore"):
            want = x.astype(np.float32).astype(np.float64)
        for mode in (0, 1, 2):
            out = np.empty_like(x)
            nat.check(lib.svk_f32_round(nat.dptr(x), nat.dptr(out), x.size, mode))
            # NaN payloads are not compared (the GPU returns its canonical NaN)
            bad = np.nonzero((out.view(np.uint64) != want.view(np.uint64)) & ~(np.isnan(out) & np.isnan(want)))[0]
            assert bad.size == 0, (mode, [hex(int(v)) for v in x.view(np.uint64)[bad[:5]]])
