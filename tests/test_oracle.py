"""The oracle is pinned before it is trusted (CPU).

oracle/ktune_oracle.c is checked against (a) the reference's own known-answer
tests (test_landscapes.cpp:41-170, acceptance.cpp:547-651,
test_tuner.cpp:209-297), (b) the golden digests the unmodified reference
produced (tests/golden/oracle_golden.json, made by make_golden.py), and
(c) when oracle/_ref is built, the reference's functions on fresh inputs.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O

ref_only = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def test_mt19937_64_standard_value():
    # [rand.predef]: the 10000th output of a default-seeded mt19937_64.
    import ctypes as C

    L = O.oracle_lib()

    class G(C.Structure):
        _fields_ = [("s", C.c_uint64 * 312), ("i", C.c_int)]

    L.ko_mt64_seed.argtypes = [C.POINTER(G), C.c_uint64]
    L.ko_mt64_next.argtypes = [C.POINTER(G)]
    L.ko_mt64_next.restype = C.c_uint64
    g = G()
    L.ko_mt64_seed(C.byref(g), 5489)
    for _ in range(9999):
        L.ko_mt64_next(C.byref(g))
    assert L.ko_mt64_next(C.byref(g)) == 9981545732273789042


def test_conv_hand_examples():
    # test_landscapes.cpp:41-68
    image = np.arange(16, dtype=np.float32)
    ones = np.ones(9, np.float32)
    assert list(O.conv_apply(image, ones, 2, 2, 3, 1.0)) == [45, 54, 81, 90]
    out = O.conv_apply(image, ones, 2, 2, 3, 0.5)
    assert out[0] == 22.5 and out[3] == 45.0
    taps = np.array([1, 0, 0, 0, 1, 0, 0, 0, 2], np.float32)
    assert list(O.conv_apply(image, taps, 2, 2, 3, 1.0)) == [25, 29, 41, 45]


def test_gemm_hand_example():
    # test_landscapes.cpp:118-134
    a = np.array([1, 2, 3, 4], np.float32)
    b = np.array([5, 6, 7, 8], np.float32)
    c = np.array([1, 1, 2, 2], np.float32)
    assert list(O.gemm_apply(a, b, c, 2, 2, 2, 2.0, 3.0)) == [55, 63, 82, 94]


def test_conv_against_independent_accumulation():
    # test_landscapes.cpp:70-116: 16x8, f=3, w=0.25, seed 99
    image = O.materialize("uniform:99", 18 * 10)
    taps = O.materialize(f"uniform:{99 ^ 0x9E3779B97F4A7C15}", 9)
    want = np.zeros(16 * 8, np.float64)
    for i in range(3):
        for j in range(3):
            for r in range(8):
                for c in range(16):
                    want[r * 16 + c] += image[(r + i) * 18 + c + j] * taps[i * 3 + j]
    got = O.conv_reference(16, 8, 3, 0.25, 99)
    assert np.allclose(got, want * 0.25, atol=1e-4)


def test_oracles_against_double_loops():
    # acceptance.cpp:547-651 (criterion 10)
    a = O.materialize("uniform:2026", 64)
    b = O.materialize(f"uniform:{2026 ^ 0x9E3779B97F4A7C15}", 64)
    got = O.gemm_reference(8, 8, 8)
    want = a.reshape(8, 8).astype(np.float64).T @ b.reshape(8, 8).astype(np.float64)
    assert np.allclose(got, want.ravel(), rtol=1e-5)
    for f in (3, 7, 11):
        img = O.materialize("uniform:2026", (64 + f - 1) ** 2).reshape(64 + f - 1, 64 + f - 1)
        taps = O.materialize(f"uniform:{2026 ^ 0x9E3779B97F4A7C15}", f * f).reshape(f, f)
        want = np.zeros((64, 64))
        for fy in range(f):
            for fx in range(f):
                want += taps[fy, fx] * img[fy:fy + 64, fx:fx + 64].astype(np.float64)
        assert np.allclose(O.conv_reference(64, 64, f), want.ravel(), rtol=1e-5)
    # identity filter is exact; alpha = 0, beta = 1 returns C exactly
    img = O.materialize("uniform:2026", 66 * 66)
    delta = np.zeros(9, np.float32)
    delta[4] = 1
    assert np.array_equal(O.conv_apply(img, delta, 64, 64, 3, 1.0),
                          img.reshape(66, 66)[1:65, 1:65].ravel())
    c0 = O.materialize(f"uniform:{2026 ^ 0xC2B2AE3D27D4EB4F}", 64)
    assert np.array_equal(O.gemm_reference(8, 8, 8, 0.0, 1.0), c0)


def test_golden_small_digests(golden):
    for case in golden["small"]:
        if case["kind"] == "conv":
            got = O.conv_reference(case["x"], case["y"], case["f"], case["w"], case["seed"])
        else:
            got = O.gemm_reference(case["m"], case["n"], case["k"], case["alpha"], case["beta"],
                                   case["seed"])
        assert O.digest(got) == case["digest"], case


@pytest.mark.parametrize("f", [3, 11])
def test_golden_full_size_conv_digest(golden, f):
    assert O.digest(O.conv_reference(8192, 4096, f)) == golden["conv_digests"][str(f)]


@pytest.mark.parametrize("m", [512, 1024, 2048])
def test_golden_gemm_digest_row_parallel_restatement(golden, m):
    # The row-parallel restatement is bit-identical to gemm_apply; 2048^3 is
    # pinned to the reference's 168 s single-core run.
    assert O.digest(O.gemm_reference(m, m, m)) == golden["gemm_digests"][str(m)]


VERIFY_CASES = [
    ([1.0, -2.5, 0.0], [1.0, -2.5, 0.0], 1e-4, 1e-6),
    ([2.0001], [2.0], 1e-4, 1e-6),
    ([1.0, 2.0, 4.0, 4.0], [1.0, 2.0, 3.0, 4.0], 1e-4, 1e-6),
    ([5e-7], [0.0], 1e-4, 1e-6),
    ([2e-6], [0.0], 1e-4, 1e-6),
    ([float("nan")], [1.0], 1e-4, 1e-6),
    ([1.0], [1.0], 0.0, 0.0),
    ([1.0000001], [1.0], 0.0, 0.0),
    ([10.5], [10.0], 0.1, 1e-6),
    ([1.0, float("nan"), 3.0, 7.0], [1.0, 2.0, 3.0, 4.0], 1e-4, 1e-6),
    ([1.0, 2.0, float("nan")], [1.0, 2.0, 3.0], 1e-4, 1e-6),
    ([float("inf"), 1.0], [1.0, 1.0], 1e-4, 1e-6),
]


def test_verify_semantics_hand_cases():
    # test_tuner.cpp:209-297
    r = O.verify(np.array([1, -2.5, 0], np.float32), np.array([1, -2.5, 0], np.float32))
    assert r["pass"] and r["max_abs_error"] == 0 and r["elements_compared"] == 3
    r = O.verify(np.array([1, 2, 4, 4], np.float32), np.array([1, 2, 3, 4], np.float32))
    assert not r["pass"] and r["element_index"] == 2 and r["max_abs_error"] == 1.0
    assert O.verify(np.array([5e-7], np.float32), np.zeros(1, np.float32))["pass"]
    assert not O.verify(np.array([2e-6], np.float32), np.zeros(1, np.float32))["pass"]
    r = O.verify(np.array([10.5], np.float32), np.array([10.0], np.float32), 0.1)
    assert r["pass"] and math.isclose(r["max_rel_error"], 0.05, abs_tol=1e-7)
    r = O.verify(np.array([1, 2, 4], np.int32), np.array([1, 2, 3], np.int32))
    assert not r["pass"] and r["element_index"] == 2 and r["max_abs_error"] == 1.0


@ref_only
def test_verify_matches_reference_including_nan_quirk():
    for cand, ref, rel, abs_ in VERIFY_CASES:
        c = np.array(cand, np.float32)
        r = np.array(ref, np.float32)
        a, b = O.verify(c, r, rel, abs_), O.ref_verify(c, r, rel, abs_)
        for k in a:
            assert a[k] == b[k] or (isinstance(a[k], float) and math.isnan(a[k])
                                    and math.isnan(b[k])), (cand, k, a, b)


@ref_only
def test_materialize_matches_reference():
    import ctypes as C

    for fill in ["uniform:0", "uniform:2026", "uniform:18446744073709551615", "ramp",
                 "constant:2.5", "none"]:
        want = np.empty(1000, np.float32)
        assert O.ref_lib().kr_materialize_f32(fill.encode(), 1000, want.ctypes.data) == 0
        assert np.array_equal(O.materialize(fill, 1000), want), fill
    want = np.empty(777, np.int32)
    O.ref_lib().kr_materialize_i32.argtypes = [C.c_char_p, C.c_size_t, C.c_void_p]
    assert O.ref_lib().kr_materialize_i32(b"uniform:77", 777, want.ctypes.data) == 0
    assert np.array_equal(O.materialize("uniform:77", 777, np.int32), want)


@ref_only
def test_restatement_bit_identical_to_reference_on_fresh_problems():
    for (x, y, f, w, s) in [(33, 17, 5, 0.7, 123), (128, 96, 9, 1.0, 4)]:
        assert O.digest(O.conv_reference(x, y, f, w, s)) == O.digest(O.ref_conv_reference(x, y, f, w, s))
    for (m, n, k, a, b, s) in [(48, 40, 33, 1.25, -0.5, 9), (64, 64, 64, 1.0, 1.0, 11)]:
        assert O.digest(O.gemm_reference(m, n, k, a, b, s)) == \
            O.digest(O.ref_gemm_reference(m, n, k, a, b, s))
