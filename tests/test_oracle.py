"""Pin the oracle (oracle/fmafft_oracle.c) before trusting it.

1. Against the golden fixtures the reference itself produced
   (tests/golden/make_golden.py) -- runs everywhere.
2. Against the reference library compiled here (oracle/_ref), bit for bit,
   when it is present.
3. Against the reference's own known-answer tests: Table I/II values
   (test_twiddle.cpp:54-120, test_analysis.cpp:66-114), op counts
   (test_fft.cpp:130-149), binary16 conversion (test_precision.cpp:93-112,
   acceptance.cpp:276-306), the FP64 oracle equivalence (test_fft.cpp:110-128).
"""
import os

import numpy as np
import pytest

from helpers import ALL_STRATEGIES, WORK_DTYPE, bit_mismatches

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


# ---- 1. golden fixtures ---------------------------------------------------------

def test_tables_match_golden(orc, golden):
    for key in golden.files:
        if not key.startswith("table/"):
            continue
        _, n, s, p = key.split("/")
        got = orc.plan_table(int(n), s, p)
        assert got.tobytes() == golden[key].tobytes(), key


@pytest.mark.parametrize("n", [2, 16, 64, 256, 1024, 4096])
def test_forward_inverse_match_golden(orc, golden, n):
    for p in ("fp16", "fp32"):
        seed, batch = golden[f"seed/{n}/{p}"]
        x = orc.random_buffer(n, int(seed), batch=int(batch))
        xr = orc.round_to(x.view(np.float64), p).view(np.complex128).reshape(int(batch), n)
        for s in ALL_STRATEGIES:
            y = orc.forward(xr, s, p).view(np.float64).astype(WORK_DTYPE[p])
            assert bit_mismatches(y, golden[f"fwd/{n}/{s}/{p}"]) == 0, (n, s, p)
            yi = orc.inverse(xr, s, p).view(np.float64).astype(WORK_DTYPE[p])
            assert bit_mismatches(yi, golden[f"inv/{n}/{s}/{p}"]) == 0, (n, s, p)


def test_measure_error_matches_golden(orc, golden):
    rows = golden["measure_error/forward/seed42/trials10"]
    for n, s, p, med, mx, nonfin in rows:
        if n > 1024:
            continue  # the O(n^2) oracle DFT at 4096 is slow; covered by _ref below
        r = orc.measure_error(int(n), ALL_STRATEGIES[int(s)], ("fp16", "fp32")[int(p)],
                              "forward", 10, 42)
        assert r["rel_l2_median"] == med or (np.isinf(med) and np.isinf(r["rel_l2_median"]))
        assert r["rel_l2_max"] == mx or (np.isinf(mx) and np.isinf(r["rel_l2_max"]))
        assert r["nonfinite_trials"] == nonfin


def test_baseline_md_error_table(golden):
    """BASELINE.md's expected errors (forward vs FP64 DFT, seed 42, 10 trials)."""
    rows = {(int(r[0]), int(r[1]), int(r[2])): r for r in
            golden["measure_error/forward/seed42/trials10"]}
    dual16 = rows[(1024, 3, 0)]
    assert f"{dual16[3]:.3g}" == "0.000835" and f"{dual16[4]:.3g}" == "0.000873"
    assert rows[(1024, 2, 0)][5] == 10  # cosine fp16: every trial non-finite
    assert rows[(1024, 1, 0)][3] > dual16[3]  # dual beats LF


# ---- 2. the reference library itself -------------------------------------------

def test_oracle_bitwise_vs_reference(orc, ref):
    for n in [2 ** m for m in range(1, 13)]:
        for s in ALL_STRATEGIES:
            for p in ("fp16", "fp32", "fp64"):
                assert orc.plan_table(n, s, p).tobytes() == ref.plan_table(n, s, p).tobytes()
                x = orc.random_buffer(n, 7 * n + 1, batch=2)
                a, ca = orc.forward(x, s, p, counters=True)
                b, cb = ref.forward(x, s, p, counters=True)
                assert bit_mismatches(a.view(np.float64), b.view(np.float64)) == 0, (n, s, p)
                assert (ca.fma_count, ca.mul_count, ca.add_count) == \
                    (cb.fma_count, cb.mul_count, cb.add_count)
                a = orc.inverse(x, s, p)
                b = ref.inverse(x, s, p)
                assert bit_mismatches(a.view(np.float64), b.view(np.float64)) == 0, (n, s, p)


def test_round_to_vs_reference(orc, ref):
    rng = np.random.RandomState(916)
    x = (1 + rng.randint(0, 1 << 52, 200000) * 2.0 ** -52) * np.exp2(rng.randint(-30, 21, 200000))
    x *= np.where(rng.randint(0, 2, 200000), -1.0, 1.0)
    x = np.concatenate([x, [0.0, -0.0, 65504.0, 65519.999, 65520.0, -65520.0, 2049.0,
                            1 + 2 ** -12, 2 ** -24, 2 ** -25, 1.5 * 2 ** -24, 1e-7, 1e300,
                            -1e300, np.inf, -np.inf, 5e-324]])
    for p in ("fp16", "fp32"):
        assert orc.round_to(x, p).tobytes() == ref.round_to(x, p).tobytes()


def test_measure_error_vs_reference(orc, ref):
    for metric in ("forward", "roundtrip"):
        for s in ALL_STRATEGIES:
            a = orc.measure_error(256, s, "fp16", metric, 4, 11)
            b = ref.measure_error(256, s, "fp16", metric, 4, 11)
            assert a == b


# ---- 3. the reference's own known answers ----------------------------------------

def test_table_one_values(orc):
    """PAPER.md:146-151 / test_twiddle.cpp:54-120."""
    lf = orc.table_stats(1024, "lf")
    assert abs(lf["t_max"] - 163.0) / 163.0 < 5e-4 and lf["argmax_k"] == 1
    assert lf["singular_count"] == 1
    cos = orc.table_stats(1024, "cosine")
    assert cos["t_max"] > 1e16 and cos["argmax_k"] == 256
    du = orc.table_stats(1024, "dual")
    assert du["t_max"] <= 1.0 and du["argmax_k"] == 128 and du["singular_count"] == 0
    assert du["cos_path_count"] == 256 and du["sin_path_count"] == 256
    eps = orc.machine_epsilon("fp16")
    assert abs(orc.cumulative_bound(du["t_max"], eps, 10) - 4.89e-3) < 1e-5
    ratio = orc.cumulative_bound(lf["t_max"], eps, 10) / orc.cumulative_bound(du["t_max"], eps, 10)
    assert abs(ratio - 235) < 1


def test_dual_ratio_bound_exhaustive(orc):
    """acceptance.cpp:136-156 (to 2^16)."""
    for m in range(1, 17):
        t = orc.build_table(2 ** m, "dual")
        assert np.all(np.abs(t["ratio"]) <= 1.0) and not t["clamped"].any()


def test_lf_clamp_entry(orc):
    t = orc.build_table(1024, "lf")
    e0 = t[0]
    assert e0["clamped"] == 1 and e0["multiplier"] == -1e-7 and e0["omega_r"] == 1.0
    assert np.signbit(e0["omega_i"]) and e0["omega_i"] == 0.0
    t3 = orc.build_table(1024, "lf", clamp_eps=1e-3)
    assert t3[0]["multiplier"] == -1e-3
    with pytest.raises(ValueError, match="clamp_eps"):
        orc.build_table(8, "lf", clamp_eps=0.0)
    with pytest.raises(ValueError, match="power of two"):
        orc.build_table(1023, "dual")


def test_op_counts(orc):
    """test_fft.cpp:130-149 / acceptance criterion 8."""
    for n in (2, 64, 1024):
        bf = (n // 2) * (n.bit_length() - 1)
        x = orc.random_buffer(n, n, batch=1)
        for s in ("lf", "cosine", "dual"):
            _, c = orc.forward(x, s, "fp64", counters=True)
            assert (c.fma_count, c.mul_count, c.add_count) == (6 * bf, 0, 0)
        _, c = orc.forward(x, "standard", "fp64", counters=True)
        assert (c.fma_count, c.mul_count, c.add_count) == (0, 4 * bf, 6 * bf)
    _, c = orc.inverse(orc.random_buffer(64, 5, batch=1), "dual", "fp64", counters=True)
    assert c.mul_count == 2 * 64


def test_fp64_oracle_equivalence(orc):
    """test_fft.cpp:110-128 / acceptance criterion 5: rel-L2 < 1e-11."""
    for m in range(1, 10):
        n = 2 ** m
        x = orc.random_buffer(n, 1000 + n, batch=1)
        ref = orc.dft(x)
        for s in ALL_STRATEGIES:
            assert orc.rel_l2(orc.forward(x, s, "fp64"), ref) < 1e-11


def test_negative_control(orc):
    """test_fft.cpp:240-250: a flipped ratio must be caught (err > 1e-3)."""
    x = orc.random_buffer(64, 13, batch=1)
    good = orc.forward(x, "dual", "fp64")
    bad = good.copy()
    bad[0, 5] = -bad[0, 5]
    assert orc.rel_l2(bad, orc.dft(x)) > 1e-3


def test_half_conversion_kat(orc):
    """acceptance.cpp:276-306 edge values."""
    cases = {65504.0: 65504.0, 65519.999: 65504.0, 65520.0: np.inf, 2049.0: 2048.0,
             1 + 2 ** -12: 1.0, 2 ** -25: 0.0, 1.5 * 2 ** -24: 2 ** -23, 1e300: np.inf}
    for x, want in cases.items():
        assert orc.round_to(np.array([x]), "fp16")[0] == want, x


def test_ctx_ops_match_reference(orc, ref):
    """The oracle's ArithmeticContext restatement == the reference's, for
    arbitrary doubles (the double-rounding of fp16 included)."""
    rng = np.random.RandomState(5)
    n = 20000
    mant = 1.0 + rng.randint(0, 1 << 52, size=(3, n)).astype(np.float64) * 2.0 ** -52
    x = np.ldexp(mant, rng.randint(-30, 18, size=(3, n))) * rng.choice([-1.0, 1.0], size=(3, n))
    for p in ("fp16", "fp32", "fp64"):
        for op in ("add", "sub", "mul", "fma"):
            a = orc.ctx_op(p, op, x[0], x[1], x[2])
            b = ref.ctx_op(p, op, x[0], x[1], x[2])
            assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), (p, op)
