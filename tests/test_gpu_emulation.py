"""The reference's fine-grained arithmetic APIs on the device, bit for bit:
ArithmeticContext::add/sub/mul/fma (precision.cpp:77-111) and the
butterfly-variant kernels (butterfly.cpp:37-90, kernel_for) -- for any double
inputs: representable ones, arbitrary doubles (double rounding exactly as the
reference does it), overflow boundaries, subnormals, signed zeros, inf, NaN."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

PRECS = ("fp16", "fp32", "fp64")
STRATS = ("standard", "lf", "cosine", "dual")


def _checker(orc):
    import oracle
    return oracle.load_ref() if oracle.ref_available() else orc


def _same(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return bool(np.all((a.view(np.uint64) == b.view(np.uint64)) | (np.isnan(a) & np.isnan(b))))


def _operands(rng, n):
    mant = 1.0 + rng.randint(0, 1 << 52, size=n).astype(np.float64) * 2.0 ** -52
    x = np.ldexp(mant, rng.randint(-30, 18, size=n)) * rng.choice([-1.0, 1.0], size=n)
    edge = np.array([0.0, -0.0, 65504.0, 65519.999, 65520.0, -65520.0, 2049.0, 2.0 ** -24,
                     2.0 ** -25, 1.5 * 2.0 ** -24, 1e-7, 1e300, -1e300, np.inf, -np.inf, np.nan,
                     3.4028235677973366e38, 3.4028234663852886e38, 1.0 + 2.0 ** -12])
    return np.concatenate([x, edge])


@pytest.mark.parametrize("precision", PRECS)
@pytest.mark.parametrize("op", ["add", "sub", "mul", "fma"])
def test_context_ops_bit_identical(dsfft, cuda, orc, precision, op):
    rng = np.random.RandomState(7 + len(op))
    n = 4000
    a = _operands(rng, n)
    b = np.roll(_operands(rng, n), 3)
    c = np.roll(_operands(rng, n), 7)
    got = dsfft.context_op(precision, op, a, b, c)
    want = _checker(orc).ctx_op(precision, op, a, b, c)
    assert _same(got, want)


@pytest.mark.parametrize("precision", PRECS)
@pytest.mark.parametrize("strategy", STRATS)
def test_butterflies_bit_identical(dsfft, cuda, orc, strategy, precision):
    """Every entry of the plan table (rounded into the precision, clamped LF
    k=0 included) against random and special operands."""
    chk = _checker(orc)
    n = 256
    rng = np.random.RandomState(11)
    tab = dsfft.build_table(n, strategy, precision)
    k = np.arange(len(tab)).repeat(3)
    entries = tab[k]
    vals = _operands(rng, 2 * len(k))[: 2 * len(k)]
    vals = np.concatenate([vals, rng.uniform(-1, 1, size=4 * len(k))])
    a = (vals[0::4][: len(k)] + 1j * vals[1::4][: len(k)])
    b = (vals[2::4][: len(k)] + 1j * vals[3::4][: len(k)])
    s, d = dsfft.butterflies(strategy, precision, a, b, entries)
    for i in range(len(k)):
        ws, wd, _ = chk.butterfly(strategy, precision, a[i], b[i], entries[i])
        assert _same([s[i].real, s[i].imag, d[i].real, d[i].imag],
                     [ws.real, ws.imag, wd.real, wd.imag]), (i, strategy, precision)


def test_unknown_arguments_raise(dsfft, cuda):
    with pytest.raises(ValueError):
        dsfft.context_op("fp16", "div", [1.0], [2.0])
    with pytest.raises(ValueError):
        dsfft.butterflies("nope", "fp16", [1j], [1j], dsfft.build_table(4, "dual", "fp16")[:1])
