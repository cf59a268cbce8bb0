"""Device error harness (dsfft_error_device / dsfft_measure_error) vs the
reference's measure_error (analysis.cpp:101-154), pinned by the golden
reports the reference itself produced (tests/golden/make_golden.py), and the
reference's acceptance criteria 6-7 (acceptance.cpp:185-242) run on the GPU.

The device dft_oracle (fft.cpp:103-121) and the sequential relative_l2_error
(analysis.cpp:41-57) are bit-identical to the reference's, so the reports are
asserted EQUAL ("Equal arguments give bit-identical reports",
analysis.hpp:96-97), not close."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")
STRATS = ("standard", "lf", "cosine", "dual")


def _close(a, b, rel):
    if np.isinf(a) or np.isinf(b):
        return np.isinf(a) and np.isinf(b)
    return abs(a - b) <= rel * abs(b)


def _same(a, b):
    return a == b or (np.isnan(a) and np.isnan(b))


def test_forward_vs_oracle_matches_reference_reports(dsfft, cuda):
    """measure_error(forward_vs_oracle) on the device == the reference's own
    reports, bit for bit (device dft_oracle + sequential rel-L2)."""
    g = np.load(GOLDEN)["measure_error/forward/seed42/trials10"]
    for n, s, p, med, mx, nonfin in g:
        r = dsfft.measure_error(int(n), STRATS[int(s)], ("fp16", "fp32")[int(p)], "forward",
                                10, 42)
        assert r["nonfinite_trials"] == nonfin
        assert _same(r["rel_l2_median"], med), (n, s, p, r, med)
        assert _same(r["rel_l2_max"], mx), (n, s, p, r, mx)


def test_roundtrip_matches_reference_reports(dsfft, cuda):
    """Acceptance criterion 6 (acceptance.cpp:185-205): fp32 roundtrip medians
    in [1e-8, 1e-6] and within 3x; equal to the reference's reports."""
    g = np.load(GOLDEN)["measure_error/roundtrip/1024/fp32/lf_dual"]
    meds = []
    for (med, mx, nonfin), s in zip(g, ("lf", "dual")):
        r = dsfft.measure_error(1024, s, "fp32", "roundtrip", 100, 42)
        assert r["nonfinite_trials"] == nonfin
        assert _same(r["rel_l2_median"], med) and _same(r["rel_l2_max"], mx)
        assert 1e-8 <= r["rel_l2_median"] <= 1e-6
        meds.append(r["rel_l2_median"])
    assert 1 / 3 <= meds[0] / meds[1] <= 3


def test_fp16_ordering_and_bound_dominance(dsfft, cuda, orc):
    """Acceptance criterion 7 (acceptance.cpp:209-242) on the GPU: dual beats
    LF on 10/10 seeds at N=1024 and both maxima stay under Eq. 11."""
    eps = 2.0 ** -11
    lf_bound = orc.cumulative_bound(orc.table_stats(1024, "lf")["t_max"], eps, 10)
    du_bound = orc.cumulative_bound(orc.table_stats(1024, "dual")["t_max"], eps, 10)
    for seed in range(1, 11):
        lf = dsfft.measure_error(1024, "lf", "fp16", "forward", 10, seed)
        du = dsfft.measure_error(1024, "dual", "fp16", "forward", 10, seed)
        assert du["rel_l2_median"] < lf["rel_l2_median"]
        assert lf["rel_l2_max"] <= lf_bound and du["rel_l2_max"] <= du_bound


def test_whole_batch_errors(dsfft, cuda, orc):
    """Every transform of a device batch gets its own error."""
    torch = cuda
    n, batch = 1024, 4096
    x = orc.random_buffer(n, 5, batch=batch)
    xr = orc.round_to(x.view(np.float64), "fp16").astype(np.float16).reshape(batch, n, 2)
    plan = dsfft.make_plan(n, "dual", "fp16")
    rep, errs = dsfft.error_device(plan, torch.from_numpy(xr).cuda(), "forward",
                                   per_transform=True)
    assert rep["trials"] == batch and rep["nonfinite_trials"] == 0
    assert errs.shape == (batch,) and np.all(errs > 0) and np.all(errs < 4.89e-3)
    assert rep["rel_l2_max"] == errs.max()
    # transforms 0..7 against the reference's own dft_oracle + relative_l2_error
    chk = _checker(orc)
    xs = xr[:8].astype(np.float64).view(np.complex128)[..., 0]
    y = chk.forward(xs, "dual", "fp16")
    d = chk.dft(xs)
    for i in range(8):
        assert errs[i] == chk.rel_l2(y[i], d[i]), i


def _checker(orc):
    import oracle
    return oracle.load_ref() if oracle.ref_available() else orc


@pytest.mark.parametrize("n", [1, 2, 3, 4, 7, 8, 12, 64, 100, 1024, 4096, 5000, 8192])
def test_dft_oracle_bit_identical(dsfft, cuda, orc, n):
    """dft_oracle on the device == fft.cpp:103-121 bit for bit, any n
    (powers of two, odd and composite sizes; smem and global paths)."""
    chk = _checker(orc)
    batch = 3 if n <= 4096 else 1
    x = orc.random_buffer(n, 500 + n, batch=batch)
    got = dsfft.dft_oracle(x)
    want = chk.dft(x)
    assert got.tobytes() == want.tobytes()


def test_dft_device_stream_and_specials(dsfft, cuda, orc):
    """Device-buffer entry on a side stream; NaN / inf / signed zeros pass
    through the DFT exactly as in the reference."""
    torch = cuda
    chk = _checker(orc)
    n = 64
    x = orc.random_buffer(n, 9, batch=4)
    x[1, 3] = complex(np.nan, 0.0)
    x[2, 5] = complex(np.inf, -0.0)
    x[3, :] = complex(-0.0, 0.0)
    t = torch.from_numpy(x.copy()).cuda()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        y = dsfft.dft_device(t, stream=s.cuda_stream)
    s.synchronize()
    got = y.cpu().numpy()
    want = chk.dft(x)
    a, b = got.view(np.uint64), want.view(np.uint64)
    same = (a == b) | (np.isnan(got.view(np.float64)) & np.isnan(want.view(np.float64)))
    assert same.all()


@pytest.mark.parametrize("metric", ["forward", "roundtrip"])
@pytest.mark.parametrize("precision", ["fp16", "fp32"])
@pytest.mark.parametrize("n", [16, 1024, 4096])
def test_measure_error_equals_reference(dsfft, cuda, orc, n, precision, metric):
    """dsfft.measure_error == the reference's measure_error, every field."""
    chk = _checker(orc)
    for strategy in ("lf", "dual", "standard"):
        got = dsfft.measure_error(n, strategy, precision, metric, 6, 1234 + n)
        want = chk.measure_error(n, strategy, precision, metric, 6, 1234 + n)
        for k in ("trials", "seed", "nonfinite_trials"):
            assert got[k] == want[k], (k, got, want)
        for k in ("rel_l2_median", "rel_l2_max"):
            assert _same(got[k], want[k]), (k, got, want)


def test_error_device_reference_choice(dsfft, cuda, orc):
    """reference="fft64" (fast, fp64 FFT) agrees with the DFT to ~1e-9
    relative; "dft" is the exact one; unknown names raise."""
    torch = cuda
    n, batch = 1024, 64
    x = orc.random_buffer(n, 3, batch=batch)
    xr = orc.round_to(x.view(np.float64), "fp32").astype(np.float32).reshape(batch, n, 2)
    plan = dsfft.make_plan(n, "dual", "fp32")
    t = torch.from_numpy(xr).cuda()
    _, e_dft = dsfft.error_device(plan, t, "forward", per_transform=True, reference="dft")
    _, e_fft = dsfft.error_device(plan, t, "forward", per_transform=True, reference="fft64")
    _, e_auto = dsfft.error_device(plan, t, "forward", per_transform=True)
    assert np.array_equal(e_dft, e_auto)
    assert np.allclose(e_fft, e_dft, rtol=1e-6, atol=0)
    with pytest.raises(ValueError):
        dsfft.error_device(plan, t, "forward", reference="bogus")
