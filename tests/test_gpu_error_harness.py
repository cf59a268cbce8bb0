"""Device error harness (dsfft_error_device / dsfft_measure_error) vs the
reference's measure_error (analysis.cpp:101-154), pinned by the golden
reports the reference itself produced (tests/golden/make_golden.py), and the
reference's acceptance criteria 6-7 (acceptance.cpp:185-242) run on the GPU."""
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


def test_forward_vs_oracle_matches_reference_reports(dsfft, cuda):
    """FP64 reference = device fp64 transform instead of the O(n^2) DFT: the
    reported errors agree with the reference's to ~1e-9 relative."""
    g = np.load(GOLDEN)["measure_error/forward/seed42/trials10"]
    for n, s, p, med, mx, nonfin in g:
        r = dsfft.measure_error(int(n), STRATS[int(s)], ("fp16", "fp32")[int(p)], "forward",
                                10, 42)
        assert r["nonfinite_trials"] == nonfin
        assert _close(r["rel_l2_median"], med, 1e-6), (n, s, p, r, med)
        assert _close(r["rel_l2_max"], mx, 1e-6), (n, s, p, r, mx)


def test_roundtrip_matches_reference_reports(dsfft, cuda):
    """Acceptance criterion 6 (acceptance.cpp:185-205): fp32 roundtrip medians
    in [1e-8, 1e-6] and within 3x; equal to the reference's reports."""
    g = np.load(GOLDEN)["measure_error/roundtrip/1024/fp32/lf_dual"]
    meds = []
    for (med, mx, nonfin), s in zip(g, ("lf", "dual")):
        r = dsfft.measure_error(1024, s, "fp32", "roundtrip", 100, 42)
        assert r["nonfinite_trials"] == nonfin
        assert _close(r["rel_l2_median"], med, 1e-9) and _close(r["rel_l2_max"], mx, 1e-9)
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
    # spot-check transform 7 against the oracle's FP64 DFT
    y = orc.forward(xr[7:8].astype(np.float64).view(np.complex128)[..., 0], "dual", "fp16")
    e7 = orc.rel_l2(y, orc.dft(xr[7:8].astype(np.float64).view(np.complex128)[..., 0]))
    assert abs(errs[7] - e7) <= 1e-6 * e7
