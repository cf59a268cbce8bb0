"""GPU parity: the sm_100a kernels through the C ABI vs the reference algorithm.

Bar (BASELINE.json north_star): fp32 bit-exact against the reference's own
fp32 path; fp16 within 2 binary16 ULP per output -- asserted here as
bit-exact, which the kernels achieve (every HFMA2 is the reference's single
rounding).  NaN payloads are compared as "both NaN".
Oracle: oracle/fmafft_oracle.c (pinned to the reference in test_oracle.py),
or the reference library itself when oracle/_ref was built.
"""
import numpy as np
import pytest

from helpers import ALL_STRATEGIES, bit_mismatches, max_ulp_fp16, ref_inputs, to_work

pytestmark = pytest.mark.gpu

SIZES = [2 ** m for m in range(1, 13)]


def _checker():
    import oracle
    return oracle.load_ref() if oracle.ref_available() else oracle.load_oracle()


def _device_run(dsfft, torch, plan, xw: np.ndarray, inverse: bool) -> np.ndarray:
    t = torch.from_numpy(np.ascontiguousarray(xw)).cuda()
    y = dsfft.execute(plan, 1 if inverse else 0, t)
    torch.cuda.synchronize()
    return y.cpu().numpy()


def _batch_for(n: int) -> int:
    return max(3, 65536 // n) + 1  # odd: exercises partial items / fp16 pair tails


@pytest.mark.parametrize("precision", ["fp32", "fp16"])
@pytest.mark.parametrize("strategy", ALL_STRATEGIES)
@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("inverse", [False, True], ids=["fwd", "inv"])
def test_bit_exact_vs_reference(dsfft, cuda, orc, n, strategy, precision, inverse):
    chk = _checker()
    batch = _batch_for(n)
    x = ref_inputs(orc, n, batch, seed=1000 + n, precision=precision)
    plan = dsfft.make_plan(n, strategy, precision)
    y = _device_run(dsfft, cuda, plan, to_work(x, precision), inverse)
    want = (chk.inverse if inverse else chk.forward)(x, strategy, precision)
    want_w = to_work(want, precision)
    bad = bit_mismatches(y, want_w)
    if precision == "fp16":
        assert max_ulp_fp16(y, want_w) <= 2  # the stated tolerance
    assert bad == 0, f"{bad} of {y.size} components differ"


@pytest.mark.parametrize("precision", ["fp32", "fp16"])
def test_many_items_per_group(dsfft, cuda, orc, precision):
    """Enough transforms that every persistent group cycles its buffer ring
    several times; spot-check a strided subset against the oracle."""
    chk = _checker()
    n = 1024
    batch = 148 * 16 * 2 * 3 + 5
    x = ref_inputs(orc, n, batch, seed=77, precision=precision)
    plan = dsfft.make_plan(n, "dual", precision)
    y = _device_run(dsfft, cuda, plan, to_work(x, precision), False)
    idx = np.r_[0:8, batch - 8:batch, 8:batch - 8:97]
    want = chk.forward(x[idx], "dual", precision)
    assert bit_mismatches(y[idx], to_work(want, precision)) == 0


def test_in_place_and_streams(dsfft, cuda, orc):
    torch = cuda
    n = 1024
    x = ref_inputs(orc, n, 64, seed=5, precision="fp16")
    plan = dsfft.make_plan(n, "dual", "fp16")
    t = torch.from_numpy(to_work(x, "fp16")).cuda()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        dsfft.forward(plan, t, out=t, stream=s.cuda_stream)
    s.synchronize()
    want = to_work(_checker().forward(x, "dual", "fp16"), "fp16")
    assert bit_mismatches(t.cpu().numpy(), want) == 0


def test_host_buffer_paths(dsfft, cuda, orc):
    """dsfft_execute_host (working precision) and dsfft_execute_f64 (the
    reference's double-carrier convention with ingest rounding)."""
    n = 256
    chk = _checker()
    raw = orc.random_buffer(n, 9, batch=301)  # unrounded doubles
    plan = dsfft.make_plan(n, "dual", "fp32")
    got = dsfft.forward_f64(plan, raw)
    want = chk.forward(raw, "dual", "fp32")  # forward rounds on ingest (fft.cpp:79-82)
    assert got.tobytes() == want.tobytes()
    xw = to_work(ref_inputs(orc, n, 301, 9, "fp32"), "fp32")
    out = np.empty_like(xw)
    dsfft.execute_host(plan, 0, xw, out, 301)
    assert bit_mismatches(out, to_work(want, "fp32")) == 0
    back = dsfft.inverse_f64(plan, got)
    assert back.tobytes() == chk.inverse(got, "dual", "fp32").tobytes()


@pytest.mark.parametrize("n,precision", [(1 << 16, "fp16"), (1 << 14, "fp32"), (1 << 20, "fp32")])
def test_host_pipeline_large_n(dsfft, cuda, orc, monkeypatch, n, precision):
    """dsfft_execute_host over small chunks: three pipe streams run chunk
    kernels concurrently -- for 2^16 fp16 / 2^14 fp32 these are the fused
    cooperative kernels -- and the result equals the reference's bits."""
    sb = 4 if precision == "fp16" else 8
    monkeypatch.setenv("DSFFT_HOST_CHUNK_MB", str(max(1, (4 * n * sb) >> 20)))
    batch = 37 if n < 1 << 20 else 5
    chk = _checker()
    x = ref_inputs(orc, n, batch, seed=n + 41, precision=precision)
    plan = dsfft.make_plan(n, "dual", precision)
    xw = to_work(x, precision)
    out = np.empty_like(xw)
    dsfft.execute_host(plan, 0, xw, out, batch)
    assert bit_mismatches(out, to_work(chk.forward(x, "dual", precision), precision)) == 0


def test_nonfinite_propagates(dsfft, cuda, orc):
    """test_fft.cpp:252-262: NaN input propagates; cosine fp16 is non-finite."""
    n = 8
    plan = dsfft.make_plan(n, "dual", "fp16")
    x = np.ones((1, n), dtype=np.complex128)
    x[0, 3] = complex(np.nan, 0.0)
    y = dsfft.forward_f64(plan, x)
    assert np.isnan(y).any()
    chk = _checker()
    xr = ref_inputs(orc, 1024, 4, 3, "fp16")
    plan = dsfft.make_plan(1024, "cosine", "fp16")
    y = _device_run(dsfft, cuda, plan, to_work(xr, "fp16"), False)
    assert not np.isfinite(y).all()
    assert bit_mismatches(y, to_work(chk.forward(xr, "cosine", "fp16"), "fp16")) == 0


def test_signed_zero_and_specials(dsfft, cuda, orc):
    chk = _checker()
    n = 64
    x = np.zeros((4, n), dtype=np.complex128)
    x[1] = -0.0
    x[2, ::3] = complex(-0.0, 0.0)
    x[3, 5] = complex(np.inf, -np.inf)
    for p in ("fp16", "fp32"):
        for s in ALL_STRATEGIES:
            plan = dsfft.make_plan(n, s, p)
            y = _device_run(dsfft, cuda, plan, to_work(x, p), False)
            assert bit_mismatches(y, to_work(chk.forward(x, s, p), p)) == 0, (p, s)


def test_errors(dsfft, cuda):
    with pytest.raises(ValueError, match="power of two"):
        dsfft.make_plan(1023, "dual", "fp16")
    with pytest.raises(ValueError, match="exceeds 2\\^24"):
        dsfft.make_plan(1 << 25, "dual", "fp16")
    with pytest.raises(ValueError, match="clamp_eps"):
        dsfft.make_plan(8, "lf", "fp32", clamp_eps=0.0)
    plan = dsfft.make_plan(64, "dual", "fp32")
    bad = cuda.zeros((2, 32, 2), dtype=cuda.float32, device="cuda")
    with pytest.raises(ValueError, match="does not match plan size"):
        dsfft.forward(plan, bad)
    with pytest.raises(ValueError, match="complex128"):
        dsfft.forward(dsfft.make_plan(64, "dual", "fp64"), bad)
    # raw C ABI: byte-count overflow and misalignment are refused, not launched
    lib = dsfft._load()
    buf = cuda.zeros(4096, dtype=cuda.uint8, device="cuda")
    ptr = buf.data_ptr()
    assert lib.dsfft_execute(plan._handle, 0, ptr, ptr, 1 << 62, None) == 1
    assert "overflows" in lib.dsfft_last_error().decode()
    assert lib.dsfft_execute(plan._handle, 0, ptr + 4, ptr + 4, 1, None) == 1
    assert "aligned" in lib.dsfft_last_error().decode()


@pytest.mark.parametrize("strategy", ALL_STRATEGIES)
@pytest.mark.parametrize("n", [2 ** m for m in (1, 2, 3, 5, 6, 8, 10, 12, 14, 16)])
@pytest.mark.parametrize("inverse", [False, True], ids=["fwd", "inv"])
def test_fp64_bit_exact(dsfft, cuda, orc, n, strategy, inverse):
    """Precision::fp64 (DFMA/DMUL/DADD per pass) == the reference's fp64."""
    chk = _checker()
    batch = 3
    x = orc.random_buffer(n, 40960 + 2 * n, batch=batch)
    plan = dsfft.make_plan(n, strategy, "fp64")
    t = cuda.from_numpy(np.ascontiguousarray(x)).cuda()
    y = dsfft.execute(plan, 1 if inverse else 0, t).cpu().numpy()
    want = (chk.inverse if inverse else chk.forward)(x, strategy, "fp64")
    assert bit_mismatches(y.view(np.float64), want.view(np.float64)) == 0


@pytest.mark.parametrize("m", [18, 20, 24])
def test_fp64_large_n(dsfft, cuda, orc, m):
    """fp64 per-pass kernels up to the 2^24 cap: bit-exact vs the reference."""
    chk = _checker()
    n = 1 << m
    x = orc.random_buffer(n, 7 + m, batch=1)
    t = cuda.from_numpy(np.ascontiguousarray(x)).cuda()
    for inverse in (False, True):
        y = dsfft.execute(dsfft.make_plan(n, "dual", "fp64"), int(inverse), t).cpu().numpy()
        want = (chk.inverse if inverse else chk.forward)(x, "dual", "fp64")
        assert bit_mismatches(y.view(np.float64), want.view(np.float64)) == 0, (m, inverse)


def test_fp64_oracle_equivalence(dsfft, cuda, orc):
    """test_fft.cpp:110-128 / acceptance criterion 5 through the device:
    every strategy within rel-L2 1e-11 of the FP64 DFT, n <= 4096."""
    for m in range(1, 13):
        n = 2 ** m
        x = orc.random_buffer(n, 40960 + 2 * n, batch=1)
        ref = orc.dft(x)
        for s in ALL_STRATEGIES:
            y = dsfft.forward_f64(dsfft.make_plan(n, s, "fp64"), x)
            assert orc.rel_l2(y, ref) < 1e-11, (n, s)


LARGE = [2 ** m for m in range(13, 21)]


@pytest.mark.parametrize("precision", ["fp32", "fp16"])
@pytest.mark.parametrize("n", LARGE)
@pytest.mark.parametrize("inverse", [False, True], ids=["fwd", "inv"])
def test_multipass_bit_exact(dsfft, cuda, orc, monkeypatch, n, precision, inverse):
    """N = 2^13..2^20: 2-3 pass-group launches (the two-launch path is forced
    where the fused one is the default; test_fused_* cover that one)."""
    monkeypatch.setenv("DSFFT_MP_FUSED", "0")
    chk = _checker()
    batch = 3 if n <= 1 << 16 else 2
    strategies = ALL_STRATEGIES if n <= 1 << 14 else ("dual", "lf")
    x = ref_inputs(orc, n, batch, seed=n + 7, precision=precision)
    for s in strategies:
        plan = dsfft.make_plan(n, s, precision)
        y = _device_run(dsfft, cuda, plan, to_work(x, precision), inverse)
        want = to_work((chk.inverse if inverse else chk.forward)(x, s, precision), precision)
        assert bit_mismatches(y, want) == 0, (n, s, precision)


@pytest.mark.parametrize("precision", ["fp32", "fp16"])
def test_multipass_at_8192(dsfft, cuda, orc, monkeypatch, precision):
    """N=8192 runs in the single kernel by default; its two-launch path
    (DSFFT_SMALL13=0) stays bit-exact too."""
    monkeypatch.setenv("DSFFT_SMALL13", "0")
    chk = _checker()
    x = ref_inputs(orc, 8192, 5, seed=8192 + 5, precision=precision)
    for inverse in (False, True):
        plan = dsfft.make_plan(8192, "dual", precision)
        y = _device_run(dsfft, cuda, plan, to_work(x, precision), inverse)
        want = to_work((chk.inverse if inverse else chk.forward)(x, "dual", precision), precision)
        assert bit_mismatches(y, want) == 0, (precision, inverse)
        assert dsfft.last_launch_count() == 2


@pytest.mark.parametrize("n,chunk_mb", [(1 << 16, 1), (1 << 20, 5)])
def test_multipass_in_place(dsfft, cuda, orc, monkeypatch, n, chunk_mb):
    """in == out through 2- and 3-group splits with odd chunks: a chunk's last
    group overwrites only input its first group has already consumed."""
    monkeypatch.setenv("DSFFT_MP_CHUNK_MB", str(chunk_mb))
    monkeypatch.setenv("DSFFT_MP_FUSED", "0")
    chk = _checker()
    x = ref_inputs(orc, n, 5, seed=n + 3, precision="fp16")
    plan = dsfft.make_plan(n, "dual", "fp16")
    t = cuda.from_numpy(to_work(x, "fp16")).cuda()
    dsfft.forward(plan, t, out=t)
    cuda.cuda.synchronize()
    want = to_work(chk.forward(x, "dual", "fp16"), "fp16")
    assert bit_mismatches(t.cpu().numpy(), want) == 0


@pytest.mark.parametrize("n", [1 << 15, 1 << 17, 1 << 19])
@pytest.mark.parametrize("precision", ["fp32", "fp16"])
@pytest.mark.parametrize("strategy", ["standard", "cosine"])
def test_multipass_other_variants(dsfft, cuda, orc, n, precision, strategy):
    """Standard and cosine through 2- and 3-group splits (cosine fp16 overflows
    to non-finite exactly where the reference does; compared as both-NaN)."""
    chk = _checker()
    x = ref_inputs(orc, n, 2, seed=n + 11, precision=precision)
    for inverse in (False, True):
        plan = dsfft.make_plan(n, strategy, precision)
        y = _device_run(dsfft, cuda, plan, to_work(x, precision), inverse)
        want = to_work((chk.inverse if inverse else chk.forward)(x, strategy, precision),
                       precision)
        assert bit_mismatches(y, want) == 0, (n, strategy, precision, inverse)


@pytest.mark.parametrize("m", [21, 22, 23, 24])
def test_multipass_largest_sizes(dsfft, cuda, orc, m):
    """Up to the reference's 2^24 cap (fft.cpp:14): one fp32 dual transform."""
    chk = _checker()
    n = 1 << m
    x = ref_inputs(orc, n, 1, seed=m, precision="fp32")
    plan = dsfft.make_plan(n, "dual", "fp32")
    y = _device_run(dsfft, cuda, plan, to_work(x, "fp32"), False)
    assert bit_mismatches(y, to_work(chk.forward(x, "dual", "fp32"), "fp32")) == 0


def test_multipass_many_chunks(dsfft, cuda, orc):
    """A batch spanning several L2 chunks (spot-checked transforms)."""
    chk = _checker()
    n = 1 << 16
    batch = 400  # 256 KiB per fp16 transform -> several 48 MiB chunks
    x = ref_inputs(orc, n, batch, seed=3, precision="fp16")
    plan = dsfft.make_plan(n, "dual", "fp16")
    y = _device_run(dsfft, cuda, plan, to_work(x, "fp16"), False)
    idx = np.array([0, 1, 191, 192, 193, 250, batch - 1])
    want = to_work(chk.forward(x[idx], "dual", "fp16"), "fp16")
    assert bit_mismatches(y[idx], want) == 0


@pytest.mark.parametrize("n,precision,chunk_mb,batch", [
    (1 << 18, "fp16", 3, 7),   # 3 transforms per chunk: odd chunks, pair straddles
    (1 << 16, "fp16", 1, 9),   # 4 per chunk, odd tail
    (1 << 20, "fp16", 5, 3),   # 3 pass groups, 1 transform per chunk
    (1 << 16, "fp32", 3, 5)])
@pytest.mark.parametrize("inverse", [False, True], ids=["fwd", "inv"])
def test_multipass_odd_chunks(dsfft, cuda, orc, monkeypatch, n, precision, chunk_mb, batch,
                              inverse):
    """Chunked batches whose chunks hold an odd number of transforms: fp16
    pair-packed intermediates and pair partners across chunk boundaries."""
    monkeypatch.setenv("DSFFT_MP_CHUNK_MB", str(chunk_mb))
    monkeypatch.setenv("DSFFT_MP_FUSED", "0")
    chk = _checker()
    x = ref_inputs(orc, n, batch, seed=n + batch, precision=precision)
    plan = dsfft.make_plan(n, "dual", precision)
    y = _device_run(dsfft, cuda, plan, to_work(x, precision), inverse)
    want = to_work((chk.inverse if inverse else chk.forward)(x, "dual", precision), precision)
    assert bit_mismatches(y, want) == 0


@pytest.mark.parametrize("n,precision", [(1024, "fp16"), (1 << 16, "fp16"), (1 << 14, "fp32"),
                                         (256, "fp64"), (2, "fp16")])
def test_one_plan_many_streams(dsfft, cuda, orc, n, precision):
    """Plans are shareable (fft.hpp:14-16): one plan executed concurrently on
    two streams from two host threads gives the single-stream bits."""
    import threading
    torch = cuda
    batch = 9 if n < (1 << 14) else 4
    x = ref_inputs(orc, n, batch, seed=n + 1, precision=precision if precision != "fp64" else
                   "fp64")
    xw = x if precision == "fp64" else to_work(x, precision)
    plan = dsfft.make_plan(n, "dual", precision)
    ins = [torch.from_numpy(np.ascontiguousarray(xw)).cuda() for _ in range(2)]
    outs = [torch.empty_like(ins[0]) for _ in range(2)]
    streams = [torch.cuda.Stream() for _ in range(2)]

    def work(i):
        for _ in range(3):
            dsfft.forward(plan, ins[i], out=outs[i], stream=streams[i].cuda_stream)

    th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    want = _checker().forward(x, "dual", precision)
    want = want if precision == "fp64" else to_work(want, precision)
    for o in outs:
        got = o.cpu().numpy()
        assert bit_mismatches(got.view(np.float64) if precision == "fp64" else got,
                              want.view(np.float64) if precision == "fp64" else want) == 0


def test_execute_multi_partitioner(dsfft, cuda, orc):
    """dsfft_execute_multi: contiguous shards on each listed device (here the
    one B200 twice, two host threads) reproduce the single-call result."""
    n, batch = 1024, 101
    x = to_work(ref_inputs(orc, n, batch, 21, "fp16"), "fp16")
    plans = [dsfft.make_plan(n, "dual", "fp16") for _ in range(2)]
    out = np.empty_like(x)
    dsfft.execute_multi(plans, 0, x, out, batch)
    single = np.empty_like(x)
    dsfft.execute_host(plans[0], 0, x, single, batch)
    assert out.tobytes() == single.tobytes()
    want = to_work(_checker().forward(ref_inputs(orc, n, batch, 21, "fp16"), "dual", "fp16"),
                   "fp16")
    assert bit_mismatches(out, want) == 0


def test_plan_lifecycle_releases_device_memory(dsfft, cuda):
    """Creating and destroying plans of every path (single kernel, multipass,
    fp64, host pipeline) returns their device memory."""
    import gc
    import numpy as np

    def cycle():
        for n, p in ((1024, "fp16"), (4096, "fp32"), (1 << 16, "fp16"), (1 << 20, "fp32"),
                     (256, "fp64")):
            plan = dsfft.make_plan(n, "dual", p)
            if p != "fp64":
                xw = np.zeros((2, n, 2), dtype=np.float16 if p == "fp16" else np.float32)
                dsfft.execute_host(plan, 0, xw, np.empty_like(xw), 2)
            del plan
        gc.collect()
        cuda.cuda.synchronize()

    cuda.cuda.synchronize()
    before, _ = cuda.cuda.mem_get_info()
    cycle()  # first use: lazy module loads (kernel code), context setup
    free0, _ = cuda.cuda.mem_get_info()
    # scratch pools are trimmed on plan destroy: only kernel code stays
    assert before - free0 < (128 << 20), (before, free0)
    for _ in range(5):
        cycle()
    free1, _ = cuda.cuda.mem_get_info()
    assert free0 - free1 < (64 << 20), (free0, free1)


@pytest.mark.parametrize("precision", ["fp16", "fp32"])
def test_headline_size_properties(dsfft, cuda, orc, precision):
    """BASELINE configs[1] at full size (N=1024, batch 2^20 fp16 / 2^19 fp32):
    64 sampled transforms bit-exact against the reference, the impulse maps to
    exact ones, and the round trip of every transform stays within the
    reference's fp32 window / the fp16 cumulative bound (analysis.cpp:61-63)."""
    torch = cuda
    n = 1024
    batch = (1 << 20) if precision == "fp16" else (1 << 19)
    wdt = torch.float16 if precision == "fp16" else torch.float32
    g = torch.Generator(device="cuda")
    g.manual_seed(99)
    x = (torch.rand((batch, n, 2), device="cuda", generator=g) * 2 - 1).to(wdt)
    x[7] = 0
    x[7, 0, 0] = 1  # impulse
    plan = dsfft.make_plan(n, "dual", precision)
    y = dsfft.forward(plan, x)
    torch.cuda.synchronize()
    idx = torch.randint(0, batch, (64,), generator=g, device="cuda").cpu().numpy()
    xs = x[idx].float().cpu().numpy().astype(np.float64)
    xs = (xs[..., 0] + 1j * xs[..., 1]).astype(np.complex128)
    want = to_work(_checker().forward(xs, "dual", precision), precision)
    assert bit_mismatches(y[idx].cpu().numpy(), want) == 0
    imp = y[7].float().cpu().numpy()
    assert (imp[:, 0] == 1).all() and (imp[:, 1] == 0).all()
    rep = dsfft.error_device(plan, x, "roundtrip")
    assert rep["trials"] == batch and rep["nonfinite_trials"] == 0
    if precision == "fp32":
        assert 1e-8 < rep["rel_l2_median"] < 1e-6  # acceptance.cpp:185-205
    else:
        assert rep["rel_l2_max"] < 2 * 0.0048935553178424129  # forward + inverse bound


@pytest.mark.parametrize("n,precision,sample", [(1 << 16, "fp16", 4), (1 << 20, "fp32", 2)])
def test_config5_size_properties(dsfft, cuda, orc, n, precision, sample):
    """BASELINE configs[4] sizes at a full 1 GiB batch: sampled transforms
    bit-exact against the reference and every transform's round trip finite
    and small (multipass path)."""
    torch = cuda
    sb = 4 if precision == "fp16" else 8
    batch = (1 << 30) // (n * sb)
    wdt = torch.float16 if precision == "fp16" else torch.float32
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    x = (torch.rand((batch, n, 2), device="cuda", generator=g) * 2 - 1).to(wdt)
    plan = dsfft.make_plan(n, "dual", precision)
    y = dsfft.forward(plan, x)
    torch.cuda.synchronize()
    idx = np.array([0, batch - 1] + list(range(1, batch - 1, max(1, batch // sample))))[:sample]
    xs = x[idx].float().cpu().numpy().astype(np.float64)
    xs = (xs[..., 0] + 1j * xs[..., 1]).astype(np.complex128)
    want = to_work(_checker().forward(xs, "dual", precision), precision)
    assert bit_mismatches(y[idx].cpu().numpy(), want) == 0
    # fp16 at 2^16: the reference's inverse scales after the transform
    # (fft.cpp:86-101), so an unscaled N*x overflows binary16 and the round trip
    # is non-finite by construction -- check the forward error instead, within
    # the paper's cumulative bound (1 + 2^-11)^16 - 1 (analysis.cpp:61-63)
    metric = "roundtrip" if precision == "fp32" else "forward"
    rep = dsfft.error_device(plan, x, metric)
    assert rep["trials"] == batch and rep["nonfinite_trials"] == 0
    assert rep["rel_l2_max"] < (5e-6 if precision == "fp32" else (1 + 2.0 ** -11) ** 16 - 1)


@pytest.mark.parametrize("n", [1 << 14, 1 << 16, 1 << 18])
@pytest.mark.parametrize("precision", ["fp16", "fp32"])
@pytest.mark.parametrize("inverse", [False, True], ids=["fwd", "inv"])
def test_fused_multipass_bit_exact(dsfft, cuda, orc, monkeypatch, n, precision, inverse):
    """The one-launch path (DSFFT_MP_FUSED=1, multipass_fused.cu): odd batch
    (a half-empty last fp16 pair), every strategy with a butterfly of its own."""
    monkeypatch.setenv("DSFFT_MP_FUSED", "1")
    chk = _checker()
    batch = 5 if n <= 1 << 16 else 3
    x = ref_inputs(orc, n, batch, seed=n + 17, precision=precision)
    for s in ("dual", "standard"):
        plan = dsfft.make_plan(n, s, precision)
        y = _device_run(dsfft, cuda, plan, to_work(x, precision), inverse)
        want = to_work((chk.inverse if inverse else chk.forward)(x, s, precision), precision)
        assert bit_mismatches(y, want) == 0, (n, s, precision, inverse)
        assert dsfft.last_launch_count() == 1


@pytest.mark.parametrize("n,precision,strategy,launches", [
    (1 << 14, "fp16", "dual", 1), (1 << 16, "fp16", "dual", 1), (1 << 18, "fp16", "dual", 2),
    (1 << 14, "fp32", "lf", 1), (1 << 16, "fp32", "dual", 2), (1 << 18, "fp32", "dual", 2),
    (1 << 15, "fp16", "dual", 2), (1 << 14, "fp16", "standard", 2),
    (1 << 16, "fp16", "cosine", 1)])
def test_default_large_n_path(dsfft, cuda, orc, monkeypatch, n, precision, strategy, launches):
    """With DSFFT_MP_FUSED unset the library takes the fused one-launch path
    exactly where the B200 A/B measured it faster (multipass.cu), bit-exact."""
    monkeypatch.delenv("DSFFT_MP_FUSED", raising=False)
    chk = _checker()
    x = ref_inputs(orc, n, 3, seed=n + 23, precision=precision)
    plan = dsfft.make_plan(n, strategy, precision)
    y = _device_run(dsfft, cuda, plan, to_work(x, precision), False)
    assert bit_mismatches(y, to_work(chk.forward(x, strategy, precision), precision)) == 0
    assert dsfft.last_launch_count() == launches


@pytest.mark.parametrize("n,precision", [(1 << 16, "fp16"), (1 << 14, "fp32")])
def test_fused_unfit_falls_back_to_two_launches(dsfft, cuda, orc, monkeypatch, n, precision):
    """A device that cannot hold one team co-resident (here: teams capped to
    fewer SMs than a team's K members) runs the same pass groups as two
    launches -- on the GPU, bit-exact -- instead of failing."""
    monkeypatch.delenv("DSFFT_MP_FUSED", raising=False)
    monkeypatch.setenv("DSFFT_FUSED_SMS", "2")
    chk = _checker()
    x = ref_inputs(orc, n, 3, seed=n + 29, precision=precision)
    plan = dsfft.make_plan(n, "dual", precision)
    y = _device_run(dsfft, cuda, plan, to_work(x, precision), True)
    assert bit_mismatches(y, to_work(chk.inverse(x, "dual", precision), precision)) == 0
    assert dsfft.last_launch_count() == 2


@pytest.mark.parametrize("lag,slots,teams", [(1, None, None), (2, None, 3), (1, 4, 1)])
def test_fused_multipass_slot_reuse(dsfft, cuda, orc, monkeypatch, lag, slots, teams):
    """Many units per team: scratch slots are reused for several generations
    (done / freed counters), with different lags, ring sizes and team counts;
    in place.  Sampled transforms against the reference."""
    monkeypatch.setenv("DSFFT_MP_FUSED", "1")
    monkeypatch.setenv("DSFFT_FUSED_LAG", str(lag))
    if slots:
        monkeypatch.setenv("DSFFT_FUSED_SLOTS", str(slots))
    if teams:
        monkeypatch.setenv("DSFFT_FUSED_TEAMS", str(teams))
    chk = _checker()
    n, batch = 1 << 14, 301
    x = ref_inputs(orc, n, batch, seed=99 + lag, precision="fp16")
    plan = dsfft.make_plan(n, "dual", "fp16")
    t = cuda.from_numpy(to_work(x, "fp16")).cuda()
    dsfft.forward(plan, t, out=t)  # in place
    cuda.cuda.synchronize()
    idx = np.array([0, 1, 2, 77, 150, 151, 298, 299, 300])
    want = to_work(chk.forward(x[idx], "dual", "fp16"), "fp16")
    assert bit_mismatches(t.cpu().numpy()[idx], want) == 0


def test_execute_validates_out(dsfft, cuda):
    """`out` must match the input exactly (advisor finding: a short or
    mistyped `out` would otherwise be written out of bounds)."""
    torch = cuda
    plan = dsfft.make_plan(1024, "dual", "fp16")
    x = torch.zeros((4, 1024, 2), dtype=torch.float16, device="cuda")
    for bad in (torch.zeros((3, 1024, 2), dtype=torch.float16, device="cuda"),
                torch.zeros((4, 1024, 2), dtype=torch.float32, device="cuda"),
                torch.zeros((4, 2, 1024), dtype=torch.float16, device="cuda").transpose(1, 2),
                torch.zeros((4, 1024, 2), dtype=torch.float16)):
        with pytest.raises(ValueError):
            dsfft.forward(plan, x, out=bad)
    with pytest.raises(ValueError):
        dsfft.forward(dsfft.make_plan(512, "dual", "fp16"), x)
    with pytest.raises(ValueError):
        dsfft.error_device(plan, x, reference="nope")
