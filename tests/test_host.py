"""CPU-side checks of the product: the C ABI library loads and exports every
symbol include/dsfft.h declares; the host table builder and ingest rounding are
bit-identical to the reference; errors mirror the reference's messages; the
product refuses to run without a B200 (no CPU fallback); the kernel schedules
are dataflow-exact (tools/schedule_check.cpp)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from helpers import ALL_STRATEGIES

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def header_symbols():
    text = open(os.path.join(ROOT, "include", "dsfft.h")).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(dsfft_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol(dsfft):
    lib = ctypes.CDLL(dsfft.library_path())
    syms = header_symbols()
    assert len(syms) >= 14
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_sm100a_only():
    """The fatbin carries sm_100a SASS (no PTX/other-arch fallback images)."""
    import paper_2604_00567_b200 as d
    out = subprocess.run(["cuobjdump", "--list-elf", d.library_path()], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    archs = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert archs == {"100a"}, archs


def test_host_tables_match_golden(dsfft):
    g = np.load(GOLDEN)
    for key in g.files:
        if key.startswith("table/"):
            _, n, s, p = key.split("/")
            assert dsfft.build_table(int(n), s, p).tobytes() == g[key].tobytes(), key


def test_host_tables_match_reference(dsfft, ref):
    for m in range(1, 21):
        n = 2 ** m
        for s in ALL_STRATEGIES:
            for p in ("fp16", "fp32", "fp64"):
                assert dsfft.build_table(n, s, p).tobytes() == ref.plan_table(n, s, p).tobytes()


def test_lf_clamp_eps_matches_reference(dsfft, ref):
    """build_table(n, linzer_feig, clamp_eps) (twiddle.cpp:74-95) for non-default
    clamps, incl. values that round to zero / subnormal in binary16."""
    for eps in (1e-3, 1e-5, 2.0 ** -24, 1e-9, 1e-12, 0.5):
        for n in (2, 16, 1024):
            got = dsfft.build_table(n, "lf", "fp64", clamp_eps=eps)
            want = ref.build_table(n, "lf", clamp_eps=eps)
            assert got.tobytes() == want.tobytes(), (eps, n)
            for p in ("fp16", "fp32"):  # the rounded entries, eps rounded once
                g = dsfft.build_table(n, "lf", p, clamp_eps=eps)
                w = want.copy()
                for f in ("multiplier", "ratio", "omega_r", "omega_i"):
                    w[f] = dsfft.widen(dsfft.round_to(want[f], p), p)
                assert g.tobytes() == w.tobytes(), (eps, n, p)


def test_table_csv_matches_reference_writer(dsfft):
    """dsfft_table_csv == the reference's write_table_csv (serialize.cpp:48-57),
    byte for byte (golden dumps produced by the reference's own serializer)."""
    g = np.load(GOLDEN)
    keys = [k for k in g.files if k.startswith("csv/")]
    assert len(keys) >= 5
    for key in keys:
        _, n, s, p = key.split("/")
        assert dsfft.table_csv(int(n), s, p).encode() == g[key].tobytes(), key
    with pytest.raises(ValueError, match="power of two"):
        dsfft.table_csv(12, "dual")


def test_bounds_csv_matches_reference_writer(dsfft):
    """dsfft_bounds_csv == write_bounds_csv (serialize.cpp:79-91) of
    reproduce_ratio_table / reproduce_cumulative_table (analysis.cpp:65-88),
    byte for byte (golden dumps from the reference's own code)."""
    g = np.load(GOLDEN)
    keys = [k for k in g.files if k.startswith("bounds/")]
    assert len(keys) >= 8
    for key in keys:
        _, n, kind, p = key.split("/")
        assert dsfft.bounds_csv(int(n), kind, p).encode() == g[key].tobytes(), key
    text = dsfft.bounds_csv(1024, "stats")
    rows = [r.split(",") for r in text.strip().split("\n")[1:]]
    # Table I: LF t_max 163 at k=1, dual 1.0, one LF singularity
    assert [r[0] for r in rows] == ["lf", "cosine", "dual"]
    assert abs(float(rows[0][1]) - 162.97) < 0.01 and rows[0][2] == "1" and rows[0][3] == "1"
    assert abs(float(rows[2][1]) - 1.0) < 1e-15 and rows[2][3] == "0"
    assert abs(float(rows[2][8]) - 235.1) < 0.01  # dual vs LF
    with pytest.raises(ValueError, match="power of two"):
        dsfft.bounds_csv(1000)
    with pytest.raises(ValueError, match="unknown statistics kind"):
        dsfft.bounds_csv(64, "histogram")


def test_ingest_rounding_matches_oracle(dsfft, orc):
    rng = np.random.RandomState(916)
    x = (1 + rng.randint(0, 1 << 52, 300000) * 2.0 ** -52) * np.exp2(rng.randint(-30, 21, 300000))
    x *= np.where(rng.randint(0, 2, 300000), -1.0, 1.0)
    x = np.concatenate([x, [0.0, -0.0, 65504.0, 65519.999, 65520.0, -65520.0, 2049.0,
                            1 + 2 ** -12, 2 ** -24, 2 ** -25, 1.5 * 2 ** -24, 1e-7, 1e300,
                            -1e300, np.inf, -np.inf, 5e-324, 3.4028235e38, 3.5e38]])
    for p in ("fp16", "fp32"):
        got = dsfft.widen(dsfft.round_to(x, p), p)
        assert got.tobytes() == orc.round_to(x, p).tobytes(), p
    # every binary16 value round-trips exactly
    allh = np.arange(1 << 16, dtype=np.uint16).view(np.float16)
    fin = allh[np.isfinite(allh)].astype(np.float64)
    assert dsfft.widen(dsfft.round_to(fin, "fp16"), "fp16").tobytes() == fin.tobytes()


def test_error_messages_mirror_reference(dsfft):
    with pytest.raises(ValueError, match="FFT size must be a power of two >= 2, got 1023"):
        dsfft.build_table(1023, "dual", "fp16")
    with pytest.raises(ValueError, match="FFT size must be a power of two >= 2, got 1"):
        dsfft.build_table(1, "dual", "fp16")
    with pytest.raises(ValueError, match="exceeds 2\\^24"):
        dsfft.build_table(1 << 25, "dual", "fp16")
    with pytest.raises(ValueError, match="clamp_eps must be positive"):
        dsfft.build_table(8, "lf", "fp32", clamp_eps=-1.0)
    with pytest.raises(ValueError, match="unknown strategy"):
        dsfft.parse_strategy("radix4")
    with pytest.raises(ValueError, match="unknown precision"):
        dsfft.parse_precision("bf16")
    assert dsfft.parse_strategy("linzer-feig") == "lf"
    assert dsfft.parse_strategy("dual_select") == "dual"


def test_no_cpu_fallback_without_device(dsfft):
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(dsfft.DsfftError, match="no CPU fallback|not sm_100"):
        dsfft.make_plan(1024, "dual", "fp16")
    # every precision runs on the device only, never emulated on the host
    with pytest.raises(dsfft.DsfftError, match="no CPU fallback|not sm_100"):
        dsfft.make_plan(64, "dual", "fp64")


def test_schedule_dataflow_exact(tmp_path):
    """Replays every shipped kernel schedule symbolically against run_passes."""
    exe = tmp_path / "sc"
    subprocess.run(["g++", "-O2", "-std=c++17", f"-I{ROOT}/paper_2604_00567_b200/csrc",
                    f"{ROOT}/tools/schedule_check.cpp", "-o", str(exe)], check=True)
    src = open(os.path.join(ROOT, "paper_2604_00567_b200", "csrc", "inst_small.cu")).read()
    cfgs = re.findall(r"Sched<(\d+), (\d+), (\d+), ([\d, ]+)>", src)
    assert len(cfgs) >= 7
    for m, le, w, stages in cfgs:
        args = [m, le, w] + [s.strip() for s in stages.split(",")]
        r = subprocess.run([str(exe)] + args, capture_output=True, text=True)
        assert r.returncode == 0 and "BAD" not in r.stdout, r.stdout
    for m in range(1, 6):  # the single-stage configs Sched<M, 5, 1, M>
        r = subprocess.run([str(exe), str(m), "5", "1", str(m)], capture_output=True, text=True)
        assert r.returncode == 0, r.stdout
