"""The C++ drop-in (include/fmafft_b200.hpp, include/fmafft/*.hpp) against
libdsfft.so:

* tests/cpp/test_compat.cpp -- this repo's own checks of the mirror;
* the REFERENCE's own unit tests (proj/tests/test_fft.cpp, test_twiddle.cpp,
  test_butterfly.cpp, test_precision.cpp) and acceptance suite
  (acceptance.cpp, criteria 2-9), compiled unmodified from /root/reference by
  tests/cpp/Makefile with only the drop-in headers on the include path (the
  binaries are built here and travel to the GPU box).  The butterfly-variant
  API and the context's scalar operations run on the device
  (dsfft_butterflies / dsfft_context_ops).

Host-only parts run on CPU, the device parts on a B200."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2604_00567_b200")
BUILD = os.path.join(ROOT, "tests", "cpp", "_build")
REF_UNIT = os.path.join(BUILD, "ref_unit")
REF_ACCEPT = os.path.join(BUILD, "ref_acceptance")


@pytest.fixture(scope="module")
def exe(tmp_path_factory, dsfft):
    out = tmp_path_factory.mktemp("cpp") / "test_compat"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT}/include",
                    os.path.join(ROOT, "tests", "cpp", "test_compat.cpp"), "-o", str(out),
                    f"-L{PKG}", "-ldsfft", f"-Wl,-rpath,{PKG}"], check=True)
    return str(out)


@pytest.fixture(scope="module")
def ref_bins(dsfft):
    """The reference's tests built against the drop-in (here: rebuilt when
    /root/reference is present; on the GPU box: the binaries built here)."""
    if os.path.isdir("/root/reference/proj/tests"):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    if not (os.path.exists(REF_UNIT) and os.path.exists(REF_ACCEPT)):
        pytest.fail("tests/cpp/_build binaries missing: run __graft_entry__.build() where "
                    "/root/reference exists")
    return REF_UNIT, REF_ACCEPT


def test_cpp_dropin_host(exe):
    r = subprocess.run([exe, "host"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


def test_cpp_csv_dumps_match_reference(exe):
    """write_table_csv / write_bounds_csv through the C++ mirror == the
    reference's own serializer output (golden dumps), byte for byte."""
    import numpy as np
    g = np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))
    r = subprocess.run([exe, "csv"], capture_output=True, text=True, check=True)
    parts = r.stdout.split("== ")[1:]
    assert len(parts) == 11
    for part in parts:
        key, body = part.split("\n", 1)
        assert body.encode() == g[key].tobytes(), key


def test_reference_twiddle_tests_through_dropin(ref_bins):
    """proj/tests/test_twiddle.cpp (12 cases, host-side table builder)."""
    r = subprocess.run([ref_bins[0], "file:test_twiddle"], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "test cases: 12 | 12 passed | 0 failed" in r.stdout, r.stdout


def test_reference_host_acceptance_through_dropin(ref_bins):
    """acceptance.cpp criteria 2, 3, 4, 9 (bounds, tables, binary16)."""
    r = subprocess.run([ref_bins[1], "2", "3", "4", "9"], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("[PASS]") == 4, r.stdout


def test_reference_precision_host_cases_through_dropin(ref_bins):
    """proj/tests/test_precision.cpp: the five host-side cases (machine
    epsilon, round_to examples / idempotence, binary16 bit-exactness)."""
    r = subprocess.run([ref_bins[0], "machine epsilon,round_to,fp16 conversion"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "test cases: 5 | 5 passed | 0 failed" in r.stdout, r.stdout


@pytest.mark.gpu
def test_cpp_dropin_device(exe, cuda):
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


@pytest.mark.gpu
def test_reference_unit_tests_through_dropin(ref_bins, cuda):
    """ALL 43 cases of the reference's test_fft.cpp, test_twiddle.cpp,
    test_butterfly.cpp and test_precision.cpp pass on the B200 through the
    drop-in: plan construction, forward/inverse vs the (device) dft_oracle,
    op accounting, the corrupted-table negative control, non-finite
    propagation, every butterfly variant and the context's rounding."""
    r = subprocess.run([ref_bins[0]], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "test cases: 43 | 43 passed | 0 failed" in r.stdout, r.stdout


@pytest.mark.gpu
def test_reference_acceptance_through_dropin(ref_bins, cuda):
    """acceptance.cpp criteria 2-9 on the B200, within the reference's own
    per-criterion time budgets (5: fp64 oracle equivalence; 6: fp32
    roundtrip; 7: fp16 ordering and bounds; 8: op counts)."""
    r = subprocess.run([ref_bins[1]] + [str(i) for i in range(2, 10)], capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("[PASS]") == 8, r.stdout
