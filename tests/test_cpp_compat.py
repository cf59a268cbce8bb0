"""Build and run the C++ drop-in test (tests/cpp/test_compat.cpp) against
libdsfft.so: host-only checks on CPU, the full suite on a B200."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2604_00567_b200")


@pytest.fixture(scope="module")
def exe(tmp_path_factory, dsfft):
    out = tmp_path_factory.mktemp("cpp") / "test_compat"
    subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT}/include",
                    os.path.join(ROOT, "tests", "cpp", "test_compat.cpp"), "-o", str(out),
                    f"-L{PKG}", "-ldsfft", f"-Wl,-rpath,{PKG}"], check=True)
    return str(out)


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


@pytest.mark.gpu
def test_cpp_dropin_device(exe, cuda):
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
