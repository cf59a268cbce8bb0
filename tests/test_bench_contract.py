"""bench.py's JSON contract, checked on CPU through the reference arm
(`--impl reference` times the reference's own CPU path; no GPU needed)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line(orc, ref):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "0", "--cpu-seconds", "1"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # exactly one JSON line
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference"
    assert d["metric"] == "batched FFT transforms/s" and d["unit"] == "transforms/s"
    assert d["value"] > 0 and d["higher_is_better"] is True and d["scaling"] == "strong"
    assert d["config"]["global_batch"] == 1 << 20 and d["cpu_baseline"]["cpu_model"]
    assert d["steps"] == 1 and d["warmup"] == 0 and d["n_gpus"] == 1
    assert d["dtype"] == "f16" and d["vs_baseline"] is None
    assert "workload" in d["config"] and d["config"]["n"] == 1024
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert cb["unit"] == d["unit"] and cb["sample"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] == 0 and e["d2h_bytes_per_step"] == 0


def test_gpus_flag_self_launches_torchrun():
    """`bench.py --gpus 2` outside torchrun re-launches itself under
    torch.distributed.run with 2 ranks, passing every flag through (including
    ones torchrun's own parser would mistake, like --n).  Without a GPU each
    rank must then stop at the device check -- never at argument parsing."""
    import pytest
    import torch
    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--n",
                        "1024", "--steps", "1", "--warmup", "3"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode != 0
    out = r.stdout + r.stderr
    assert "ambiguous option" not in out and "unrecognized arguments" not in out, out[-2000:]
    assert out.count("bench.py: no CUDA device") == 2, out[-2000:]


def test_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode != 0 and "WORLD_SIZE=3" in r.stderr
