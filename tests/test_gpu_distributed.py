"""Batch sharding on the product (BASELINE configs[3]):

* dsfft_fill_uniform keys every sample by its GLOBAL transform index, so a
  shard generated alone equals the same rows of the whole batch (checked
  against a NumPy restatement, bit for bit, after the reference's round_to);
* bench.py --gpus 2 (self-launched under torch.distributed.run, two ranks;
  the gloo control plane lets them share this box's one GPU -- their kernels
  never wait on each other, there is no data-path collective) produces
  shards whose concatenation equals the 1-rank output bit for bit, reports
  n_gpus 2 and strong scaling over the global batch;
* the shards are the reference's transform of the same inputs."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from helpers import bit_mismatches, synth_reference, to_work

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _checker(orc):
    import oracle
    return oracle.load_ref() if oracle.ref_available() else orc


@pytest.mark.parametrize("precision", ["fp16", "fp32"])
def test_fill_uniform_global_index(dsfft, cuda, orc, precision):
    n, first, count, seed = 256, 37, 11, 99
    got = dsfft.synthetic_batch(n, first, count, seed, precision).cpu().numpy()
    raw = synth_reference(n, first, count, seed)
    want = orc.round_to(raw, precision).astype(got.dtype)
    assert bit_mismatches(got, want) == 0
    whole = dsfft.synthetic_batch(n, 0, first + count, seed, precision).cpu().numpy()
    assert whole[first:].tobytes() == got.tobytes()


def test_shards_equal_whole_batch(dsfft, cuda):
    from paper_2604_00567_b200.distributed import make_shard, sharded_forward
    plan = dsfft.make_plan(1024, "dual", "fp16")
    whole = sharded_forward(plan, make_shard(plan, 0, 1, 7, global_batch=1001))
    parts = [sharded_forward(plan, make_shard(plan, r, 3, 7, global_batch=1001))
             for r in range(3)]
    cuda.cuda.synchronize()
    assert [p.start for p in parts] == [0, 333, 667] and parts[-1].stop == 1001
    got = np.concatenate([p.y.cpu().numpy() for p in parts])
    assert got.tobytes() == whole.y.cpu().numpy().tobytes()


def _bench(args, env_extra=None):
    env = dict(os.environ, **(env_extra or {}))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args,
                       capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_two_ranks_bit_equal_to_one(tmp_path, orc):
    common = ["--n", "1024", "--global-batch", "4099", "--steps", "3", "--warmup", "3",
              "--no-e2e", "--no-cpu", "--no-accuracy", "--sustained-seconds", "0"]
    one = _bench(common + ["--gpus", "1", "--dump", str(tmp_path / "one")])
    two = _bench(common + ["--gpus", "2", "--dump", str(tmp_path / "two")],
                 {"DSFFT_DIST_BACKEND": "gloo"})
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert two["scaling"] == "strong" and two["config"]["global_batch"] == 4099
    assert two["gpu_launches"] == 3  # one fft_small_kernel per step per rank
    y1 = np.load(tmp_path / "one" / "shard0.npy")
    parts = [np.load(tmp_path / "two" / f"shard{r}.npy") for r in range(2)]
    ranges = [tuple(np.load(tmp_path / "two" / f"range{r}.npy")) for r in range(2)]
    assert ranges == [(0, 2049), (2049, 4099)]
    assert np.concatenate(parts).tobytes() == y1.tobytes()
    # and the reference's own forward of the same (regenerated) inputs
    chk = _checker(orc)
    rows = np.r_[0:3, 2047:2052, 4096:4099]
    x = orc.round_to(synth_reference(1024, 0, 4099, 20260419)[rows], "fp16")
    want = chk.forward(x.view(np.complex128)[..., 0], "dual", "fp16")
    assert bit_mismatches(y1[rows], to_work(want, "fp16")) == 0


def test_bench_rejects_wrong_world(tmp_path):
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--steps", "1", "--warmup", "3"], capture_output=True, text=True,
                       timeout=300, cwd=ROOT, env=env)
    assert r.returncode != 0 and "WORLD_SIZE=1" in r.stderr
