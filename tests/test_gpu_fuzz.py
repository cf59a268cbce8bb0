"""Randomised GPU parity (seeded): random sizes, strategies, precisions,
directions, odd batches, in-place or not -- every case bit-exact against the
reference (or the oracle).  Plus CUDA-graph capture of dsfft_execute."""
import os

import numpy as np
import pytest

from helpers import ALL_STRATEGIES, bit_mismatches, ref_inputs, to_work

pytestmark = pytest.mark.gpu


def _checker():
    import oracle
    return oracle.load_ref() if oracle.ref_available() else oracle.load_oracle()


# DSFFT_FUZZ_CASES / DSFFT_FUZZ_SEED widen the sweep for soak runs
_CASES = int(os.environ.get("DSFFT_FUZZ_CASES", "40"))
_SEED = int(os.environ.get("DSFFT_FUZZ_SEED", "1234"))
_MAXM = int(os.environ.get("DSFFT_FUZZ_MAXM", "15"))


@pytest.mark.parametrize("case", range(_CASES))
def test_random_cases(dsfft, cuda, orc, monkeypatch, case):
    torch = cuda
    rng = np.random.RandomState(_SEED + case)
    m = int(rng.choice(list(range(1, 16)) + list(range(16, _MAXM + 1))))
    n = 1 << m
    precision = str(rng.choice(["fp16", "fp32", "fp64"]))
    strategy = str(rng.choice(ALL_STRATEGIES))
    inverse = bool(rng.randint(2))
    in_place = bool(rng.randint(2))
    max_batch = max(1, (1 << 17) >> m)
    batch = int(rng.randint(1, max_batch + 1))
    # large-N path: the library default, forced two-launch, or forced fused
    fused = int(rng.randint(3)) - 1
    if fused < 0:
        monkeypatch.delenv("DSFFT_MP_FUSED", raising=False)
    else:
        monkeypatch.setenv("DSFFT_MP_FUSED", str(fused))
    x = ref_inputs(orc, n, batch, seed=case, precision=precision)
    xw = x if precision == "fp64" else to_work(x, precision)
    plan = dsfft.make_plan(n, strategy, precision)
    t = torch.from_numpy(np.ascontiguousarray(xw)).cuda()
    y = dsfft.execute(plan, int(inverse), t, out=t if in_place else None)
    torch.cuda.synchronize()
    got = y.cpu().numpy()
    want = (_checker().inverse if inverse else _checker().forward)(x, strategy, precision)
    if precision == "fp64":
        assert bit_mismatches(got.view(np.float64), want.view(np.float64)) == 0
    else:
        assert bit_mismatches(got, to_work(want, precision)) == 0, (n, strategy, precision,
                                                                   inverse, batch)


@pytest.mark.parametrize("n,precision", [(1024, "fp16"), (1 << 15, "fp16"), (512, "fp32"),
                                         (1 << 16, "fp16"), (1 << 14, "fp32"), (1 << 20, "fp32")])
def test_cuda_graph_capture(dsfft, cuda, orc, n, precision):
    """dsfft_execute is stream-ordered and capturable: a captured graph replays
    the same bits (multipass scratch becomes graph memory nodes; the fused
    one-launch path at 2^16 fp16 / 2^14 fp32 is a cooperative kernel node)."""
    torch = cuda
    batch = 8 if n < 1 << 20 else 2
    x = ref_inputs(orc, n, batch, seed=3, precision=precision)
    xt = torch.from_numpy(to_work(x, precision)).cuda()
    yt = torch.empty_like(xt)
    plan = dsfft.make_plan(n, "dual", precision)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        dsfft.forward(plan, xt, out=yt, stream=s.cuda_stream)  # warm-up (kernel attributes)
    s.synchronize()
    yt.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        dsfft.forward(plan, xt, out=yt, stream=s.cuda_stream)
    g.replay()
    torch.cuda.synchronize()
    want = to_work(_checker().forward(x, "dual", precision), precision)
    assert bit_mismatches(yt.cpu().numpy(), want) == 0
