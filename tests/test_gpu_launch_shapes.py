"""Bit-exactness across launch shapes: every ring depth / tile-group count /
lag the tuning knobs allow (tools/gpu_tune.sh) runs the same butterflies, so
any mbarrier / ring / flag ordering bug would surface here as a mismatch under
some shape (compute-sanitizer is closed on this pool; this is the race
evidence we can produce).  Small batches that still cycle every ring."""
import numpy as np
import pytest

from helpers import bit_mismatches, ref_inputs, to_work

pytestmark = pytest.mark.gpu


def _checker():
    import oracle
    return oracle.load_ref() if oracle.ref_available() else oracle.load_oracle()


def _run(dsfft, torch, orc, n, precision, batch, inverse=False, seed=0):
    x = ref_inputs(orc, n, batch, seed=seed or n + batch, precision=precision)
    plan = dsfft.make_plan(n, "dual", precision)
    t = torch.from_numpy(to_work(x, precision)).cuda()
    y = dsfft.execute(plan, int(inverse), t)
    torch.cuda.synchronize()
    want = (_checker().inverse if inverse else _checker().forward)(x, "dual", precision)
    return bit_mismatches(y.cpu().numpy(), to_work(want, precision))


@pytest.mark.parametrize("stages", [1, 2, 3, 4])
@pytest.mark.parametrize("groups", [1, 4, 8, 16])
@pytest.mark.parametrize("n,precision", [(64, "fp16"), (1024, "fp16"), (1024, "fp32"),
                                         (4096, "fp16")])
def test_single_kernel_shapes(dsfft, cuda, orc, monkeypatch, n, precision, groups, stages):
    monkeypatch.setenv("DSFFT_STAGES", str(stages))
    monkeypatch.setenv("DSFFT_GROUPS", str(groups))
    batch = 148 * 4 * 2 + 3  # several items per group, odd tail
    assert _run(dsfft, cuda, orc, n, precision, batch) == 0


@pytest.mark.parametrize("stages,groups", [(1, 1), (2, 1), (1, 2), (3, 2), (2, 4)])
@pytest.mark.parametrize("n,precision", [(1 << 14, "fp16"), (1 << 16, "fp32"),
                                         (1 << 19, "fp16")])
def test_multipass_shapes(dsfft, cuda, orc, monkeypatch, n, precision, stages, groups):
    monkeypatch.setenv("DSFFT_MP_FUSED", "0")  # the shapes are the two-launch kernel's
    monkeypatch.setenv("DSFFT_MP_STAGES", str(stages))
    monkeypatch.setenv("DSFFT_MP_GROUPS", str(groups))
    assert _run(dsfft, cuda, orc, n, precision, 5 if n <= 1 << 16 else 3, inverse=True) == 0


@pytest.mark.parametrize("lag,slots,teams", [(1, 2, None), (3, 8, None), (2, 6, 2), (1, 4, 1)])
@pytest.mark.parametrize("n,precision", [(1 << 14, "fp32"), (1 << 16, "fp16")])
def test_fused_shapes(dsfft, cuda, orc, monkeypatch, n, precision, lag, slots, teams):
    """The one-launch kernel's team / ring / lag protocol under tight rings
    (R = 2 units: every slot reused immediately) and few teams."""
    monkeypatch.setenv("DSFFT_MP_FUSED", "1")
    monkeypatch.setenv("DSFFT_FUSED_LAG", str(lag))
    monkeypatch.setenv("DSFFT_FUSED_SLOTS", str(slots))
    if teams:
        monkeypatch.setenv("DSFFT_FUSED_TEAMS", str(teams))
    assert _run(dsfft, cuda, orc, n, precision, 37 if n == 1 << 14 else 13) == 0


@pytest.mark.parametrize("mask", [1, 2, 3])
@pytest.mark.parametrize("precision", ["fp16", "fp32"])
def test_s10_tile_widths(dsfft, cuda, orc, monkeypatch, precision, mask):
    """s = 10 pass groups on 8- or 16-column tiles (DSFFT_MP_CW10MASK; the
    default is 8 for the fp32 first group only), N = 2^20, inverse."""
    monkeypatch.setenv("DSFFT_MP_CW10MASK", str(mask))
    assert _run(dsfft, cuda, orc, 1 << 20, precision, 3, inverse=True) == 0
