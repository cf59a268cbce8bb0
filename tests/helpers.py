"""Shared test helpers: reference-protocol inputs and bitwise comparison."""
from __future__ import annotations

import numpy as np

WORK_DTYPE = {"fp16": np.float16, "fp32": np.float32}
ALL_STRATEGIES = ("standard", "lf", "cosine", "dual")


def ref_inputs(orc, n: int, batch: int, seed: int, precision: str) -> np.ndarray:
    """Reference protocol (analysis.cpp:120-130): one SplitMix64 stream, 2n
    uniform [-1,1) draws per transform (re then im), rounded into the working
    precision.  Returns complex128 [batch, n] holding representable values."""
    x = orc.random_buffer(n, seed, batch=batch)
    r = orc.round_to(x.view(np.float64), precision)
    return r.view(np.complex128).reshape(batch, n)


def to_work(x: np.ndarray, precision: str) -> np.ndarray:
    """complex128 (already rounded) -> interleaved working precision [.., n, 2]."""
    v = x.view(np.float64).reshape(*x.shape, 2)
    return v.astype(WORK_DTYPE[precision])  # exact: values are representable


def from_work(y: np.ndarray) -> np.ndarray:
    return y.astype(np.float64).view(np.complex128)[..., 0]


def bit_mismatches(a: np.ndarray, b: np.ndarray) -> int:
    """Count components whose bits differ, treating every NaN as equal."""
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    assert a.dtype == b.dtype and a.shape == b.shape
    ui = {2: np.uint16, 4: np.uint32, 8: np.uint64}[a.dtype.itemsize]
    same = a.view(ui) == b.view(ui)
    both_nan = np.isnan(a) & np.isnan(b)
    return int(np.count_nonzero(~(same | both_nan)))


def max_ulp_fp16(a: np.ndarray, b: np.ndarray) -> int:
    """Max distance in binary16 ULPs between finite components."""
    def ordered(x):
        u = x.view(np.uint16).astype(np.int32)
        return np.where(u & 0x8000, 0x8000 - (u & 0x7FFF), u + 0x8000)
    fin = np.isfinite(a) & np.isfinite(b)
    if not fin.any():
        return 0
    return int(np.max(np.abs(ordered(a[fin]) - ordered(b[fin]))))


def synth_reference(n: int, first: int, count: int, seed: int) -> np.ndarray:
    """NumPy restatement of dsfft_fill_uniform (csrc/synth.cu) before the
    working-precision rounding: float64 [count, n, 2] uniform [-1, 1) from a
    splitmix64 hash of (seed, global component index)."""
    with np.errstate(over="ignore"):
        c = np.uint64(2 * first * n) + np.arange(2 * n * count, dtype=np.uint64)
        z = np.uint64(seed) + np.uint64(0x9E3779B97F4A7C15) * (c + np.uint64(1))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return (2.0 * u - 1.0).reshape(count, n, 2)
