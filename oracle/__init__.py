"""TEST INFRASTRUCTURE ONLY -- ctypes loaders for the parity oracle.

``load_oracle()`` returns the C restatement (oracle/liboracle.so, built from
fmafft_oracle.c) and ``load_ref()`` the reference library compiled unmodified
from /root/reference (oracle/_ref/libfmafft_ref.so).  Both expose the same
function set (prefix ``orc_`` / ``ref_``) wrapped by :class:`CpuFft`.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this package; the product
(paper_2604_00567_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfmafft_ref.so")

STRATEGIES = {"standard": 0, "lf": 1, "cosine": 2, "dual": 3}
PRECISIONS = {"fp16": 0, "fp32": 1, "fp64": 2}


class Entry(C.Structure):
    _fields_ = [("multiplier", C.c_double), ("ratio", C.c_double),
                ("path", C.c_int32), ("clamped", C.c_int32),
                ("omega_r", C.c_double), ("omega_i", C.c_double)]


ENTRY_DTYPE = np.dtype([("multiplier", "<f8"), ("ratio", "<f8"), ("path", "<i4"),
                        ("clamped", "<i4"), ("omega_r", "<f8"), ("omega_i", "<f8")])


class Counters(C.Structure):
    _fields_ = [("fma_count", C.c_uint64), ("add_count", C.c_uint64),
                ("mul_count", C.c_uint64)]


class ErrorReport(C.Structure):
    _fields_ = [("n", C.c_uint64), ("strategy", C.c_int32), ("precision", C.c_int32),
                ("metric", C.c_int32), ("pad_", C.c_int32), ("trials", C.c_uint64),
                ("seed", C.c_uint64), ("rel_l2_median", C.c_double),
                ("rel_l2_max", C.c_double), ("nonfinite_trials", C.c_uint64)]


def build(quiet: bool = True) -> None:
    """Compile liboracle.so (and _ref when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


_DP = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


class CpuFft:
    """Thin typed wrapper over liboracle.so / libfmafft_ref.so."""

    def __init__(self, path: str, prefix: str):
        self.path = path
        self.prefix = prefix
        self.lib = C.CDLL(path)
        f = self._f
        f("last_error").restype = C.c_char_p
        f("round_to").restype = C.c_double
        f("round_to").argtypes = [C.c_double, C.c_int]
        f("round_array").argtypes = [_DP, _DP, C.c_size_t, C.c_int]
        f("machine_epsilon").restype = C.c_double
        f("machine_epsilon").argtypes = [C.c_int]
        for name in ("build_table",):
            f(name).argtypes = [C.c_size_t, C.c_int, C.c_double, C.c_void_p]
        f("plan_table").argtypes = [C.c_size_t, C.c_int, C.c_int, C.c_void_p]
        for name in ("forward", "inverse"):
            f(name).argtypes = [C.c_size_t, C.c_int, C.c_int, _DP, _DP, C.c_size_t,
                                C.c_int, C.POINTER(Counters)]
        f("butterfly").argtypes = [C.c_int, C.c_int, _DP, _DP, C.POINTER(Entry), _DP,
                                   C.POINTER(Counters)]
        f("ctx_op").argtypes = [C.c_int, C.c_int, _DP, _DP, _DP, _DP, C.c_size_t]
        f("rel_l2").restype = C.c_double
        f("rel_l2").argtypes = [_DP, _DP, C.c_size_t]
        f("cumulative_bound").restype = C.c_double
        f("cumulative_bound").argtypes = [C.c_double, C.c_double, C.c_uint]
        f("splitmix_uniform").argtypes = [C.c_uint64, _DP, C.c_size_t]
        f("measure_error").argtypes = [C.c_size_t, C.c_int, C.c_int, C.c_int,
                                       C.c_size_t, C.c_uint64, C.POINTER(ErrorReport)]
        f("table_stats").argtypes = [C.c_size_t, C.c_int, C.POINTER(C.c_double)] + \
            [C.POINTER(C.c_uint64)] * 4

    def _f(self, name):
        return getattr(self.lib, f"{self.prefix}_{name}")

    def _check(self, rc: int) -> None:
        if rc != 0:
            raise ValueError(self._f("last_error")().decode())

    # -- precision --------------------------------------------------------
    def round_to(self, x, precision: str):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty_like(x)
        self._f("round_array")(x.ravel(), out.ravel(), x.size, PRECISIONS[precision])
        return out

    def machine_epsilon(self, precision: str) -> float:
        return self._f("machine_epsilon")(PRECISIONS[precision])

    # -- tables -----------------------------------------------------------
    def build_table(self, n: int, strategy: str, clamp_eps: float = 1e-7):
        out = np.zeros(max(n // 2, 1), dtype=ENTRY_DTYPE)
        self._check(self._f("build_table")(n, STRATEGIES[strategy], clamp_eps,
                                           out.ctypes.data))
        return out[: n // 2]

    def plan_table(self, n: int, strategy: str, precision: str):
        out = np.zeros(max(n // 2, 1), dtype=ENTRY_DTYPE)
        self._check(self._f("plan_table")(n, STRATEGIES[strategy], PRECISIONS[precision],
                                          out.ctypes.data))
        return out[: n // 2]

    def table_stats(self, n: int, strategy: str):
        t = C.c_double()
        a, s, c, si = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        self._check(self._f("table_stats")(n, STRATEGIES[strategy], C.byref(t), C.byref(a),
                                           C.byref(s), C.byref(c), C.byref(si)))
        return dict(t_max=t.value, argmax_k=a.value, singular_count=s.value,
                    cos_path_count=c.value, sin_path_count=si.value)

    # -- transforms -------------------------------------------------------
    def _run(self, name, x, strategy, precision, threads):
        x = np.ascontiguousarray(x, dtype=np.complex128)
        n = x.shape[-1]
        batch = x.size // n if n else 0
        src = x.view(np.float64).ravel()
        out = np.empty_like(src)
        cnt = Counters()
        self._check(self._f(name)(n, STRATEGIES[strategy], PRECISIONS[precision], src, out,
                                  batch, threads, C.byref(cnt)))
        return out.view(np.complex128).reshape(x.shape), cnt

    def forward(self, x, strategy: str, precision: str, threads: int = 0,
                counters: bool = False):
        y, c = self._run("forward", x, strategy, precision, threads)
        return (y, c) if counters else y

    def inverse(self, x, strategy: str, precision: str, threads: int = 0,
                counters: bool = False):
        y, c = self._run("inverse", x, strategy, precision, threads)
        return (y, c) if counters else y

    def butterfly(self, strategy, precision, a, b, entry):
        e = Entry(*[entry[k] for k in ("multiplier", "ratio", "path", "clamped",
                                       "omega_r", "omega_i")])
        out = np.zeros(4)
        cnt = Counters()
        self._check(self._f("butterfly")(STRATEGIES[strategy], PRECISIONS[precision],
                                         np.array([a.real, a.imag]),
                                         np.array([b.real, b.imag]), C.byref(e), out,
                                         C.byref(cnt)))
        return complex(out[0], out[1]), complex(out[2], out[3]), cnt

    def ctx_op(self, precision: str, op: str, a, b, c=None):
        """ArithmeticContext::add/sub/mul/fma elementwise (precision.cpp:77-111)."""
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        c = np.ascontiguousarray(c if c is not None else np.zeros_like(a), dtype=np.float64)
        out = np.empty_like(a)
        self._f("ctx_op")(PRECISIONS[precision], ("add", "sub", "mul", "fma").index(op), a, b, c,
                          out, a.size)
        return out

    def dft(self, x):
        x = np.ascontiguousarray(x, dtype=np.complex128)
        n = x.shape[-1]
        src = x.view(np.float64).ravel()
        out = np.empty_like(src)
        if self.prefix == "orc":
            self.lib.orc_dft.argtypes = [C.c_size_t, _DP, _DP, C.c_size_t, C.c_int]
            self.lib.orc_dft(n, src, out, x.size // n, 0)
        else:
            self.lib.ref_dft.argtypes = [C.c_size_t, _DP, _DP, C.c_size_t]
            self.lib.ref_dft(n, src, out, x.size // n)
        return out.view(np.complex128).reshape(x.shape)

    def rel_l2(self, x, y) -> float:
        x = np.ascontiguousarray(x, dtype=np.complex128)
        y = np.ascontiguousarray(y, dtype=np.complex128)
        return self._f("rel_l2")(x.view(np.float64).ravel(), y.view(np.float64).ravel(),
                                 x.size)

    def cumulative_bound(self, t_max: float, eps: float, m: int) -> float:
        return self._f("cumulative_bound")(t_max, eps, m)

    def uniform(self, seed: int, count: int):
        out = np.empty(count, dtype=np.float64)
        self._f("splitmix_uniform")(seed, out, count)
        return out

    def random_buffer(self, n: int, seed: int, batch: Optional[int] = None):
        """Reference protocol: one SplitMix64 stream, re then im per sample
        (analysis.cpp:120-125; tests' random_buffer test_fft.cpp:16-24)."""
        cnt = 2 * n * (batch or 1)
        v = self.uniform(seed, cnt).view(np.complex128)
        return v.reshape(batch, n) if batch else v

    def measure_error(self, n, strategy, precision, metric, trials, seed):
        rep = ErrorReport()
        self._check(self._f("measure_error")(n, STRATEGIES[strategy],
                                             PRECISIONS[precision],
                                             0 if metric == "roundtrip" else 1, trials,
                                             seed, C.byref(rep)))
        return {k: getattr(rep, k) for k, _ in ErrorReport._fields_ if k != "pad_"}


_cache = {}


def load_oracle() -> CpuFft:
    if "orc" not in _cache:
        if not os.path.exists(ORACLE_SO):
            build()
        _cache["orc"] = CpuFft(ORACLE_SO, "orc")
    return _cache["orc"]


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def load_ref() -> CpuFft:
    if "ref" not in _cache:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference)")
        _cache["ref"] = CpuFft(REF_SO, "ref")
    return _cache["ref"]
