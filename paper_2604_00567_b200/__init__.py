"""B200-native batched dual-select FFT (arXiv 2604.00567) -- Python host side.

A thin mirror of the reference's plan/execute API (``fmafft::make_plan``,
``forward``, ``inverse``, ``Strategy``, ``Precision``; /root/reference/proj/core/
include/fmafft/{fft,twiddle,precision}.hpp) over the C ABI of ``libdsfft.so``
(include/dsfft.h).  All compute runs in the sm_100a kernels; if the library is
missing or no B200 is present, calls raise -- there is no CPU fallback.

Device API (torch tensors are used as plain device buffers):
    plan = make_plan(1024, "dual", "fp16")
    y = forward(plan, x)      # x: cuda tensor [batch, n] complex32/complex64
                              #    or [batch, n, 2] float16/float32
Reference calling convention (double-carrier SampleBuffers, ingest rounding):
    y = forward_f64(plan, x)  # x: numpy complex128 [batch, n] or [n]
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

__all__ = ["Strategy", "Precision", "FftPlan", "make_plan", "forward", "inverse",
           "execute", "forward_f64", "inverse_f64", "execute_host", "execute_multi",
           "round_to", "widen", "build_table", "table_csv", "bounds_csv", "error_device",
           "measure_error", "dft_oracle", "dft_device", "make_plan_from_table", "fill_uniform", "synthetic_batch", "context_op", "butterflies",
           "last_launch_count", "parse_strategy", "parse_precision", "library_path",
           "DsfftError"]

_PKG = os.path.dirname(os.path.abspath(__file__))
# DSFFT_LIBRARY: load another build of the library (A/B timing of two builds)
_LIB_PATH = os.environ.get("DSFFT_LIBRARY") or os.path.join(_PKG, "libdsfft.so")

# fmafft::Strategy / Precision declaration order (twiddle.hpp:14, precision.hpp:12)
STRATEGIES = {"standard": 0, "lf": 1, "cosine": 2, "dual": 3}
PRECISIONS = {"fp16": 0, "fp32": 1, "fp64": 2}
_STRATEGY_ALIASES = {"standard": "standard", "lf": "lf", "linzer-feig": "lf",
                     "linzer_feig": "lf", "cosine": "cosine", "dual": "dual",
                     "dual-select": "dual", "dual_select": "dual"}


class Strategy:
    standard = "standard"
    linzer_feig = "lf"
    cosine = "cosine"
    dual_select = "dual"


class Precision:
    fp16 = "fp16"
    fp32 = "fp32"
    fp64 = "fp64"


def parse_strategy(name: str) -> str:
    """twiddle.cpp:45-53 (throws std::invalid_argument -> ValueError)."""
    try:
        return _STRATEGY_ALIASES[name]
    except KeyError:
        raise ValueError(f"unknown strategy: {name}") from None


def parse_precision(name: str) -> str:
    """precision.cpp:54-59."""
    if name not in PRECISIONS:
        raise ValueError(f"unknown precision: {name}")
    return name


class DsfftError(RuntimeError):
    pass


class _Entry(C.Structure):
    _fields_ = [("multiplier", C.c_double), ("ratio", C.c_double), ("path", C.c_int32),
                ("clamped", C.c_int32), ("omega_r", C.c_double), ("omega_i", C.c_double)]


ENTRY_DTYPE = np.dtype([("multiplier", "<f8"), ("ratio", "<f8"), ("path", "<i4"),
                        ("clamped", "<i4"), ("omega_r", "<f8"), ("omega_i", "<f8")])

_lib = None


def library_path() -> str:
    return _LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} is not built; run `python -m paper_2604_00567_b200.build`"
                          " (there is no CPU fallback)")
    lib = C.CDLL(_LIB_PATH)
    vp, sz, i = C.c_void_p, C.c_size_t, C.c_int
    lib.dsfft_last_error.restype = C.c_char_p
    lib.dsfft_plan_create.argtypes = [sz, i, i, C.c_double, i, C.POINTER(vp)]
    lib.dsfft_plan_destroy.argtypes = [vp]
    lib.dsfft_plan_info.argtypes = [vp, C.POINTER(sz), C.POINTER(C.c_uint), C.POINTER(i),
                                    C.POINTER(i)]
    lib.dsfft_plan_table.argtypes = [vp, vp, sz]
    lib.dsfft_build_table.argtypes = [sz, i, i, C.c_double, vp, sz]
    lib.dsfft_execute.argtypes = [vp, i, vp, vp, sz, vp]
    lib.dsfft_execute_host.argtypes = [vp, i, vp, vp, sz, vp]
    lib.dsfft_execute_f64.argtypes = [vp, i, vp, vp, sz]
    lib.dsfft_round_to.argtypes = [vp, vp, sz, i]
    lib.dsfft_widen.argtypes = [vp, vp, sz, i]
    lib.dsfft_sample_bytes.restype = sz
    lib.dsfft_sample_bytes.argtypes = [i]
    lib.dsfft_last_launch_count.restype = C.c_uint64
    _lib = lib
    return lib


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = _load().dsfft_last_error().decode()
    if rc == 1:
        raise ValueError(msg)            # std::invalid_argument in the reference
    if rc == 2:
        raise NotImplementedError(msg)
    raise DsfftError(msg)


@dataclass(eq=False)
class FftPlan:
    """Mirror of fmafft::FftPlan (fft.hpp:17-23) owning a device plan (the
    handle is destroyed with the object; plans are shareable, not copyable)."""
    n: int
    m: int
    strategy: str
    precision: str
    device: int
    _handle: C.c_void_p

    @property
    def table(self) -> np.ndarray:
        """FftPlan::table.entries: the rounded n/2 records (TwiddleEntry fields)."""
        out = np.zeros(max(self.n // 2, 1), dtype=ENTRY_DTYPE)
        _check(_load().dsfft_plan_table(self._handle, out.ctypes.data, out.size))
        return out[: self.n // 2]

    def __reduce_ex__(self, protocol):
        raise TypeError("FftPlan owns a device plan and cannot be copied or pickled; "
                        "share the object or call make_plan again")

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h and _lib is not None:
            _lib.dsfft_plan_destroy(h)
            self._handle = None


def make_plan(n: int, strategy: str = "dual", precision: str = "fp32",
              clamp_eps: float = 1e-7, device: int = 0) -> FftPlan:
    """fmafft::make_plan (fft.cpp:56-72): n a power of two in [2, 2^24]."""
    strategy = parse_strategy(strategy)
    precision = parse_precision(precision)
    h = C.c_void_p()
    _check(_load().dsfft_plan_create(int(n), STRATEGIES[strategy], PRECISIONS[precision],
                                     float(clamp_eps), int(device), C.byref(h)))
    m = int(n).bit_length() - 1
    return FftPlan(int(n), m, strategy, precision, device, h)


def make_plan_from_table(n: int, strategy: str, precision: str, table: np.ndarray,
                         device: int = 0) -> FftPlan:
    """A plan over a caller-supplied rounded table (FftPlan::table.entries,
    possibly edited -- the reference's FftPlan is a plain struct): the records
    are packed and uploaded as given (dsfft_plan_create_with_table)."""
    strategy = parse_strategy(strategy)
    precision = parse_precision(precision)
    t = np.ascontiguousarray(table, dtype=ENTRY_DTYPE)
    lib = _load()
    lib.dsfft_plan_create_with_table.argtypes = [C.c_size_t, C.c_int, C.c_int, C.c_void_p,
                                                 C.c_size_t, C.c_int, C.POINTER(C.c_void_p)]
    h = C.c_void_p()
    _check(lib.dsfft_plan_create_with_table(int(n), STRATEGIES[strategy], PRECISIONS[precision],
                                            t.ctypes.data, t.size, int(device), C.byref(h)))
    return FftPlan(int(n), int(n).bit_length() - 1, strategy, precision, device, h)


def bounds_csv(n: int, kind: str = "stats", precision: str = "fp16") -> str:
    """write_bounds_csv (serialize.cpp:79-91) of reproduce_ratio_table(n)
    (kind "stats": the CLI `stats` command) or reproduce_cumulative_table(n,
    precision) (kind "bounds")."""
    kinds = {"stats": 0, "ratio": 0, "bounds": 1, "cumulative": 1}
    if kind not in kinds:
        raise ValueError(f"unknown statistics kind: {kind}")
    lib = _load()
    lib.dsfft_bounds_csv.restype = C.c_size_t
    lib.dsfft_bounds_csv.argtypes = [C.c_size_t, C.c_int, C.c_int, C.c_char_p, C.c_size_t]
    args = (int(n), kinds[kind], PRECISIONS[parse_precision(precision)])
    need = lib.dsfft_bounds_csv(*args, None, 0)
    if need == 0:
        raise ValueError(lib.dsfft_last_error().decode())
    buf = C.create_string_buffer(need)
    lib.dsfft_bounds_csv(*args, buf, need)
    return buf.value.decode()


def table_csv(n: int, strategy: str, precision: str = "fp64", clamp_eps: float = 1e-7) -> str:
    """write_table_csv (serialize.cpp:48-57) of build_table (fp64, the CLI
    `twiddles` dump) or of the plan's rounded table (fp16 / fp32)."""
    lib = _load()
    lib.dsfft_table_csv.restype = C.c_size_t
    lib.dsfft_table_csv.argtypes = [C.c_size_t, C.c_int, C.c_int, C.c_double, C.c_char_p,
                                    C.c_size_t]
    args = (int(n), STRATEGIES[parse_strategy(strategy)], PRECISIONS[parse_precision(precision)],
            float(clamp_eps))
    need = lib.dsfft_table_csv(*args, None, 0)
    if need == 0:
        raise ValueError(lib.dsfft_last_error().decode())
    buf = C.create_string_buffer(need)
    lib.dsfft_table_csv(*args, buf, need)
    return buf.value.decode()


def build_table(n: int, strategy: str, precision: str = "fp64",
                clamp_eps: float = 1e-7) -> np.ndarray:
    """Host table builder: make_plan's rounded table (fp64: build_table)."""
    out = np.zeros(max(int(n) // 2, 1), dtype=ENTRY_DTYPE)
    _check(_load().dsfft_build_table(int(n), STRATEGIES[parse_strategy(strategy)],
                                     PRECISIONS[parse_precision(precision)], float(clamp_eps),
                                     out.ctypes.data, out.size))
    return out[: int(n) // 2]


def sample_bytes(precision: str) -> int:
    return 4 if precision == "fp16" else 8 if precision == "fp32" else 16


def _torch_view(x, plan: FftPlan):
    import torch
    want_c = {"fp16": torch.complex32, "fp32": torch.complex64,
              "fp64": torch.complex128}[plan.precision]
    want_r = {"fp16": torch.float16, "fp32": torch.float32,
              "fp64": torch.float64}[plan.precision]
    if x.dtype == want_c:
        n = x.shape[-1]
    elif x.dtype == want_r and x.shape[-1] == 2:
        n = x.shape[-2]
    else:
        raise ValueError(f"{plan.precision} plan needs {want_c} or {want_r}[..., 2] data, "
                         f"got {x.dtype}")
    if n != plan.n:
        raise ValueError(f"buffer length {n} does not match plan size {plan.n}")
    if not x.is_cuda:
        raise ValueError("device API needs a CUDA tensor (use forward_f64 for host data)")
    if not x.is_contiguous():
        raise ValueError("tensor must be contiguous")
    if x.device.index != plan.device:
        raise ValueError(f"tensor is on cuda:{x.device.index}, plan on cuda:{plan.device}")
    batch = x.numel() // (plan.n * (2 if x.dtype == want_r else 1))
    return batch


def _check_out(x, out) -> None:
    """`out` must be a buffer the kernels can write exactly like `x`."""
    if out.dtype != x.dtype or out.numel() != x.numel():
        raise ValueError(f"out ({out.dtype}, {out.numel()} elements) does not match the input "
                         f"({x.dtype}, {x.numel()} elements)")
    if not out.is_cuda or out.device.index != x.device.index:
        raise ValueError("out must be on the same CUDA device as the input")
    if not out.is_contiguous():
        raise ValueError("out must be contiguous")


def execute(plan: FftPlan, direction: int, x, out=None, stream=None):
    """Batched transform of a CUDA tensor (direction 0 forward, 1 inverse)."""
    import torch
    batch = _torch_view(x, plan)
    if out is None:
        out = torch.empty_like(x)
    else:
        _check_out(x, out)
    if stream is None:
        stream = torch.cuda.current_stream(x.device).cuda_stream
    _check(_load().dsfft_execute(plan._handle, direction, x.data_ptr(), out.data_ptr(), batch,
                                 stream))
    return out


def forward(plan: FftPlan, x, out=None, stream=None):
    """fmafft::forward (fft.hpp:33) on a batch of device transforms."""
    return execute(plan, 0, x, out, stream)


def inverse(plan: FftPlan, x, out=None, stream=None):
    """fmafft::inverse (fft.hpp:38) on a batch of device transforms."""
    return execute(plan, 1, x, out, stream)


def _check_host(plan: FftPlan, h_in: np.ndarray, h_out: np.ndarray, batch: int) -> None:
    need = int(batch) * plan.n * sample_bytes(plan.precision)
    if h_in.nbytes < need or h_out.nbytes < need:
        raise ValueError(f"host buffers hold {h_in.nbytes} / {h_out.nbytes} bytes, "
                         f"batch {batch} needs {need}")
    if not (h_in.flags.c_contiguous and h_out.flags.c_contiguous):
        raise ValueError("host buffers must be C-contiguous")


def execute_host(plan: FftPlan, direction: int, h_in: np.ndarray, h_out: np.ndarray,
                 batch: int, stream: int = 0) -> None:
    """Host buffers in the working precision (pinned for full overlap)."""
    _check_host(plan, h_in, h_out, batch)
    _check(_load().dsfft_execute_host(plan._handle, direction, h_in.ctypes.data,
                                      h_out.ctypes.data, batch, stream))


def _f64_call(plan: FftPlan, direction: int, x) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.complex128)
    if x.shape[-1] != plan.n:
        raise ValueError(f"buffer length {x.shape[-1]} does not match plan size {plan.n}")
    out = np.empty_like(x)
    batch = x.size // plan.n
    _check(_load().dsfft_execute_f64(plan._handle, direction, x.ctypes.data, out.ctypes.data,
                                     batch))
    return out


def forward_f64(plan: FftPlan, x) -> np.ndarray:
    """The reference's exact convention: complex128 in, ingest round_to, device
    transform, result widened to complex128 (SampleBuffer, fft.hpp:12)."""
    return _f64_call(plan, 0, x)


def inverse_f64(plan: FftPlan, x) -> np.ndarray:
    return _f64_call(plan, 1, x)


def round_to(x, precision: str) -> np.ndarray:
    """round_to (precision.cpp:61-75) through the product's own converter."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    p = PRECISIONS[parse_precision(precision)]
    dt = {0: np.uint16, 1: np.float32, 2: np.float64}[p]
    raw = np.empty(x.shape, dtype=dt)
    _check(_load().dsfft_round_to(x.ctypes.data, raw.ctypes.data, x.size, p))
    return raw


def widen(raw: np.ndarray, precision: str) -> np.ndarray:
    p = PRECISIONS[parse_precision(precision)]
    raw = np.ascontiguousarray(raw)
    out = np.empty(raw.shape, dtype=np.float64)
    _check(_load().dsfft_widen(raw.ctypes.data, out.ctypes.data, raw.size, p))
    return out


def last_launch_count() -> int:
    return int(_load().dsfft_last_launch_count())


def execute_multi(plans, direction: int, h_in: np.ndarray, h_out: np.ndarray,
                  batch: int) -> None:
    """Batch partitioner over devices (dsfft_execute_multi): plans[i] runs the
    contiguous shard i of the host batch on its own device."""
    if not plans:
        raise ValueError("no plans")
    _check_host(plans[0], h_in, h_out, batch)
    lib = _load()
    lib.dsfft_execute_multi.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                        C.c_size_t]
    arr = (C.c_void_p * len(plans))(*[p._handle for p in plans])
    _check(lib.dsfft_execute_multi(C.cast(arr, C.c_void_p), len(plans), direction,
                                   h_in.ctypes.data, h_out.ctypes.data, batch))


class _ErrorReport(C.Structure):
    _fields_ = [("n", C.c_uint64), ("strategy", C.c_int32), ("precision", C.c_int32),
                ("metric", C.c_int32), ("pad_", C.c_int32), ("trials", C.c_uint64),
                ("seed", C.c_uint64), ("rel_l2_median", C.c_double),
                ("rel_l2_max", C.c_double), ("nonfinite_trials", C.c_uint64)]


def _report(rep: "_ErrorReport") -> dict:
    return {k: getattr(rep, k) for k, _ in _ErrorReport._fields_ if k != "pad_"}


_METRICS = {"roundtrip": 0, "forward": 1, "forward_vs_oracle": 1}
_REFERENCES = {"auto": 0, "dft": 1, "fft64": 2}


def error_device(plan: FftPlan, x, metric: str = "forward", stream=None,
                 per_transform: bool = False, reference: str = "auto"):
    """Device error harness over a device batch (dsfft_error_device_ex): the
    reference's ErrorReport (analysis.hpp:58-68) for every transform in `x`.
    reference: "dft" (dft_oracle, bit-identical reports), "fft64" (the fp64
    FFT) or "auto" (DFT for n <= 4096)."""
    import torch
    batch = _torch_view(x, plan)
    if reference not in _REFERENCES:
        raise ValueError(f"unknown error reference: {reference}")
    lib = _load()
    lib.dsfft_error_device_ex.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_size_t,
                                          C.c_void_p, C.POINTER(_ErrorReport), C.c_void_p]
    rep = _ErrorReport()
    errs = np.empty(batch, dtype=np.float64) if per_transform else None
    if stream is None:
        stream = torch.cuda.current_stream(x.device).cuda_stream
    _check(lib.dsfft_error_device_ex(plan._handle, _METRICS[metric], _REFERENCES[reference],
                                     x.data_ptr(), batch, stream, C.byref(rep),
                                     errs.ctypes.data if errs is not None else None))
    return (_report(rep), errs) if per_transform else _report(rep)


def fill_uniform(out, n: int, first_transform: int, seed: int, precision: str,
                 stream=None):
    """dsfft_fill_uniform: fill the CUDA tensor `out` (working precision,
    [count, n, 2] or complex) with transforms [first, first + count) of the
    synthetic batch `seed` -- keyed by the global transform index, so a shard
    equals the same rows of the whole batch."""
    import torch
    p = PRECISIONS[parse_precision(precision)]
    want = {0: torch.float16, 1: torch.float32, 2: torch.float64}[p]
    if out.dtype not in (want, {0: torch.complex32, 1: torch.complex64,
                                2: torch.complex128}[p]):
        raise ValueError(f"{precision} batch needs {want} storage, got {out.dtype}")
    if not out.is_cuda or not out.is_contiguous():
        raise ValueError("fill_uniform needs a contiguous CUDA tensor")
    comps = out.numel() * (2 if out.is_complex() else 1)
    if comps % (2 * n):
        raise ValueError("tensor does not hold whole transforms of n samples")
    if stream is None:
        stream = torch.cuda.current_stream(out.device).cuda_stream
    lib = _load()
    lib.dsfft_fill_uniform.argtypes = [C.c_void_p, C.c_size_t, C.c_uint64, C.c_size_t,
                                       C.c_uint64, C.c_int, C.c_int, C.c_void_p]
    _check(lib.dsfft_fill_uniform(out.data_ptr(), int(n), int(first_transform),
                                  comps // (2 * n), int(seed), p, out.device.index, stream))
    return out


def synthetic_batch(n: int, first_transform: int, count: int, seed: int, precision: str,
                    device: int = 0, stream=None):
    """A new [count, n, 2] CUDA tensor from fill_uniform."""
    import torch
    dt = {"fp16": torch.float16, "fp32": torch.float32, "fp64": torch.float64}[
        parse_precision(precision)]
    out = torch.empty((count, n, 2), dtype=dt, device=torch.device("cuda", device))
    return fill_uniform(out, n, first_transform, seed, precision, stream)


_OPS = {"add": 0, "sub": 1, "mul": 2, "fma": 3}


def context_op(precision: str, op: str, a, b, c=None, device: int = 0) -> np.ndarray:
    """ArithmeticContext::add/sub/mul/fma (precision.cpp:77-111) elementwise on
    the device, rounded exactly as the reference rounds (dsfft_context_ops)."""
    if op not in _OPS:
        raise ValueError(f"unknown operation: {op}")
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    c = np.ascontiguousarray(c if c is not None else np.zeros_like(a), dtype=np.float64)
    if not (a.shape == b.shape == c.shape):
        raise ValueError("operand shapes differ")
    out = np.empty_like(a)
    lib = _load()
    lib.dsfft_context_ops.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_size_t, C.c_int]
    _check(lib.dsfft_context_ops(PRECISIONS[parse_precision(precision)], _OPS[op], a.ctypes.data,
                                 b.ctypes.data, c.ctypes.data, out.ctypes.data, a.size,
                                 int(device)))
    return out


def butterflies(strategy: str, precision: str, a, b, entries, device: int = 0):
    """The butterfly-variant API (butterfly.hpp:22-61) on the device: complex128
    arrays a, b and an ENTRY_DTYPE array of table entries -> (sum, diff)."""
    a = np.ascontiguousarray(a, dtype=np.complex128)
    b = np.ascontiguousarray(b, dtype=np.complex128)
    e = np.ascontiguousarray(entries, dtype=ENTRY_DTYPE)
    if not (a.shape == b.shape == e.shape):
        raise ValueError("operand shapes differ")
    out = np.empty(a.shape + (2,), dtype=np.complex128)
    lib = _load()
    lib.dsfft_butterflies.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_size_t, C.c_int]
    _check(lib.dsfft_butterflies(STRATEGIES[parse_strategy(strategy)],
                                 PRECISIONS[parse_precision(precision)], a.ctypes.data,
                                 b.ctypes.data, e.ctypes.data, out.ctypes.data, a.size,
                                 int(device)))
    return out[..., 0], out[..., 1]


def dft_oracle(x, device: int = 0) -> np.ndarray:
    """fmafft::dft_oracle (fft.hpp:44, fft.cpp:103-121) on the device,
    bit-identical: complex128 [..., n] in and out (any n)."""
    x = np.ascontiguousarray(x, dtype=np.complex128)
    n = x.shape[-1]
    out = np.empty_like(x)
    lib = _load()
    lib.dsfft_dft_oracle.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t, C.c_int]
    _check(lib.dsfft_dft_oracle(x.ctypes.data, out.ctypes.data, n, x.size // max(n, 1),
                                int(device)))
    return out


def dft_device(x, out=None, stream=None):
    """dft_oracle over a CUDA complex128 tensor [..., n] (stream-ordered)."""
    import torch
    if x.dtype != torch.complex128 or not x.is_cuda or not x.is_contiguous():
        raise ValueError("dft_device needs a contiguous CUDA complex128 tensor")
    if out is None:
        out = torch.empty_like(x)
    else:
        _check_out(x, out)
    if stream is None:
        stream = torch.cuda.current_stream(x.device).cuda_stream
    n = x.shape[-1]
    lib = _load()
    lib.dsfft_dft_device.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t, C.c_int,
                                     C.c_void_p]
    _check(lib.dsfft_dft_device(x.data_ptr(), out.data_ptr(), n, x.numel() // max(n, 1),
                                x.device.index, stream))
    return out


def measure_error(n: int, strategy: str, precision: str, metric: str = "forward",
                  trials: int = 100, seed: int = 42, device: int = 0) -> dict:
    """measure_error (analysis.cpp:101-154) with every transform on the device."""
    lib = _load()
    lib.dsfft_measure_error.argtypes = [C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_size_t,
                                        C.c_uint64, C.c_int, C.POINTER(_ErrorReport)]
    rep = _ErrorReport()
    _check(lib.dsfft_measure_error(int(n), STRATEGIES[parse_strategy(strategy)],
                                   PRECISIONS[parse_precision(precision)], _METRICS[metric],
                                   int(trials), int(seed), int(device), C.byref(rep)))
    return _report(rep)
