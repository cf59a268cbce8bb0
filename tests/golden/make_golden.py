"""Generate tests/golden/golden.npz from the REFERENCE itself.

The reference (fmafft core, compiled unmodified from /root/reference by
oracle/Makefile into oracle/_ref/libfmafft_ref.so) is run here, in the dev
container, and its outputs are frozen as small fixtures so that parity stays
pinned on machines without /root/reference (the GPU box):

  * plan tables (rounded TwiddleEntry records) for every strategy/precision at
    n in {2, 8, 64, 1024} and the dual/LF tables at 4096;
  * forward and inverse outputs (working-precision bits) for seeded
    reference-protocol inputs at n in {2, 16, 64, 256, 1024, 4096};
  * measure_error reports (BASELINE.md's table: seed 42, 10 trials);
  * Table I / II statistics at n=1024.

  python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402

STRATS = ("standard", "lf", "cosine", "dual")
WDT = {"fp16": np.float16, "fp32": np.float32}


def main():
    ref = oracle.load_ref()
    out = {}
    for n in (2, 8, 64, 1024):
        for s in STRATS:
            for p in ("fp16", "fp32", "fp64"):
                out[f"table/{n}/{s}/{p}"] = ref.plan_table(n, s, p)
    for s in ("dual", "lf"):
        out[f"table/4096/{s}/fp16"] = ref.plan_table(4096, s, "fp16")
    for n in (2, 16, 64, 256, 1024, 4096):
        batch = 3 if n >= 1024 else 5
        seed = 500 + n
        x = ref.random_buffer(n, seed, batch=batch)
        for p in ("fp16", "fp32"):
            xr = ref.round_to(x.view(np.float64), p).view(np.complex128).reshape(batch, n)
            for s in STRATS:
                y = ref.forward(xr, s, p)
                out[f"fwd/{n}/{s}/{p}"] = y.view(np.float64).astype(WDT[p])
                yi = ref.inverse(xr, s, p)
                out[f"inv/{n}/{s}/{p}"] = yi.view(np.float64).astype(WDT[p])
            out[f"seed/{n}/{p}"] = np.array([seed, batch])
    rows = []
    for n in (64, 256, 1024, 4096):
        for s in STRATS:
            for p in ("fp16", "fp32"):
                r = ref.measure_error(n, s, p, "forward", 10, 42)
                rows.append([n, ("standard", "lf", "cosine", "dual").index(s), 0 if p == "fp16" else 1,
                             r["rel_l2_median"], r["rel_l2_max"], r["nonfinite_trials"]])
    out["measure_error/forward/seed42/trials10"] = np.array(rows, dtype=np.float64)
    rt = []
    for s in ("lf", "dual"):
        r = ref.measure_error(1024, s, "fp32", "roundtrip", 100, 42)
        rt.append([r["rel_l2_median"], r["rel_l2_max"], r["nonfinite_trials"]])
    out["measure_error/roundtrip/1024/fp32/lf_dual"] = np.array(rt)
    stats = []
    for s in ("lf", "cosine", "dual"):
        st = ref.table_stats(1024, s)
        stats.append([st["t_max"], st["argmax_k"], st["singular_count"], st["cos_path_count"],
                      st["sin_path_count"]])
    out["table_stats/1024/lf_cosine_dual"] = np.array(stats, dtype=np.float64)
    # write_table_csv (serialize.cpp:48-57), when the reference's serializer
    # was built (oracle/Makefile links it if nlohmann/json.hpp is available)
    import ctypes as C
    lib = ref.lib
    if hasattr(lib, "ref_table_csv"):
        lib.ref_table_csv.restype = C.c_size_t
        lib.ref_table_csv.argtypes = [C.c_size_t, C.c_int, C.c_int, C.c_double, C.c_char_p,
                                      C.c_size_t]
        for n, s, p in ((64, 3, 2), (64, 1, 2), (1024, 3, 0), (256, 2, 1), (8, 0, 2)):
            need = lib.ref_table_csv(n, s, p, 1e-7, None, 0)
            buf = C.create_string_buffer(need)
            lib.ref_table_csv(n, s, p, 1e-7, buf, need)
            out[f"csv/{n}/{STRATS[s]}/{('fp16', 'fp32', 'fp64')[p]}"] = \
                np.frombuffer(buf.value, dtype=np.uint8)
    # write_bounds_csv of reproduce_ratio_table / reproduce_cumulative_table
    # (the CLI `stats` and `bounds` commands)
    if hasattr(lib, "ref_bounds_csv"):
        lib.ref_bounds_csv.restype = C.c_size_t
        lib.ref_bounds_csv.argtypes = [C.c_size_t, C.c_int, C.c_int, C.c_char_p, C.c_size_t]
        for n, kind, p in ((1024, 0, 0), (64, 0, 0), (1 << 20, 0, 0), (2, 0, 0),
                           (1024, 1, 0), (1024, 1, 1), (4096, 1, 2), (8, 1, 0)):
            need = lib.ref_bounds_csv(n, kind, p, None, 0)
            buf = C.create_string_buffer(need)
            lib.ref_bounds_csv(n, kind, p, buf, need)
            out[f"bounds/{n}/{('stats', 'bounds')[kind]}/{('fp16', 'fp32', 'fp64')[p]}"] = \
                np.frombuffer(buf.value, dtype=np.uint8)
    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path), "bytes,", len(out), "arrays")


if __name__ == "__main__":
    main()
