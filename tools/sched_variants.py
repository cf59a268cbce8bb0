"""Build variant libraries of libdsfft.so whose single-kernel schedule for one
N is overridden (two-word values: fp32 and fp16 transform pairs), for same-box
A/B runs:

  python tools/sched_variants.py 12 5,4,4,4,4 ...   # LOG_E,W,S0[,S1[,S2[,S3]]]
  DSFFT_LIBRARY=paper_2604_00567_b200/build/variants/m12_1.so python bench.py --n 4096

Each variant recompiles only inst_small.cu for that N and relinks with the
package's other objects.  Prints one `label<TAB>path` line per variant."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_00567_b200 import build as B  # noqa: E402


def main():
    m, scheds = int(sys.argv[1]), sys.argv[2:]
    B.build()
    out_dir = os.path.join(B.OBJ, "variants")
    os.makedirs(out_dir, exist_ok=True)
    objs = [o for o, _, _ in B.jobs() if not o.endswith(f"inst_m{m}.o")]
    src = os.path.join(B.CSRC, "inst_small.cu")
    for i, sched in enumerate(scheds):
        obj = os.path.join(out_dir, f"inst_m{m}_{i}.o")
        lib = os.path.join(out_dir, f"m{m}_{i}.so")
        v = [int(x) for x in sched.split(",")]
        v += [0] * (6 - len(v))
        defs = [f"-DDSFFT_OV_{k}={x}" for k, x in zip(("E", "W", "S0", "S1", "S2", "S3"), v)]
        B._run([B.NVCC] + B.NVFLAGS + [f"-DDSFFT_M={m}"] + defs + ["-c", src, "-o", obj])
        subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-o", lib] + objs + [obj, "-lpthread"],
                       check=True)
        print(f"{sched}\t{os.path.relpath(lib, B.ROOT)}")


if __name__ == "__main__":
    main()
