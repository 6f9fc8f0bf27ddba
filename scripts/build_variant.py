"""Build a variant of libgpbbmm.so with extra nvcc defines for one source
(A/B diagnostics on the GPU box; the product build is _build.build()):

  [REPLACES=kv_sym.cu] python scripts/build_variant.py NAME SRC.cu [-DFOO=1 ...]
    -> scripts/variants/lib_NAME.so (other objects reused from _lib/)

Run with GPBBMM_LIB=scripts/variants/lib_NAME.so to load it instead."""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from paper_1903_08114_b200 import _build as B  # noqa: E402


def main():
    name, src, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
    B.build()
    out = os.path.join(HERE, "variants")
    os.makedirs(out, exist_ok=True)
    obj = os.path.join(out, f"{name}_{src.replace('.cu', '.o')}")
    cmd = [B.nvcc(), *B.ARCH, *B.FLAGS, *defs, "-c", os.path.join(B.CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    sys.stderr.write("\n".join(l for l in r.stderr.splitlines() if "registers" in l or "spill" in l or "error" in l))
    sys.stderr.write("\n")
    if r.returncode:
        sys.stderr.write(r.stdout + r.stderr)
        sys.exit(1)
    # a source outside the product list stands in for REPLACES (default: src)
    rep = os.environ.get("REPLACES", src)
    assert rep in B.SOURCES, f"{rep} is not a library source"
    objs = [obj if s == rep else os.path.join(B.LIBDIR, s.replace(".cu", ".o")) for s in B.SOURCES]
    lib = os.path.join(out, f"lib_{name}.so")
    r = subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", lib, *objs, "-lcudart", "-Xlinker", "--no-undefined"],
                       capture_output=True, text=True)
    if r.returncode:
        sys.stderr.write(r.stdout + r.stderr)
        sys.exit(1)
    print(lib)


if __name__ == "__main__":
    main()
