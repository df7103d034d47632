"""Build an A/B variant of libhfb200.so with extra nvcc defines (experiments only;
the product is built by paper_1811_07717_b200/build.py with no variants).

    python tools/build_variant.py OUT.so -DNAME=VALUE ...
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                "paper_1811_07717_b200"))
import build as B  # noqa: E402

out, defs = sys.argv[1], sys.argv[2:]
cmd = [B.nvcc_path(), *B.ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
       *defs, "-I", os.path.join(B.ROOT, "include"), *[os.path.join(B.CSRC, s) for s in B.SOURCES],
       "-o", out]
subprocess.run(cmd, check=True)
print(out)
