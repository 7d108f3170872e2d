"""Build an A/B variant of the library with extra nvcc defines:

  python tools/variant.py NAME [--src=path/to/stmg_kernels.cu] -DFOO=1 ...
-> paper_1411_0519_b200/_variant_NAME.so (load it with STMG_LIB=<path>).
--src compiles another kernels source (e.g. `git show HEAD:...` saved to /tmp)
with the in-tree headers, for before/after comparisons.
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1411_0519_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
src = os.path.join(B.CSRC, "stmg_kernels.cu")
for d in list(defs):
    if d.startswith("--src="):
        src = d[6:]
        defs.remove(d)
B.build()
obj = os.path.join(B.OBJ, f"stmg_kernels_{name}.o")
subprocess.run([B.nvcc()] + B.NVFLAGS + ["-I" + B.CSRC] + defs + ["-c", src, "-o", obj],
               check=True)
others = [os.path.join(B.OBJ, os.path.splitext(s)[0] + ".o") for s in B.SOURCES if s != "stmg_kernels.cu"]
out = os.path.join(B.PKG, f"_variant_{name}.so")
subprocess.run([B.nvcc()] + B.ARCH + ["-shared", "-o", out, obj] + others + ["-cudart", "static"],
               check=True)
print(out)
