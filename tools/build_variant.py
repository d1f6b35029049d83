"""Experiment helper: link a variant of libsgwg.so whose fast kernels are
compiled with extra -D flags (load it with SGWG_LIB=<path>).

    python tools/build_variant.py out.so -DSGWG_PLANE_MINB=4 [...]
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2007_10196_b200 import build as B  # noqa: E402

out, defs = sys.argv[1], sys.argv[2:]
B.build()
variant = ["k_fast.cu", "k_field.cu"]  # the TUs that take experiment -D flags
objs = []
for u in B.UNITS:
    if u in variant:
        obj = os.path.join(B.OBJ, u.replace(".cu", "_variant.o"))
        cmd = [B.NVCC, "-c", os.path.join(B.CSRC, u), "-o", obj] + B.COMMON + B.UNITS[u] + defs
        subprocess.run(cmd, check=True, capture_output=True)
        objs.append(obj)
    else:
        objs.append(os.path.join(B.OBJ, u.replace(".cu", ".o")))
subprocess.run([B.NVCC, "-shared", "-o", out] + objs + B.ARCH + ["-lnccl", "-lcudart"], check=True)
print(out)
