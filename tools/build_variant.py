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
obj = os.path.join(B.OBJ, "k_fast_variant.o")
cmd = [B.NVCC, "-c", os.path.join(B.CSRC, "k_fast.cu"), "-o", obj] + B.COMMON + B.UNITS["k_fast.cu"] + defs
subprocess.run(cmd, check=True, capture_output=True)
objs = [os.path.join(B.OBJ, u.replace(".cu", ".o")) for u in B.UNITS if u != "k_fast.cu"] + [obj]
subprocess.run([B.NVCC, "-shared", "-o", out] + objs + B.ARCH + ["-lnccl", "-lcudart"], check=True)
print(out)
