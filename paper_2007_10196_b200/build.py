"""In-tree build of the CUDA extension ``libsgwg.so`` (sm_100a only).

The kernels are compiled with nvcc directly (no JIT cache) so the shared
object travels with the repository snapshot to the GPU box:

* ``k_exact.cu``  -- reference-order arithmetic, ``--fmad=false`` (bitwise parity)
* ``k_fast.cu``   -- FMA-contracted, divide-reduced arithmetic
* ``k_field.cu``  -- Vlasov-Poisson moment + spectral Poisson
* ``k_diag.cu``   -- diagnostics of the combined field (mass, min/max, error norms)
* ``sgwg_api.cu`` -- host runtime behind the C ABI (include/sgwg.h), links NCCL
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
OBJ = os.path.join(CSRC, "obj")
LIB = os.path.join(HERE, "libsgwg.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
          "-Xcompiler", "-ffp-contract=off", f"-I{os.path.join(ROOT, 'include')}"] + ARCH

UNITS = {
    "k_exact.cu": ["--fmad=false", "-Xptxas", "-v"],
    "k_fast.cu": ["--fmad=true", "-Xptxas", "-v"],
    "k_field.cu": ["--fmad=true"],
    "k_diag.cu": ["--fmad=true"],
    "sgwg_api.cu": ["--fmad=false"],
}
HEADERS = ["kernels.cuh", "sgwg_internal.h", "dt_device.cuh", "field_device.cuh", "pdl.cuh",
           "plane4d.cuh"]


def _stale(obj, deps):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def _digest(deps, cmd):
    """Content hash of a unit's sources and command line (file times are not trusted: an
    object that looked fresh once hid a source change from the GPU runs)."""
    import hashlib
    h = hashlib.sha256(" ".join(cmd).encode())
    for d in deps:
        with open(d, "rb") as f:
            h.update(f.read())
    return h.hexdigest()


def _compile(src, flags, verbose):
    obj = os.path.join(OBJ, src.replace(".cu", ".o"))
    deps = [os.path.join(CSRC, src)] + [os.path.join(CSRC, h) for h in HEADERS] + [
        os.path.join(ROOT, "include", "sgwg.h"), __file__]
    cmd = [NVCC, "-c", os.path.join(CSRC, src), "-o", obj] + COMMON + flags
    want = _digest(deps, cmd)
    stamp = obj + ".sha256"
    if os.path.exists(obj) and os.path.exists(stamp) and open(stamp).read().strip() == want:
        return obj, "", False
    if os.path.exists(stamp):
        os.remove(stamp)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        if os.path.exists(obj):
            os.remove(obj)
        raise RuntimeError(f"nvcc failed for {src}:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    with open(stamp, "w") as f:
        f.write(want)
    return obj, (r.stdout + r.stderr) if verbose else "", True


def build(verbose: bool = False) -> str:
    """Compile (incrementally) and link ``libsgwg.so``; return its path."""
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(UNITS)) as ex:
        futs = [ex.submit(_compile, s, f, verbose) for s, f in UNITS.items()]
        results = [f.result() for f in futs]
    objs = [o for o, _, _ in results]
    for _, log, _ in results:
        if log:
            sys.stdout.write(log)
    if any(c for _, _, c in results) or _stale(LIB, objs):
        cmd = [NVCC, "-shared", "-o", LIB] + objs + ARCH + ["-lnccl", "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
