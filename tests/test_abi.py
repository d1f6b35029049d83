"""C-ABI surface (CPU): the in-tree libsgwg.so loads without a GPU, exports
every function include/sgwg.h declares, and the Python mirror binds them all.
No compute calls here (no GPU); calls that need one fail loudly."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sgwg.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sgwg_[a-z0-9_]+)\s*\(", src)) - {"sgwg_stop_cb", "sgwg_ic_fn"})


@pytest.fixture(scope="module")
def lib():
    from paper_2007_10196_b200 import build, sgwg
    if not os.path.exists(sgwg.LIB_PATH):
        build.build()
    return sgwg.load()


def test_library_exports_every_declared_symbol(lib):
    from paper_2007_10196_b200 import sgwg
    out = subprocess.run(["nm", "-D", "--defined-only", sgwg.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (sgwg_[a-z0-9_]+)", out))
    decl = declared()
    assert len(decl) >= 30
    missing = [s for s in decl if s not in exported]
    assert not missing, missing


def test_python_mirror_binds_every_symbol(lib):
    from paper_2007_10196_b200 import sgwg
    assert sorted(sgwg.SIGNATURES) == declared()
    for name in declared():
        assert getattr(lib, name) is not None


def test_no_gpu_fails_loudly(lib):
    """Without a usable GPU the product raises; there is no CPU fallback."""
    import torch
    from paper_2007_10196_b200 import sgwg
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(sgwg.SgwgError):
        sgwg.Context(0)


def test_pure_host_entry_points(lib):
    from paper_2007_10196_b200 import sgwg
    lv = sgwg.enumerate_combination_levels(2, 3)
    assert [tuple(r) for r in lv] == [(0, 2), (0, 3), (1, 1), (1, 2), (2, 0), (2, 1), (3, 0)]
    with pytest.raises(ValueError):
        sgwg.enumerate_combination_levels(5, 3)
    with pytest.raises(ValueError):
        sgwg.enumerate_combination_levels(3, 1)
    assert lib.sgwg_version() == 1
