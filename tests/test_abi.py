"""C-ABI library checks that need no GPU: it loads and exports every symbol include/kpp.h
declares; the binding refuses to run without CUDA (no CPU fallback)."""
import ctypes
import os
import re

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "kpp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s+([a-z_0-9]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    from paper_2501_11673_b200 import build
    build.build()
    return ctypes.CDLL(build.LIB)


def test_header_declares_api():
    names = declared_symbols()
    for must in ("kpp_setup", "kpp_solve", "cdpp_setup", "cdpp_solve", "kpp_destroy",
                 "kpp_setup_dist", "cdpp_setup_dist", "kpp_get_unique_id", "kpp_get_schedule"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_status_strings(lib):
    lib.kpp_status_str.restype = ctypes.c_char_p
    assert lib.kpp_status_str(0) == b"ok"
    assert b"positive" in lib.kpp_status_str(5)
    lib.kpp_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.kpp_version()


def test_sm100a_code_in_library():
    """The library carries sm_100a SASS and the FP64 tensor-core instruction (DMMA)."""
    import shutil
    import subprocess
    from paper_2501_11673_b200 import build
    build.build()
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([cuobjdump, "-sass", build.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "DMMA" in out


def test_binding_refuses_cpu_tensors():
    import paper_2501_11673_b200 as kpp
    A = torch.zeros(8, 8, dtype=torch.float64)
    with pytest.raises(kpp.KppError):
        kpp.kpp_setup(A, 4)


def test_column_slabs_partition():
    import paper_2501_11673_b200 as kpp
    for n, P in [(131072, 8), (4096, 3), (10, 4)]:
        sl = kpp.column_slabs(n, P)
        assert sl[0][0] == 0 and sl[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(sl, sl[1:]))
