"""CPU-side checks of the C ABI: the library builds for sm_100a, loads, and
exports every entry point include/relcp.h declares; without a GPU the
context refuses to start (no CPU fallback)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "relcp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(relcp_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2506_14097_b200 import build, relcp
    path = build.build()
    lib = ctypes.CDLL(path)
    names = _declared()
    assert len(names) >= 14
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(relcp.EXPORTS)


def test_sm100a_cubin_in_library():
    import subprocess
    from paper_2506_14097_b200 import build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.build()], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_default_params_and_no_gpu_refusal():
    import torch
    from paper_2506_14097_b200 import relcp
    L = relcp.load()
    p = relcp.default_params()
    assert p.max_recursions == 50 and p.eps_ncp == 1e-5 and p.cutoff == 0.1 and p.lcp_tol == 1e-8
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    h = ctypes.c_void_p()
    assert L.relcp_create(ctypes.byref(h), ctypes.byref(p), None) == relcp.E_CUDA
    with pytest.raises(RuntimeError):
        relcp.Context()
    bad = relcp.default_params(dt=-1.0)
    assert L.relcp_create(ctypes.byref(h), ctypes.byref(bad), None) == relcp.E_ARG


def test_binding_refuses_bad_buffers():
    """The binding validates every tensor it hands to the C ABI: host, wrong
    dtype, strided or short buffers raise ValueError before any kernel can
    dereference them; optional arguments may be None."""
    import torch
    from paper_2506_14097_b200 import relcp as R
    f = torch.float64
    assert R._dptr(None, f, 3, "vel", optional=True) is None
    with pytest.raises(ValueError, match="required"):
        R._dptr(None, f, 3, "pos")
    with pytest.raises(ValueError, match="CUDA"):
        R._dptr(torch.zeros(8, dtype=f), f, 3, "pos")  # host tensor
    with pytest.raises(ValueError):
        R._dptr(torch.zeros(8, dtype=torch.float32), f, 3, "pos")
    with pytest.raises(ValueError):
        R._dptr(torch.zeros(4, 4, dtype=f).T, f, 3, "pos")
    with pytest.raises(ValueError):
        R._dptr(torch.zeros(2, dtype=f), f, 3, "pos")
    with pytest.raises(ValueError):
        R._dptr([0.0, 1.0, 2.0], f, 3, "pos")
