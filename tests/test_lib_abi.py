"""CPU-only checks of the C ABI library (no compute calls: there is no GPU
here).  libbrng.so builds for sm_100a, loads, and exports exactly the
symbols include/brng.h declares; host-side validation answers without a
launch; the product path has no oracle import and no CPU fallback."""
import ctypes as C
import importlib.util
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "brng.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^BRNG_API\s+(?:const\s+)?\w+\*?\s+(brng_\w+)\(", src, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_1412_4825_b200 import _build
    path = _build.build()
    return C.CDLL(path), path


def test_header_declares_the_north_star_calls():
    names = _declared()
    for must in ("brng_create", "brng_uniform_f32", "brng_gaussian_f32", "brng_exponential_f32",
                 "brng_gamma_f64", "brng_dirichlet_f32", "brng_gibbs_triangle"):
        assert must in names


def test_exports_every_declared_symbol(lib):
    L, path = lib
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True,
                         check=True).stdout
    exported = sorted(set(re.findall(r" T (brng_\w+)$", out, re.M)))
    assert exported == _declared()
    for name in _declared():
        getattr(L, name)


def test_binding_covers_header():
    import paper_1412_4825_b200 as B
    assert sorted(B.brng.EXPORTED) == _declared()
    for name in _declared():
        assert callable(getattr(B, name))


def test_built_for_sm100a(lib):
    _, path = lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", path],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_host_validation_without_launch():
    import paper_1412_4825_b200 as B
    raw = B.brng.raw_call
    assert B.brng_version() == 1
    assert B.brng_status_string(0) == "ok"
    assert "CUDA" in B.brng_status_string(-3)
    # null handle / null pointers -> BRNG_ERR_NULL, synchronously
    for name, nargs in (("brng_raw_u32", 3), ("brng_uniform_f32", 5), ("brng_gaussian_f64", 5),
                        ("brng_exponential_f32", 4), ("brng_gamma_f64", 6),
                        ("brng_dirichlet_f32", 6), ("brng_set_offset", 2),
                        ("brng_destroy", 1), ("brng_synchronize", 1)):
        args = [None] + [0] * (nargs - 1)
        assert raw(name, *args) == -1, name
    assert raw("brng_gibbs_triangle", None, 1, 1, None, None, 0, None, None, None, None,
               None) == -1
    assert raw("brng_create", 1, 0, None) == -1


def test_binding_checks_element_size_and_length():
    """The binding refuses arrays whose dtype or length does not match what
    the C call would touch (no memory corruption from a wrong tensor)."""
    import numpy as np
    import paper_1412_4825_b200 as B
    p = B.brng._ptr
    a = np.zeros(8)
    assert p(a, 8, 8) == a.ctypes.data and p(None, 8, 8) is None and p(1234, 8, 8) == 1234
    with pytest.raises(TypeError):
        p(np.zeros(8, np.float32), 8, 8)            # f32 array for an f64 call
    with pytest.raises(ValueError):
        p(a, 8, 9)                                  # too short
    with pytest.raises(ValueError):
        p(np.zeros((4, 4))[:, ::2], 8, 4)           # not contiguous
    with pytest.raises(TypeError):                  # before any C call (no GPU needed)
        B.brng_gaussian_f64(1, np.zeros(4, np.float32), np.zeros(4), np.zeros(4), 4)
    with pytest.raises(ValueError):
        B.brng_gibbs_triangle(1, 10, 3, totals=np.zeros(B.TOTALS_LEN - 1))


def test_create_without_gpu_reports_cuda_error():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1412_4825_b200 as B
    with pytest.raises(B.brng.BrngError) as e:
        B.brng_create(1, 0)
    assert e.value.status == -3


def test_product_path_has_no_oracle_or_fallback(tmp_path):
    pkg = os.path.join(ROOT, "paper_1412_4825_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                src = open(os.path.join(dirpath, f)).read()
                for bad in ("import oracle", "from oracle", "liboracle", "orc_", "oracle.c"):
                    assert bad not in src, f"{f}: {bad}"
    # without libbrng.so the binding refuses to import (no CPU fallback)
    shutil.copy(os.path.join(pkg, "brng.py"), tmp_path / "brng.py")
    spec = importlib.util.spec_from_file_location("brng_nolib", tmp_path / "brng.py")
    mod = importlib.util.module_from_spec(spec)
    with pytest.raises(ImportError):
        spec.loader.exec_module(mod)
