"""The measurement tools and bench.py at least compile (they run only on a
GPU box, so a syntax error would otherwise surface there first)."""
import glob
import os
import py_compile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FILES = sorted(glob.glob(os.path.join(ROOT, "tools", "*.py"))) + [os.path.join(ROOT, "bench.py"),
                                                                   os.path.join(ROOT, "__graft_entry__.py")]


@pytest.mark.parametrize("path", FILES, ids=[os.path.relpath(p, ROOT) for p in FILES])
def test_compiles(path, tmp_path):
    py_compile.compile(path, cfile=str(tmp_path / "x.pyc"), doraise=True)


CU = sorted(glob.glob(os.path.join(ROOT, "tools", "*.cu")))
NVCC = "/usr/local/cuda/bin/nvcc"


@pytest.mark.skipif(not os.path.exists(NVCC), reason="no nvcc")
@pytest.mark.parametrize("path", CU, ids=[os.path.relpath(p, ROOT) for p in CU])
def test_microbenchmarks_compile_for_sm100a(path, tmp_path):
    import subprocess
    subprocess.run([NVCC, "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-c", path, "-o",
                    str(tmp_path / "x.o")], check=True, capture_output=True)
