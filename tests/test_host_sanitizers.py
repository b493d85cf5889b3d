"""AddressSanitizer + UndefinedBehaviorSanitizer builds of the host code
(VERDICT r01 item 7), run in the CPU tier:

- the CPU oracle (oracle/oracle.c), every entry point with edge and invalid
  parameters in exactly-sized heap blocks (tests/host_asan/oracle_driver.c);
- the C ABI's host logic (paper_1412_4825_b200/csrc/brng.cpp: validation,
  cursor reservation/overflow, host-buffer chunking and staging, scratch
  growth, teardown) linked against a host-memory fake of the CUDA runtime
  and fake launches that encode the global unit each chunk was given
  (tests/host_asan/*.cpp), checking every element's placement and that
  brng_destroy releases every allocation.
"""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
H = os.path.join(ROOT, "tests", "host_asan")
SAN = ["-O1", "-g", "-fsanitize=address,undefined", "-fno-sanitize-recover=undefined",
       "-fno-omit-frame-pointer"]
ENV = dict(os.environ, ASAN_OPTIONS="detect_leaks=1:abort_on_error=0",
           UBSAN_OPTIONS="print_stacktrace=1")


def _run(cmd_build, exe, tmp_path):
    r = subprocess.run(cmd_build, capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    r = subprocess.run([exe], capture_output=True, text=True, env=ENV, timeout=600)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-4000:])
    return r.stdout


@pytest.mark.skipif(shutil.which("gcc") is None, reason="no gcc")
def test_oracle_asan_ubsan(tmp_path):
    exe = str(tmp_path / "oracle_asan")
    out = _run(["gcc", "-std=c11", "-ffp-contract=off", *SAN, "oracle/oracle.c",
                os.path.join(H, "oracle_driver.c"), "-lm", "-o", exe], exe, tmp_path)
    assert "oracle_asan ok" in out


@pytest.mark.skipif(shutil.which("g++") is None or
                    not os.path.exists("/usr/local/cuda/include/cuda_runtime.h"),
                    reason="no g++ or CUDA headers")
def test_c_abi_host_logic_asan_ubsan(tmp_path):
    exe = str(tmp_path / "host_asan")
    out = _run(["g++", "-std=c++17", *SAN, "-I", "include", "-I", "/usr/local/cuda/include",
                "paper_1412_4825_b200/csrc/brng.cpp", os.path.join(H, "fake_cuda.cpp"),
                os.path.join(H, "fake_kernels.cpp"), os.path.join(H, "driver.cpp"), "-o", exe],
               exe, tmp_path)
    assert "host_asan ok" in out
