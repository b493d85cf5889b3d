"""Independent pin of the GPU Philox4x32-10 (K1): brng_raw_u32 must equal
cuRAND's device Philox (curand_init(seed, stream, 4 pos) + curand4) word for
word -- an implementation that shares nothing with brng or the oracle
(SURVEY.md §4 tier 2).  Edge counters: 32-bit carries of the block cursor,
streams with high bits set, 64-bit seeds."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest
import torch

from tests.gpu_util import dev, handle

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)
import paper_1412_4825_b200 as B  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def curand_lib(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("curand") / "libxcheck.so")
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-O2", "-gencode",
                           "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
                           "-cudart", "shared",
                           os.path.join(ROOT, "tests", "cuda", "curand_xcheck.cu"), "-o", out])
    L = C.CDLL(out)
    L.curand_blocks.argtypes = [C.c_uint64] * 4 + [C.c_void_p, C.c_void_p]
    return L


@pytest.mark.parametrize("seed,stream,cursor", [
    (42, 0, 0), (7, 1, 123456789), (0xDEADBEEFCAFEF00D, 3, 0),
    (11, 0xFFFFFFFF, 2**32 - 100),            # block cursor crosses 2^32
    (3, 2**40 + 5, 2**61 - 50),               # high stream bits, large cursor
    (2**64 - 1, 2**64 - 1, 2**62 - 5000),     # all-ones key and stream
    # (cuRAND's word offset 4 pos is 64-bit: blocks >= 2^62 are out of its reach)
])
def test_raw_words_equal_curand(curand_lib, seed, stream, cursor):
    nblk = 4099
    got = torch.empty(4 * nblk, dtype=torch.int32, device=dev())
    ref = torch.empty_like(got)
    with handle(seed, stream, cursor) as h:
        B.brng_raw_u32(h, got, 4 * nblk)
    s = torch.cuda.current_stream().cuda_stream
    assert curand_lib.curand_blocks(seed, stream, cursor, nblk, ref.data_ptr(), s) == 0
    torch.cuda.synchronize()
    a, b = got.cpu().numpy().view(np.uint32), ref.cpu().numpy().view(np.uint32)
    assert np.array_equal(a, b), int(np.flatnonzero(a != b)[0])
