"""Host-side validation of the C ABI on a real device (include/brng.h
"Errors"): problems are reported synchronously with no launch and no cursor
change; n == 0 is a no-op."""
import pytest
import torch

pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)
import paper_1412_4825_b200 as B  # noqa: E402
from tests.gpu_util import dev, handle  # noqa: E402

raw = B.brng.raw_call


def test_error_codes_and_cursor_untouched():
    x = torch.empty(16, dtype=torch.float64, device=dev())
    with handle(1, 0, 123) as h:
        # n == 0: no-op
        assert raw("brng_gamma_f64", h, x.data_ptr(), x.data_ptr(), x.data_ptr(), 0, None) == 0
        assert raw("brng_uniform_f64", h, x.data_ptr(), x.data_ptr(), x.data_ptr(), 0) == 0
        assert B.brng_get_offset(h) == 123
        # null required pointers
        assert raw("brng_gaussian_f64", h, None, x.data_ptr(), x.data_ptr(), 4) == -1
        assert raw("brng_gamma_f64", h, x.data_ptr(), None, x.data_ptr(), 4, None) == -1
        # k == 0
        assert raw("brng_dirichlet_f64", h, x.data_ptr(), 2, 0, x.data_ptr(), None) == -2
        # burn_in > n_sweeps; n_sweeps beyond the histogram bound
        assert raw("brng_gibbs_triangle", h, 4, 3, None, None, 4, None, None, None, None,
                   None) == -2
        assert raw("brng_gibbs_triangle", h, 4, 1 << 22, None, None, 0, None, None, None, None,
                   None) == -2
        assert B.brng_get_offset(h) == 123
        # cursor overflow past 2^64 (Gamma reserves 256 blocks per sample)
        B.brng_set_offset(h, (1 << 64) - 1000)
        assert raw("brng_gamma_f64", h, x.data_ptr(), x.data_ptr(), x.data_ptr(), 16, None) == -5
        assert raw("brng_uniform_f64", h, x.data_ptr(), x.data_ptr(), x.data_ptr(), 16) == 0
        assert B.brng_get_offset(h) == (1 << 64) - 1000 + 8
        # unknown dist / dtype of the batch fill
        assert raw("brng_batch_fill", h, 99, 0, 0.0, 1.0, x.data_ptr(), 4) == -4
        assert raw("brng_batch_fill", h, 2, 7, 0.0, 1.0, x.data_ptr(), 4) == -4
        assert B.brng_status_string(-5) == "Philox cursor overflow"
        torch.cuda.synchronize()


def test_handles_are_independent_and_keyed():
    n = 1000
    with handle(5, 0) as h1, handle(5, 1) as h2, handle(6, 0) as h3:
        o = [torch.empty(n, dtype=torch.float64, device=dev()) for _ in range(3)]
        for h, out in zip((h1, h2, h3), o):
            B.brng_std_uniform_f64(h, out, n)
        assert not torch.equal(o[0], o[1]) and not torch.equal(o[0], o[2])
        assert B.brng_get_key(h2) == (5, 1)


def test_stream_switch_orders_the_handles_work():
    """A handle's calls share device scratch (the Gamma/Dirichlet work
    counter, the Gibbs partials): after brng_set_cuda_stream the new stream
    waits for the old one, so back-to-back calls on two streams give the
    results of the same calls on one stream."""
    import workloads
    n = 1 << 25                  # ~0.4 ms kernels: the second call is enqueued mid-run
    p = workloads.cfg3_params(n, seed=11, device=dev())
    ref = [torch.empty(n, dtype=torch.float64, device=dev()) for _ in range(2)]
    got = [torch.empty(n, dtype=torch.float64, device=dev()) for _ in range(2)]
    with handle(11, 0) as h:
        for o in ref:
            B.brng_gamma_f64(h, p["alpha"], p["beta"], o, n)
        torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    h = B.brng_create(11, 0)
    try:
        B.brng_set_cuda_stream(h, s1.cuda_stream)
        B.brng_gamma_f64(h, p["alpha"], p["beta"], got[0], n)
        B.brng_set_cuda_stream(h, s2.cuda_stream)
        B.brng_gamma_f64(h, p["alpha"], p["beta"], got[1], n)
        torch.cuda.synchronize()
        assert B.brng_device_errors(h) == 0
    finally:
        B.brng_destroy(h)
    assert torch.equal(got[0], ref[0]) and torch.equal(got[1], ref[1])
