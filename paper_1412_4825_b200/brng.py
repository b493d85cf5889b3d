"""Thin Python binding of libbrng's C ABI (include/brng.h) -- marshalling only.

Every function has the C name and argument order; arrays may be torch
tensors (device or host), numpy arrays (host) or raw integer addresses.
Every step of the hot path runs in the CUDA kernels of libbrng.so; there is
no CPU or PyTorch fallback: if the library cannot be loaded, importing this
module raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BRNG_LIB") or os.path.join(_HERE, "libbrng.so")  # BRNG_LIB: tools only

GAMMA_STRIDE = 256
GAMMA_MAX_TRIAL = 255
TOTALS_HDR = 16
TOTALS_LEN = TOTALS_HDR + 256

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libbrng.so not built at {LIB_PATH}: run __graft_entry__.build() "
                      "(python -m paper_1412_4825_b200._build)")
_lib = C.CDLL(LIB_PATH)

_u64, _vp, _int = C.c_uint64, C.c_void_p, C.c_int
_H = C.c_void_p

_SIGS = {
    "brng_create": [_u64, _u64, C.POINTER(_H)],
    "brng_destroy": [_H],
    "brng_set_cuda_stream": [_H, _vp],
    "brng_get_offset": [_H, C.POINTER(_u64)],
    "brng_set_offset": [_H, _u64],
    "brng_get_key": [_H, C.POINTER(_u64), C.POINTER(_u64)],
    "brng_device_errors": [_H, C.POINTER(_u64)],
    "brng_reset_device_errors": [_H],
    "brng_synchronize": [_H],
    "brng_raw_u32": [_H, _vp, _u64],
    "brng_std_uniform_f32": [_H, _vp, _u64],
    "brng_std_uniform_f64": [_H, _vp, _u64],
    "brng_uniform_f32": [_H, _vp, _vp, _vp, _u64],
    "brng_uniform_f64": [_H, _vp, _vp, _vp, _u64],
    "brng_gaussian_f32": [_H, _vp, _vp, _vp, _u64],
    "brng_gaussian_f64": [_H, _vp, _vp, _vp, _u64],
    "brng_exponential_f32": [_H, _vp, _vp, _u64],
    "brng_exponential_f64": [_H, _vp, _vp, _u64],
    "brng_batch_fill": [_H, _int, _int, C.c_double, C.c_double, _vp, _u64],
    "brng_log_uniform_f32": [_H, _vp, _u64],
    "brng_log_uniform_f64": [_H, _vp, _u64],
    "brng_laplace_f32": [_H, _vp, _vp, _vp, _u64],
    "brng_laplace_f64": [_H, _vp, _vp, _vp, _u64],
    "brng_weibull_f32": [_H, _vp, _vp, _vp, _u64],
    "brng_weibull_f64": [_H, _vp, _vp, _vp, _u64],
    "brng_gamma_f32": [_H, _vp, _vp, _vp, _u64, _vp],
    "brng_gamma_f64": [_H, _vp, _vp, _vp, _u64, _vp],
    "brng_dirichlet_f32": [_H, _vp, _u64, _u64, _vp, _vp],
    "brng_dirichlet_f64": [_H, _vp, _u64, _u64, _vp, _vp],
    "brng_gibbs_triangle": [_H, _u64, _u64, _vp, _vp, _u64, _vp, _vp, _vp, _vp, _vp],
    "brng_lda_gibbs": [_H, _u64, C.c_uint32, C.c_uint32, _u64, _vp, _vp, _vp, _vp, _vp, _vp,
                       C.c_uint32, _int],
}
for _name, _args in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _int
_lib.brng_status_string.argtypes = [_int]
_lib.brng_status_string.restype = C.c_char_p
_lib.brng_version.restype = _int

EXPORTED = sorted(list(_SIGS) + ["brng_status_string", "brng_version"])


class BrngError(RuntimeError):
    def __init__(self, fn, status):
        self.status = status
        super().__init__(f"{fn}: {brng_status_string(status)} ({status})")


def _ptr(x, itemsize=None, count=None):
    """torch.Tensor / numpy array / int / None -> address (no copies).

    For tensors and arrays the element size and length are checked against
    what the C call will touch (itemsize bytes x count elements), so a wrong
    dtype or a short array raises instead of corrupting memory.  Raw integer
    addresses are passed through unchecked."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    dp = getattr(x, "data_ptr", None)
    if dp is not None:
        if not x.is_contiguous():
            raise ValueError("brng: arrays must be contiguous")
        size, length, addr = x.element_size(), x.numel(), dp()
    else:
        ct = getattr(x, "ctypes", None)
        if ct is None:
            raise TypeError(f"brng: unsupported array type {type(x)}")
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("brng: arrays must be contiguous")
        size, length, addr = x.itemsize, x.size, ct.data
    if itemsize is not None and size != itemsize:
        raise TypeError(f"brng: expected {itemsize}-byte elements, got {size}-byte")
    if count is not None and length < count:
        raise ValueError(f"brng: array of {length} elements, the call needs {count}")
    return addr


def _check(fn, st):
    if st != 0:
        raise BrngError(fn, st)
    return st


def brng_status_string(status: int) -> str:
    return _lib.brng_status_string(status).decode()


def brng_version() -> int:
    return _lib.brng_version()


def brng_create(seed: int, stream_id: int = 0) -> int:
    h = _H()
    _check("brng_create", _lib.brng_create(seed, stream_id, C.byref(h)))
    return h.value


def brng_destroy(h) -> int:
    return _check("brng_destroy", _lib.brng_destroy(h))


def brng_set_cuda_stream(h, cuda_stream) -> int:
    return _check("brng_set_cuda_stream", _lib.brng_set_cuda_stream(h, cuda_stream))


def brng_get_offset(h) -> int:
    v = _u64()
    _check("brng_get_offset", _lib.brng_get_offset(h, C.byref(v)))
    return v.value


def brng_set_offset(h, cursor: int) -> int:
    return _check("brng_set_offset", _lib.brng_set_offset(h, cursor))


def brng_get_key(h):
    s, st = _u64(), _u64()
    _check("brng_get_key", _lib.brng_get_key(h, C.byref(s), C.byref(st)))
    return s.value, st.value


def brng_device_errors(h) -> int:
    v = _u64()
    _check("brng_device_errors", _lib.brng_device_errors(h, C.byref(v)))
    return v.value


def brng_reset_device_errors(h) -> int:
    return _check("brng_reset_device_errors", _lib.brng_reset_device_errors(h))


def brng_synchronize(h) -> int:
    return _check("brng_synchronize", _lib.brng_synchronize(h))


def _fill(name, h, n, *arrays):
    size = 8 if name.endswith("f64") else 4
    return _check(name, getattr(_lib, name)(h, *[_ptr(a, size, n) for a in arrays], n))


def brng_raw_u32(h, out, n):
    return _fill("brng_raw_u32", h, n, out)


def brng_std_uniform_f32(h, out, n):
    return _fill("brng_std_uniform_f32", h, n, out)


def brng_std_uniform_f64(h, out, n):
    return _fill("brng_std_uniform_f64", h, n, out)


def brng_uniform_f32(h, a, b, out, n):
    return _fill("brng_uniform_f32", h, n, a, b, out)


def brng_uniform_f64(h, a, b, out, n):
    return _fill("brng_uniform_f64", h, n, a, b, out)


def brng_gaussian_f32(h, mu, sigma, out, n):
    return _fill("brng_gaussian_f32", h, n, mu, sigma, out)


def brng_gaussian_f64(h, mu, sigma, out, n):
    return _fill("brng_gaussian_f64", h, n, mu, sigma, out)


def brng_exponential_f32(h, lam, out, n):
    return _fill("brng_exponential_f32", h, n, lam, out)


def brng_exponential_f64(h, lam, out, n):
    return _fill("brng_exponential_f64", h, n, lam, out)


DIST = {"uniform": 2, "gaussian": 3, "exponential": 4, "laplace": 6, "weibull": 7}
DTYPE = {"f32": 0, "f64": 1}


def brng_batch_fill(h, dist, dtype, p0, p1, out, n):
    """Fixed-parameter fill; dist/dtype are the BRNG_DIST_*/BRNG_DTYPE_* codes."""
    size = 8 if dtype == DTYPE["f64"] else 4
    return _check("brng_batch_fill", _lib.brng_batch_fill(h, dist, dtype, p0, p1,
                                                          _ptr(out, size, n), n))


def brng_log_uniform_f32(h, out, n):
    return _fill("brng_log_uniform_f32", h, n, out)


def brng_log_uniform_f64(h, out, n):
    return _fill("brng_log_uniform_f64", h, n, out)


def brng_laplace_f32(h, mu, beta, out, n):
    return _fill("brng_laplace_f32", h, n, mu, beta, out)


def brng_laplace_f64(h, mu, beta, out, n):
    return _fill("brng_laplace_f64", h, n, mu, beta, out)


def brng_weibull_f32(h, alpha, beta, out, n):
    return _fill("brng_weibull_f32", h, n, alpha, beta, out)


def brng_weibull_f64(h, alpha, beta, out, n):
    return _fill("brng_weibull_f64", h, n, alpha, beta, out)


def brng_gamma_f32(h, alpha, beta, out, n, trials=None):
    return _check("brng_gamma_f32", _lib.brng_gamma_f32(
        h, _ptr(alpha, 4, n), _ptr(beta, 4, n), _ptr(out, 4, n), n, _ptr(trials, 1, n)))


def brng_gamma_f64(h, alpha, beta, out, n, trials=None):
    return _check("brng_gamma_f64", _lib.brng_gamma_f64(
        h, _ptr(alpha, 8, n), _ptr(beta, 8, n), _ptr(out, 8, n), n, _ptr(trials, 1, n)))


def brng_dirichlet_f32(h, alpha, n_rows, k, out, trials=None):
    m = n_rows * k
    return _check("brng_dirichlet_f32", _lib.brng_dirichlet_f32(
        h, _ptr(alpha, 4, m), n_rows, k, _ptr(out, 4, m), _ptr(trials, 1, m)))


def brng_dirichlet_f64(h, alpha, n_rows, k, out, trials=None):
    m = n_rows * k
    return _check("brng_dirichlet_f64", _lib.brng_dirichlet_f64(
        h, _ptr(alpha, 8, m), n_rows, k, _ptr(out, 8, m), _ptr(trials, 1, m)))


def brng_gibbs_triangle(h, n_chains, n_sweeps, x0=None, y0=None, burn_in=0, out_x=None,
                        out_y=None, chain_stats=None, final_xy=None, totals=None):
    c, s = n_chains, n_chains * n_sweeps
    return _check("brng_gibbs_triangle", _lib.brng_gibbs_triangle(
        h, n_chains, n_sweeps, _ptr(x0, 8, c), _ptr(y0, 8, c), burn_in, _ptr(out_x, 8, s),
        _ptr(out_y, 8, s), _ptr(chain_stats, 8, 5 * c), _ptr(final_xy, 8, 2 * c),
        _ptr(totals, 8, TOTALS_LEN)))


def raw_call(name, *args):
    """Call any exported symbol with raw arguments and return its status
    (used by the error-path tests; no checking)."""
    return getattr(_lib, name)(*args)


LDA_INLINE, LDA_RING, LDA_BULK = 0, 1, 2
LDA_MAX_K = 1024


def brng_lda_gibbs(h, n_docs, k, v, n_tokens, doc_off, words, phi, alpha, z, theta=None,
                   n_iter=1, mode=LDA_INLINE):
    """LDA fold-in Gibbs (NEXT row N4, include/brng.h): n_iter iterations on
    device arrays; z (u16) is updated in place."""
    return _check("brng_lda_gibbs", _lib.brng_lda_gibbs(
        h, n_docs, k, v, n_tokens, _ptr(doc_off, 8, n_docs + 1), _ptr(words, 4, n_tokens),
        _ptr(phi, 8, v * k), _ptr(alpha, 8, k), _ptr(z, 2, n_tokens),
        _ptr(theta, 8, n_docs * k), n_iter, mode))
