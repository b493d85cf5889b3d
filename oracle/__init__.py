"""CPU oracle for the BatchRNG hot path -- TEST INFRASTRUCTURE ONLY.

Thin numpy/ctypes wrapper over ``oracle/oracle.c`` (plain single-threaded C,
fp64, ``-ffp-contract=off``).  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this.
It never imports ``paper_1412_4825_b200`` and the CUDA path never imports it.

Every function cites the PAPER.md passage (P:Lnn) or DESIGN.md reading (R-nn)
it implements; the pins live in ``tests/test_oracle_*.py``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

GAMMA_STRIDE = 256          # blocks reserved per Gamma sample (R-11)
GAMMA_MAX_TRIAL = 255
TOTALS_HDR = 16             # Gibbs totals header length (R-18)
TOTALS_LEN = TOTALS_HDR + 256


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (plain gcc, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
               "-fPIC", "-shared", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None
_lock = threading.Lock()

u64, u32, i32, dbl = C.c_uint64, C.c_uint32, C.c_int, C.c_double
vp = C.c_void_p


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = C.CDLL(build())
            L.orc_philox4x32_10.argtypes = [vp, vp, vp]
            L.orc_block.argtypes = [u64, u64, u64, vp]
            L.orc_u24.argtypes = [u32]; L.orc_u24.restype = dbl
            L.orc_u53.argtypes = [u32, u32]; L.orc_u53.restype = dbl
            L.orc_u32d.argtypes = [u32]; L.orc_u32d.restype = dbl
            L.orc_cos2pi.argtypes = [dbl]; L.orc_cos2pi.restype = dbl
            L.orc_sin2pi.argtypes = [dbl]; L.orc_sin2pi.restype = dbl
            L.orc_box_muller.argtypes = [dbl, dbl, i32]; L.orc_box_muller.restype = dbl
            for nm in ("orc_raw_u32", "orc_std_uniform_f32", "orc_std_uniform_f64"):
                getattr(L, nm).argtypes = [u64, u64, u64, vp, u64]
            for sfx in ("f32", "f64"):
                getattr(L, "orc_uniform_" + sfx).argtypes = [u64, u64, u64, vp, vp, vp, u64, u64]
                getattr(L, "orc_gaussian_" + sfx).argtypes = [u64, u64, u64, vp, vp, vp, u64, u64]
                getattr(L, "orc_exponential_" + sfx).argtypes = [u64, u64, u64, vp, vp, u64, u64]
                getattr(L, "orc_gamma_" + sfx).argtypes = [u64, u64, u64, vp, vp, vp, vp, u64, u64]
                getattr(L, "orc_dirichlet_" + sfx).argtypes = [u64, u64, u64, vp, u64, vp, vp,
                                                               u64, u64, vp]
                for nm in ("orc_uniform_", "orc_gaussian_", "orc_exponential_", "orc_gamma_",
                           "orc_dirichlet_"):
                    getattr(L, nm + sfx).restype = u64
            for sfx in ("f32", "f64"):
                getattr(L, "orc_log_uniform_" + sfx).argtypes = [u64, u64, u64, vp, u64, u64]
                getattr(L, "orc_laplace_" + sfx).argtypes = [u64, u64, u64, vp, vp, vp, u64, u64]
                getattr(L, "orc_weibull_" + sfx).argtypes = [u64, u64, u64, vp, vp, vp, u64, u64]
                getattr(L, "orc_laplace_" + sfx).restype = u64
                getattr(L, "orc_weibull_" + sfx).restype = u64
            L.orc_mt_trial.argtypes = [dbl, dbl, dbl, dbl, dbl, vp, vp, vp]
            L.orc_mt_trial.restype = i32
            L.orc_mt_consts.argtypes = [dbl, vp, vp]
            L.orc_mt_trial_uniforms.argtypes = [u64, u64, u64, u64, u32, vp, vp, vp]
            L.orc_gamma_one.argtypes = [u64, u64, u64, u64, dbl, dbl, vp, vp]
            L.orc_gamma_one.restype = dbl
            L.orc_gibbs_triangle.argtypes = [u64, u64, u64, u64, u64, vp, vp, u64,
                                             vp, vp, vp, vp, vp]
            L.orc_gibbs_triangle.restype = u64
            _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


# --------------------------------------------------------------------------
# 1-2. Philox4x32-10 and word -> uniform conversions (R-01..R-04)
# --------------------------------------------------------------------------
def philox4x32_10(ctr, key) -> np.ndarray:
    """One Philox4x32-10 block: ctr = 4 u32, key = 2 u32 -> 4 u32."""
    c = _c(ctr, np.uint32); k = _c(key, np.uint32); out = np.zeros(4, np.uint32)
    lib().orc_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def block(seed: int, stream: int, pos: int) -> np.ndarray:
    """Counter map (R-02): key=(lo,hi seed), ctr=(lo,hi pos, lo,hi stream)."""
    out = np.zeros(4, np.uint32)
    lib().orc_block(seed, stream, pos, _p(out))
    return out


def u24(w: int) -> float:
    return lib().orc_u24(w)


def u53(lo: int, hi: int) -> float:
    return lib().orc_u53(lo, hi)


def u32d(w: int) -> float:
    return lib().orc_u32d(w)


def cos2pi(u: float) -> float:
    return lib().orc_cos2pi(u)


def sin2pi(u: float) -> float:
    return lib().orc_sin2pi(u)


def box_muller(u_r: float, u_theta: float, use_sin: bool) -> float:
    return lib().orc_box_muller(u_r, u_theta, int(use_sin))


def raw_u32(seed, stream, base, n) -> np.ndarray:
    out = np.zeros(n, np.uint32)
    lib().orc_raw_u32(seed, stream, base, _p(out), n)
    return out


def std_uniform(seed, stream, base, n, dtype=np.float64) -> np.ndarray:
    out = np.zeros(n, dtype)
    f = lib().orc_std_uniform_f64 if dtype == np.float64 else lib().orc_std_uniform_f32
    f(seed, stream, base, _p(out), n)
    return out


def _sfx(dtype):
    return "f64" if np.dtype(dtype) == np.float64 else "f32"


# --------------------------------------------------------------------------
# 3. Reducible distributions (R-06, R-07, R-12)
#    i0 = index of the first sample computed (for sampled parity at full size)
# --------------------------------------------------------------------------
def uniform(seed, stream, base, a, b, i0=0, dtype=None):
    dtype = dtype or a.dtype
    a = _c(a, dtype); b = _c(b, dtype); out = np.empty(a.shape, dtype)
    nbad = getattr(lib(), "orc_uniform_" + _sfx(dtype))(seed, stream, base, _p(a), _p(b),
                                                         _p(out), i0, a.size)
    return out, int(nbad)


def gaussian(seed, stream, base, mu, sigma, i0=0, dtype=None):
    dtype = dtype or mu.dtype
    mu = _c(mu, dtype); sigma = _c(sigma, dtype); out = np.empty(mu.shape, dtype)
    nbad = getattr(lib(), "orc_gaussian_" + _sfx(dtype))(seed, stream, base, _p(mu),
                                                          _p(sigma), _p(out), i0, mu.size)
    return out, int(nbad)


def exponential(seed, stream, base, lam, i0=0, dtype=None):
    dtype = dtype or lam.dtype
    lam = _c(lam, dtype); out = np.empty(lam.shape, dtype)
    nbad = getattr(lib(), "orc_exponential_" + _sfx(dtype))(seed, stream, base, _p(lam),
                                                             _p(out), i0, lam.size)
    return out, int(nbad)


# --------------------------------------------------------------------------
# 3b. NEXT row N2: log-uniform, Laplace, Weibull (R-30)
# --------------------------------------------------------------------------
def log_uniform(seed, stream, base, n, i0=0, dtype=np.float64):
    out = np.empty(n, dtype)
    getattr(lib(), "orc_log_uniform_" + _sfx(dtype))(seed, stream, base, _p(out), i0, n)
    return out


def laplace(seed, stream, base, mu, beta, i0=0, dtype=None):
    dtype = dtype or mu.dtype
    mu = _c(mu, dtype); beta = _c(beta, dtype); out = np.empty(mu.shape, dtype)
    nbad = getattr(lib(), "orc_laplace_" + _sfx(dtype))(seed, stream, base, _p(mu), _p(beta),
                                                         _p(out), i0, mu.size)
    return out, int(nbad)


def weibull(seed, stream, base, alpha, beta, i0=0, dtype=None):
    dtype = dtype or alpha.dtype
    alpha = _c(alpha, dtype); beta = _c(beta, dtype); out = np.empty(alpha.shape, dtype)
    nbad = getattr(lib(), "orc_weibull_" + _sfx(dtype))(seed, stream, base, _p(alpha),
                                                         _p(beta), _p(out), i0, alpha.size)
    return out, int(nbad)


# --------------------------------------------------------------------------
# 4. Gamma (Marsaglia-Tsang; R-08..R-11)
# --------------------------------------------------------------------------
def mt_consts(alpha: float):
    d = C.c_double(); c = C.c_double()
    lib().orc_mt_consts(alpha, C.byref(d), C.byref(c))
    return d.value, c.value


def mt_trial(d, c, u_r, u_theta, U):
    """Return (accepted, g, margin, 1+cz) of one Marsaglia-Tsang trial."""
    g = C.c_double(np.nan); m = C.c_double(); t = C.c_double()
    acc = lib().orc_mt_trial(d, c, u_r, u_theta, U, C.byref(g), C.byref(m), C.byref(t))
    return bool(acc), g.value, m.value, t.value


def mt_trial_uniforms(seed, stream, base, i, t):
    a = C.c_double(); b = C.c_double(); U = C.c_double()
    lib().orc_mt_trial_uniforms(seed, stream, base, i, t, C.byref(a), C.byref(b), C.byref(U))
    return a.value, b.value, U.value


def gamma_one(seed, stream, base, i, alpha, beta):
    t = C.c_uint32(); bad = C.c_int()
    g = lib().orc_gamma_one(seed, stream, base, i, alpha, beta, C.byref(t), C.byref(bad))
    return g, t.value, bool(bad.value)


def gamma(seed, stream, base, alpha, beta, i0=0, dtype=None):
    """Returns (out, trials u8, n_invalid) for samples i0 .. i0+len-1."""
    dtype = dtype or alpha.dtype
    alpha = _c(alpha, dtype); beta = _c(beta, dtype)
    out = np.empty(alpha.shape, dtype); tr = np.zeros(alpha.shape, np.uint8)
    nbad = getattr(lib(), "orc_gamma_" + _sfx(dtype))(seed, stream, base, _p(alpha), _p(beta),
                                                       _p(out), _p(tr), i0, alpha.size)
    return out, tr, int(nbad)


def gamma_tie_margin(seed, stream, base, i, alpha, t):
    """Oracle margin of trial t of sample i (for the tie rule)."""
    d, c = mt_consts(alpha)
    ur, ut, U = mt_trial_uniforms(seed, stream, base, i, t)
    _, _, m, onepcz = mt_trial(d, c, ur, ut, U)
    return m, onepcz, d


# --------------------------------------------------------------------------
# 5. Dirichlet (P:L34 footnote; R-13).  alpha: [n_rows, K]
# --------------------------------------------------------------------------
def dirichlet(seed, stream, base, alpha, row0=0, dtype=None):
    dtype = dtype or alpha.dtype
    alpha = _c(alpha, dtype)
    n_rows, k = alpha.shape
    out = np.empty(alpha.shape, dtype); tr = np.zeros(alpha.shape, np.uint8)
    scratch = np.empty(k, np.float64)
    nbad = getattr(lib(), "orc_dirichlet_" + _sfx(dtype))(seed, stream, base, _p(alpha), k,
                                                           _p(out), _p(tr), row0, n_rows,
                                                           _p(scratch))
    return out, tr, int(nbad)


# --------------------------------------------------------------------------
# 6. Gibbs triangle (Eq. 1 / Fig. 1; R-14..R-19)
# --------------------------------------------------------------------------
def gibbs_triangle(seed, stream_id, base, n_chains, n_sweeps, x0=None, y0=None, burn_in=0,
                   want_samples=True):
    """Returns dict(out_x, out_y [n_sweeps, n_chains], chain_stats [5, n_chains],
    final_xy [2, n_chains], totals [272], n_invalid)."""
    x0a = None if x0 is None else _c(x0, np.float64)
    y0a = None if y0 is None else _c(y0, np.float64)
    ox = np.empty((n_sweeps, n_chains)) if want_samples else None
    oy = np.empty((n_sweeps, n_chains)) if want_samples else None
    st = np.empty((5, n_chains)); fx = np.empty((2, n_chains)); tot = np.zeros(TOTALS_LEN)
    nbad = lib().orc_gibbs_triangle(seed, stream_id, base, n_chains, n_sweeps, _p(x0a), _p(y0a),
                                    burn_in, _p(ox), _p(oy), _p(st), _p(fx), _p(tot))
    return dict(out_x=ox, out_y=oy, chain_stats=st, final_xy=fx, totals=tot,
                n_invalid=int(nbad))


# --------------------------------------------------------------------------
# Threaded driver for the CPU baseline: P workers, each a single-threaded oracle
# call on a disjoint contiguous slice (ctypes releases the GIL during calls).
# --------------------------------------------------------------------------
def run_parallel(fn, slices, n_threads):
    """fn(lo, hi) for each (lo, hi) in slices on n_threads Python threads."""
    it = iter(slices)
    it_lock = threading.Lock()

    def worker():
        while True:
            with it_lock:
                nxt = next(it, None)
            if nxt is None:
                return
            fn(*nxt)

    ths = [threading.Thread(target=worker) for _ in range(n_threads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()


# --------------------------------------------------------------------------
# 8. NEXT row N4: LDA fold-in Gibbs, the paper's LDA use ("sample from
#    a Dirichlet distribution whose parameters are updated during each
#    iteration"; footnote: Dirichlet from normalised Gammas) with a fixed
#    topic-word matrix phi.  Reading R-33, one iteration at
#    cursor `base`:
#      n_dk  = #{tokens of doc d with z = k}
#      theta = Dirichlet(alpha + n_d.) drawn as brng_dirichlet_f64 at `base`
#              (component (d, k) = Gamma sample d K + k, beta = 1)
#      u_j   = standard uniform f64 sample j at base + 256 D K
#      z_j   = first k with fl(u_j C_j) < c_jk, c_jk = fl(c_j,k-1 + fl(theta_dk
#              phi[w_j, k])), C_j = c_j,K-1 (else the last k with p > 0)
#    Built from oracle.dirichlet and oracle.std_uniform; the categorical step
#    is plain Python floats in the stated order.
# --------------------------------------------------------------------------
def lda_span(n_docs, k, n_tokens):
    """Philox blocks one LDA iteration consumes (R-33)."""
    return GAMMA_STRIDE * n_docs * k + (n_tokens + 1) // 2


def lda_counts(doc_off, z, k):
    """n_dk = #{tokens of doc d assigned topic k} (f64 [D, K])."""
    D = len(doc_off) - 1
    n = np.zeros((D, k))
    for d in range(D):
        for j in range(int(doc_off[d]), int(doc_off[d + 1])):
            n[d, int(z[j])] += 1.0
    return n


def lda_categorical(theta_d, phi_w, u):
    """z for one token: returns (z, x, c) with x = fl(u C) and c the running
    sums, so a caller can classify a disagreement as a rounding tie."""
    c = []
    acc = 0.0
    last = 0
    for kk in range(len(theta_d)):
        p = float(theta_d[kk]) * float(phi_w[kk])
        acc = acc + p
        c.append(acc)
        if p > 0.0:
            last = kk
    x = float(u) * acc
    for kk in range(len(c)):
        if x < c[kk]:
            return kk, x, c
    return last, x, c


def lda_iteration(seed, stream, base, doc_off, words, phi, alpha, z):
    """One fold-in Gibbs iteration (R-33).  phi: [V, K] f64, alpha: [K] f64,
    z: current topics [T].  Returns dict(z, theta [D, K], trials, x [T],
    cum (list of running-sum lists per token))."""
    doc_off = np.asarray(doc_off, np.int64)
    D, K = len(doc_off) - 1, phi.shape[1]
    T = int(doc_off[-1])
    rows = np.asarray(alpha, np.float64)[None, :] + lda_counts(doc_off, z, K)
    theta, trials, _ = dirichlet(seed, stream, base, rows, dtype=np.float64)
    u = std_uniform(seed, stream, base + GAMMA_STRIDE * D * K, T, np.float64)
    z_new = np.empty(T, np.int64)
    xs = np.empty(T)
    cums = []
    for d in range(D):
        for j in range(int(doc_off[d]), int(doc_off[d + 1])):
            zz, x, c = lda_categorical(theta[d], phi[int(words[j])], u[j])
            z_new[j] = zz
            xs[j] = x
            cums.append(c)
    return dict(z=z_new, theta=theta, trials=trials, rows=rows, u=u, x=xs, cum=cums)
