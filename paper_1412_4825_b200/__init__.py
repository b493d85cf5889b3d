"""paper_1412_4825_b200 -- B200-native varying-parameter random deviates.

The data-parallel hot path of arXiv 1412.4825 (BatchRNG): per-sample
uniform / Gaussian / exponential transforms of Philox4x32-10 standard
deviates, per-sample-alpha Marsaglia-Tsang Gamma, Dirichlet rows and Gibbs
chains on the triangle, as hand-written sm_100a kernels behind a C ABI
(include/brng.h, libbrng.so).  ``brng`` is the thin ctypes binding;
``shard`` holds the multi-GPU host logic (counter-range sharding and the
NCCL reduction of Gibbs totals).
"""
from . import brng  # noqa: F401  (raises ImportError if libbrng.so is missing)
from .brng import *  # noqa: F401,F403

__all__ = list(brng.EXPORTED)
