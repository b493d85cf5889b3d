"""Seeded synthetic inputs for the five BASELINE.json configs.

This module holds NONE of the method's arithmetic: it only draws the
per-sample PARAMETER arrays (the "parameters read as elements of an array in
memory" of PAPER.md P:L82-83) with torch's own generator, so the CUDA
path (paper_1412_4825_b200) and the CPU oracle (oracle/) are fed identical
bytes.  Both sides import it; it imports neither.

Recipes:
  cfg2  mu ~ U(-10,10), sigma ~ logU(1e-3,1e3), a ~ U(-1,0),
        b = a + logU(1e-3,1e3)                      N = 2^28, fp32, seed 7
  cfg3  alpha ~ logU(0.05,200), beta ~ logU(0.1,10) N = 2^26, fp64, seed 11
  cfg4  support ~ Bernoulli(0.1) per (d,k), n ~ Poisson(2) on the support,
        alpha = 0.1 + n                             D = 1e6, K = 256, fp32, seed 3
  cfg1/cfg5 need no parameter arrays (Gibbs from (0.5, 0.5)).
logU(lo,hi) = exp(ln lo + V (ln hi - ln lo)), V ~ U[0,1) from torch.rand in
fp64, then cast.  The deviates themselves use Philox key = the config seed,
stream 0 (cfg1/cfg5: stream = chain id), cursor 0.
"""
from __future__ import annotations

import math

import torch

CFG1 = dict(name="cfg1_gibbs_1024x1000", seed=42, n_chains=1024, n_sweeps=1000)
CFG2 = dict(name="cfg2_fill_2^28_f32", seed=7, n=1 << 28)
CFG3 = dict(name="cfg3_gamma_2^26_f64", seed=11, n=1 << 26)
CFG4 = dict(name="cfg4_dirichlet_1e6x256_f32", seed=3, n_docs=1_000_000, k=256)
CFG5 = dict(name="cfg5_gibbs_2^24x4096", seed=42, n_chains=1 << 24, n_sweeps=4096)


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def _logu(g, n, lo, hi, device):
    v = torch.rand(n, generator=g, dtype=torch.float64, device=device)
    return torch.exp(math.log(lo) + v * (math.log(hi) - math.log(lo)))


def _u(g, n, lo, hi, device):
    v = torch.rand(n, generator=g, dtype=torch.float64, device=device)
    return lo + (hi - lo) * v


def cfg2_params(n: int, seed: int = 7, device="cpu"):
    """Gaussian (mu, sigma) and uniform (a, b) parameter arrays, fp32 [n]."""
    g = _gen(seed, device)
    mu = _u(g, n, -10.0, 10.0, device).to(torch.float32)
    sigma = _logu(g, n, 1e-3, 1e3, device).to(torch.float32)
    a32 = _u(g, n, -1.0, 0.0, device).to(torch.float32)
    b = (a32.to(torch.float64) + _logu(g, n, 1e-3, 1e3, device)).to(torch.float32)
    return dict(mu=mu, sigma=sigma, a=a32, b=b)


def exp_params(n: int, seed: int = 7, device="cpu", dtype=torch.float32):
    """Exponential rate lambda ~ logU(1e-3, 1e3) (extra on-path check)."""
    g = _gen(seed + 1000, device)
    return _logu(g, n, 1e-3, 1e3, device).to(dtype)


def cfg3_params(n: int, seed: int = 11, device="cpu", dtype=torch.float64):
    """Gamma shape alpha ~ logU(0.05,200), scale beta ~ logU(0.1,10)."""
    g = _gen(seed, device)
    alpha = _logu(g, n, 0.05, 200.0, device).to(dtype)
    beta = _logu(g, n, 0.1, 10.0, device).to(dtype)
    return dict(alpha=alpha, beta=beta)


def cfg4_params(n_docs: int, k: int = 256, seed: int = 3, device="cpu",
                dtype=torch.float32):
    """LDA-shaped Dirichlet alpha [n_docs, k] = 0.1 + n_dk on a 10% support."""
    g = _gen(seed, device)
    support = torch.rand(n_docs, k, generator=g, device=device) < 0.1
    rate = torch.full((n_docs, k), 2.0, dtype=torch.float32, device=device)
    n = torch.poisson(rate, generator=g)
    alpha = 0.1 + torch.where(support, n, torch.zeros_like(n)).to(torch.float64)
    return alpha.to(dtype)


# NEXT row N4 (reading R-33): a synthetic LDA fold-in corpus.  Documents'
# lengths ~ 1 + Poisson(mean_len - 1); each document mixes a few topics of a
# fixed topic-word matrix phi (topic rows ~ Dirichlet(beta) over the
# vocabulary, drawn with torch's own generator); initial topics uniform.
LDA = dict(name="lda_foldin_100k_docs_K64", seed=5, n_docs=100_000, k=64, v=20_000,
           mean_len=150, alpha=0.1, beta=0.05)


def lda_corpus(n_docs: int, k: int, v: int, mean_len: float, seed: int = 5,
               beta: float = 0.05, device="cpu"):
    """dict(doc_off u64 [D+1], words u32 [T], phi f64 [V, K], z0 u16 [T], n_tokens)."""
    g = _gen(seed, "cpu")
    lens = 1 + torch.poisson(torch.full((n_docs,), float(mean_len - 1)), generator=g).long()
    doc_off = torch.zeros(n_docs + 1, dtype=torch.int64)
    doc_off[1:] = torch.cumsum(lens, 0)
    T = int(doc_off[-1])
    gam = torch._standard_gamma(torch.full((k, v), float(beta), dtype=torch.float64),
                                generator=g)
    phi_kv = gam / gam.sum(dim=1, keepdim=True)
    # each document draws its words from 3 of the topics (LDA-shaped corpus)
    doc_topics = torch.randint(0, k, (n_docs, 3), generator=g)
    tok_doc = torch.repeat_interleave(torch.arange(n_docs), lens)
    pick = doc_topics[tok_doc, torch.randint(0, 3, (T,), generator=g)]
    words = torch.empty(T, dtype=torch.int64)
    for t in range(k):
        sel = (pick == t).nonzero().squeeze(1)
        if sel.numel():
            words[sel] = torch.multinomial(phi_kv[t], sel.numel(), replacement=True, generator=g)
    z0 = torch.randint(0, k, (T,), generator=g)
    # int64 / int32 / int16 carry the u64 / u32 / u16 bits the C ABI reads
    return dict(doc_off=doc_off.to(device), words=words.to(torch.int32).to(device),
                phi=phi_kv.t().contiguous().to(device), z0=z0.to(torch.int16).to(device),
                n_tokens=T)
