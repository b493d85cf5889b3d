"""Hash of the LDA consumer's outputs (z, theta after n iterations) for a few
shapes and all three sources, for comparing builds (BRNG_LIB=...).

usage: BRNG_LIB=tools/variants/x.so python tools/lda_hash.py"""
import hashlib
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1412_4825_b200 as B  # noqa: E402
import workloads as W  # noqa: E402

dev = torch.device("cuda:0")
for (D, K, V, L) in ((20000, 64, 5000, 150), (5000, 256, 3000, 40), (3000, 7, 500, 60),
                     (2000, 1024, 800, 90), (4000, 30, 900, 33)):
    c = W.lda_corpus(D, K, V, L, seed=K, beta=0.05)
    d = {k: v.to(dev) for k, v in c.items() if k != "n_tokens"}
    alpha = torch.full((K,), 0.1, dtype=torch.float64, device=dev)
    hs = []
    for mode in (0, 1, 2):
        z = d["z0"].clone()
        th = torch.empty(D, K, dtype=torch.float64, device=dev)
        h = B.brng_create(5, 0)
        B.brng_lda_gibbs(h, D, K, V, c["n_tokens"], d["doc_off"], d["words"], d["phi"], alpha, z,
                         th, 3, mode)
        torch.cuda.synchronize()
        hh = hashlib.sha1(z.cpu().numpy().tobytes() + th.cpu().numpy().tobytes()).hexdigest()[:12]
        hs.append(hh)
        B.brng_destroy(h)
    print(f"D={D} K={K}: {' '.join(hs)}", flush=True)
