"""Run the LDA consumer (bench shape: D = 100k, K = 64, V = 20k, ~15M tokens)
for a few iterations in one process, for ncu captures.

usage: python tools/run_lda.py [mode 0|1|2] [K] [mean_len] [n_iter]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1412_4825_b200 as B  # noqa: E402
import workloads as W  # noqa: E402

mode = int(sys.argv[1]) if len(sys.argv) > 1 else 0
K = int(sys.argv[2]) if len(sys.argv) > 2 else 64
L = int(sys.argv[3]) if len(sys.argv) > 3 else 150
n_iter = int(sys.argv[4]) if len(sys.argv) > 4 else 2
D, V = 100_000, 20_000
dev = torch.device("cuda:0")
c = W.lda_corpus(D, K, V, L, seed=1, beta=0.05)
d = {k: v.to(dev) for k, v in c.items() if k != "n_tokens"}
alpha = torch.full((K,), 0.1, dtype=torch.float64, device=dev)
h = B.brng_create(5, 0)
B.brng_set_cuda_stream(h, torch.cuda.current_stream().cuda_stream)
z = d["z0"].clone()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(2):
    e0.record()
    B.brng_lda_gibbs(h, D, K, V, c["n_tokens"], d["doc_off"], d["words"], d["phi"], alpha, z,
                     None, n_iter, mode)
    e1.record()
    torch.cuda.synchronize()
print(f"mode {mode} K {K}: {e0.elapsed_time(e1) / n_iter:.3f} ms/iteration, "
      f"T = {c['n_tokens']}, z sum {int(z.long().sum())}")
B.brng_destroy(h)
