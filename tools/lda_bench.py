"""NEXT row N4 measurement: the LDA fold-in Gibbs consumer (brng_lda_gibbs)
with its three deviate sources on the workloads.LDA corpus (D = 100k
documents, K = 64 topics, V = 20k words, ~15M tokens), n_iter iterations per
call, CUDA events on the handle's stream, after warm-up.

usage: python tools/lda_bench.py [n_iter] > profiles/r02_lda.json
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1412_4825_b200 as B  # noqa: E402
import workloads as W  # noqa: E402


def bench_shape(h, D, K, V, mean_len, alpha_v, seed, beta, n_iter):
    dev = torch.device("cuda:0")
    c = W.lda_corpus(D, K, V, mean_len, seed=seed, beta=beta)
    T = c["n_tokens"]
    d = {k: v.to(dev) for k, v in c.items() if k != "n_tokens"}
    alpha = torch.full((K,), alpha_v, dtype=torch.float64, device=dev)
    res = {"workload": f"LDA fold-in: D={D} docs, K={K}, V={V}, T={T} tokens "
                       f"(lengths 1+Poisson({mean_len - 1})), alpha={alpha_v}, "
                       f"phi rows ~ Dirichlet({beta}); {n_iter} iterations per call",
           "per_iteration": {"gamma_draws": D * K, "tokens": T,
                             "philox_blocks": 256 * D * K + (T + 1) // 2}}

    def timed(fn, reps=3):
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return min(ts)
    z_ref = None
    for name, mode in (("inline", B.LDA_INLINE), ("ring", B.LDA_RING), ("bulk", B.LDA_BULK)):
        z = d["z0"].clone()
        B.brng_lda_gibbs(h, D, K, V, T, d["doc_off"], d["words"], d["phi"], alpha, z, None,
                         2, mode)                      # warm-up (allocates ring/bulk scratch)
        torch.cuda.synchronize()

        def run():
            z.copy_(d["z0"])
            B.brng_set_offset(h, 0)
            B.brng_lda_gibbs(h, D, K, V, T, d["doc_off"], d["words"], d["phi"], alpha, z, None,
                             n_iter, mode)
        ms = timed(run) / n_iter
        same = None
        if z_ref is None:
            z_ref = z.clone()
        else:
            same = bool(torch.equal(z, z_ref))
        res[name] = {"ms_per_iteration": round(ms, 3), "Mtokens_per_s": round(T / ms / 1e3, 1),
                     "identical_to_inline": same}
    # the RNG share of an iteration: the same deviates from the bulk C-ABI calls
    # (Dirichlet rows alpha + n and the token uniforms), timed alone
    rows = alpha[None, :].expand(D, K).contiguous() + 1.0
    th = torch.empty(D, K, dtype=torch.float64, device=dev)
    u = torch.empty(T, dtype=torch.float64, device=dev)
    res["rng_alone_ms"] = {
        "dirichlet_f64": round(timed(lambda: B.brng_dirichlet_f64(h, rows, D, K, th, None)), 3),
        "std_uniform_f64": round(timed(lambda: B.brng_std_uniform_f64(h, u, T)), 3)}
    return res


def main():
    n_iter = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    cfg = W.LDA
    h = B.brng_create(cfg["seed"], 0)
    B.brng_set_cuda_stream(h, torch.cuda.current_stream().cuda_stream)
    out = {"headline": bench_shape(h, cfg["n_docs"], cfg["k"], cfg["v"], cfg["mean_len"],
                                   cfg["alpha"], cfg["seed"], cfg["beta"], n_iter),
           "rng_heavy": bench_shape(h, 50_000, 256, 20_000, 40, cfg["alpha"], cfg["seed"],
                                    cfg["beta"], n_iter)}
    out["errors"] = B.brng_device_errors(h)
    B.brng_destroy(h)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
