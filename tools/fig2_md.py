"""Render profiles/r01_fig2.md from the JSON that tools/fig2.py prints.

usage: python tools/fig2_md.py profiles/r01_fig2.json > profiles/r01_fig2.md
The paper columns are PAPER.md's Fig. 2 numbers (CCPS of VSL
Batch / VSL OAAT / BatchRNG on a 2.6 GHz Xeon E5-2670), context only.
"""
import json
import sys

PAPER = {  # distribution: (batch CCPS, OAAT CCPS, BatchRNG CCPS, speedup) -- P:L97-119
    "uniform": (4.3, 65.1, 12.4, 5.2), "gaussian": (25.5, 1105.4, 34.6, 31.9),
    "exponential": (12.2, 646.0, 14.2, 45.5), "laplace": (15.7, 706.4, 41.9, 16.9),
    "weibull": (16.3, 857.6, 22.9, 37.5), "gamma": (51.0, 1316.0, 84.0, 15.7),
}


def main():
    d = json.load(open(sys.argv[1]))
    out = [f"# NEXT row N1: the paper's Fig. 2 on one B200 (binary64, n = {d['n']})", "",
           "GPU analogues of the paper's columns (P:L79-85): batch = fixed-parameter call "
           "(`brng_batch_fill`); OAAT-naive = one n=1 call (kernel launch) per sample; brng = "
           "per-sample parameters read from HBM (fused kernels); two-pass = standard deviates "
           "materialised in HBM then a separate transform; torch = stock PyTorch with "
           "per-sample parameters. Times are ns/sample (best of 5, CUDA events). Paper "
           "columns: CCPS on a 2.6 GHz Xeon E5-2670 (P:L97-119), context only. "
           "`tools/fig2.py`, rendered by `tools/fig2_md.py`.", "",
           "| distribution | batch ns | OAAT-naive ns | brng ns | two-pass ns | torch ns | "
           "brng / batch | OAAT / brng | paper batch / OAAT / BatchRNG CCPS (speedup) |",
           "|---|---|---|---|---|---|---|---|---|"]
    hbm = []
    for k, v in d["rows"].items():
        g = lambda c: v.get(c, {}).get("ns_per_sample")  # noqa: E731
        f = lambda x: "—" if x is None else f"{x:.4f}" if x < 1 else f"{x:.0f}"  # noqa: E731
        p = PAPER.get(k)
        pc = f"{p[0]} / {p[1]} / {p[2]} ({p[3]}x)" if p else "—"
        out.append(f"| {k} | {f(g('batch'))} | {f(g('oaat_naive'))} | {f(g('brng'))} | "
                   f"{f(g('two_pass'))} | {f(g('torch'))} | {v['brng_over_batch_time']:.3f} | "
                   f"{v['speedup_oaat_over_brng']:.0f}x | {pc} |")
        b = v["brng"]
        if "GB_per_s" in b:
            hbm.append(f"{k} {b['GB_per_s']:.1f} GB/s ({b['hbm_frac']:.0%})")
    out += ["", "brng HBM throughput (per-sample parameters + output, 8 B each; fraction of "
            "the measured HBM peak): " + ", ".join(hbm), ""]
    print("\n".join(out))


if __name__ == "__main__":
    main()
