"""Summarise ncu captures (.ncu-rep) and an ncu launch list (.csv) into
profiles/: a markdown table per kernel and a JSON of the key metrics.

usage: python tools/ncu_summary.py OUT_PREFIX launches.csv rep1.ncu-rep [rep2 ...]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "time_ms": ("gpu__time_duration.sum", 1e-6),          # ns -> ms
    "dram_read_GB": ("dram__bytes_read.sum", None),
    "dram_write_GB": ("dram__bytes_write.sum", None),
    "dram_pct_peak": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "issue_active_pct": ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", 1),
    "fmaheavy_pct": ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", 1),
    "fp64_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "alu_pct": ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "xu_pct": ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "threads_per_inst": ("smsp__thread_inst_executed_per_inst_executed.ratio", 1),
    "warp_inst": ("smsp__inst_executed.sum", 1),
    "regs": ("launch__registers_per_thread", 1),
    "grid": ("launch__grid_size", 1),
    "block": ("launch__block_size", 1),
}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        m = {"kernel": d.get("Kernel Name", "")[:90]}
        for k, (name, scale) in KEYS.items():
            v = d.get(name)
            if v in (None, ""):
                continue
            v = float(v.replace(",", ""))
            unit = u.get(name, "")
            if k.endswith("_GB"):
                v = v / {"byte": 1e9, "Kbyte": 1e6, "Mbyte": 1e3, "Gbyte": 1}.get(unit, 1e9)
            elif k == "time_ms":
                v = v * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1,
                         "ms": 1, "second": 1e3, "s": 1e3}.get(unit, 1e-6)
            m[k] = round(v, 4)
        if "dram_read_GB" in m:
            m["traffic_GB"] = round(m["dram_read_GB"] + m.get("dram_write_GB", 0), 4)
        res.append(m)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    out = []
    for r in rows[hi + 1:]:
        v = float(r[vi].replace(",", ""))
        v = v * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1,
                 "ms": 1}.get(r[ui], 1e-6)
        out.append((r[ki], v))
    return out


def main():
    prefix, lcsv, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    kern = []
    for rep in reps:
        kern += raw(rep)
    ll = launches(lcsv)
    ours = [(k, t) for k, t in ll if "brng" in k]
    tot = sum(t for _, t in ours)
    md = ["# ncu summary (" + prefix + ")", "",
          "## Launch list (our kernels, one bench step incl. warm-up; cold-cache, serialised)", "",
          "| kernel | ms | share |", "|---|---|---|"]
    for k, t in ours:
        md.append(f"| `{k[:80]}` | {t:.4f} | {t / tot:.3%} |")
    # per kernel: launches, mean ms per launch, share of all our kernel time
    # (every step launches the same list, so this is also the share of a step)
    agg = {}
    for k, t in ours:
        n, s = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, s + t)
    md += ["", "## Per kernel (share of the step)", "",
           "| kernel | launches | mean ms | share |", "|---|---|---|---|"]
    for k, (n, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        md.append(f"| `{k[:80]}` | {n} | {s / n:.4f} | {s / tot:.2%} |")
    md += ["", "## Full captures", "", "| kernel | " + " | ".join(KEYS) + " | traffic_GB |",
           "|" + "---|" * (len(KEYS) + 2)]
    for m in kern:
        md.append(f"| `{m['kernel'][:60]}` | " + " | ".join(str(m.get(k, "")) for k in KEYS) +
                  f" | {m.get('traffic_GB', '')} |")
    open(prefix + ".md", "w").write("\n".join(md) + "\n")
    json.dump({"launches": ours, "kernels": kern}, open(prefix + ".json", "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
