"""Dynamic instruction and stall-sample breakdown of one kernel from an
`ncu --set full --import-source on` capture (SASS source page).

usage: python tools/ncu_src_breakdown.py REP.ncu-rep N_UNITS [--lines K]

Prints warp-level instructions executed per unit (x32 / N_UNITS: thread-slot
equivalents at full warps), by opcode, with the stall samples on each opcode,
and optionally the K hottest SASS lines.
"""
import argparse
import collections
import csv
import io
import re
import subprocess


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         check=True, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ix = {k: hdr.index(k) for k in ("Address", "Source", "Instructions Executed",
                                    "Warp Stall Sampling (All Samples)",
                                    "Thread Instructions Executed")}
    res = []
    for r in rows[2:]:
        try:
            n = int(r[ix["Instructions Executed"]])
        except (ValueError, IndexError):
            continue
        res.append(dict(addr=r[ix["Address"]], src=r[ix["Source"]].strip(), n=n,
                        th=int(r[ix["Thread Instructions Executed"]] or 0),
                        stall=int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)))
    return res


def opcode(src):
    s = re.sub(r"^@!?U?P\w+\s+", "", src)
    op = s.split()[0] if s else "?"
    for pre in ("IMAD.WIDE", "IMAD.HI", "IMAD.MOV", "IMAD.IADD", "IMAD.SHL", "IMAD.X"):
        if op.startswith(pre):
            return pre
    return op.split(".")[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("units", type=float)
    ap.add_argument("--lines", type=int, default=0)
    a = ap.parse_args()
    rows = load(a.rep)
    tot = sum(r["n"] for r in rows)
    st = sum(r["stall"] for r in rows)
    th = sum(r["th"] for r in rows)
    print(f"warp instructions {tot}, per unit x32: {tot * 32 / a.units:.1f}, "
          f"avg active threads {th / max(tot, 1):.2f}, stall samples {st}")
    by, sb = collections.Counter(), collections.Counter()
    for r in rows:
        by[opcode(r["src"])] += r["n"]
        sb[opcode(r["src"])] += r["stall"]
    for k, v in by.most_common(40):
        print(f"  {k:12s} {v * 32 / a.units:8.2f}/unit  stall {100 * sb[k] / max(st, 1):5.1f}%")
    if a.lines:
        hot = sorted(range(len(rows)), key=lambda i: -rows[i]["stall"])[:a.lines]
        print("hottest lines by stall samples:")
        for i in sorted(hot):
            r = rows[i]
            print(f"  {i:5d} {r['n'] * 32 / a.units:6.2f}/unit stall {r['stall']:6d}  {r['src'][:80]}")


if __name__ == "__main__":
    main()
