#!/usr/bin/env python
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list into per-kernel shares.

usage: python scripts/ncu_launches.py gpurun_out/launches.csv [out.md]
(ncu per-launch times are cold-cache and serialised: compare SHARES, not absolutes.)"""
import collections
import csv
import re
import sys


def kname(full: str) -> str:
    s = full
    s = re.sub(r"^void\s+", "", s)
    s = s.split("(", 1)[0] if not s.startswith("kz::(anonymous") else s
    s = s.replace("kz::(anonymous namespace)::", "")
    s = re.sub(r"\(.*$", "", s)
    return s.strip()


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= mi or not r[mi]:
            continue
        v = float(r[mi].replace(",", ""))
        v *= {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(r[ui], 1)
        n = kname(r[ki])
        agg[n][0] += 1
        agg[n][1] += v
    tot = sum(v[1] for v in agg.values())
    lines = ["| kernel | launches | total ms | share | avg us |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {v[0]} | {v[1] / 1e6:.3f} | {100 * v[1] / tot:.1f}% | {v[1] / v[0] / 1e3:.1f} |")
    out = "\n".join(lines)
    print(out)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(out + "\n")


if __name__ == "__main__":
    main()
