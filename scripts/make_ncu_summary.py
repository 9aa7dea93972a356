#!/usr/bin/env python
"""profiles/ncu_summary.json from one round's `ncu --set full` captures (scripts/profile_round.sh): per kaze
profile class (kaze_get_profile names), DRAM bytes per launch = dram__bytes_read.sum + dram__bytes_write.sum of
the captured launch (32 images of 1920x1200 per launch, bench launch configuration; ncu flushes caches between
replays, so this is cold-cache traffic).  'hessian' is one kaze launch unit = the mean of hess_first and hess_det
(kaze_get_profile counts the pair as two launches).  bench.py reads it for roofline.traffic.

usage: python scripts/make_ncu_summary.py <dir with prof_*.ncu-rep> <round tag>"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import summarise  # noqa: E402

MAP = {"cols": "aos_cols", "rows": "aos_rows", "cond": "cond", "nms": "nms_mark", "desc": "describe",
       "emit": "kp_emit", "pre": "prefilter", "khist": "k_hist", "hfused": "hessian"}


def main():
    d, tag = sys.argv[1], sys.argv[2]
    res, raw = {}, {}
    for f in sorted(os.listdir(d)):
        if not (f.startswith("prof_") and f.endswith(".ncu-rep")):
            continue
        t = f[5:-8]
        rows = summarise(os.path.join(d, f))
        if not rows:
            continue
        r = rows[0]
        raw[t] = r
        if t in MAP:
            res[MAP[t]] = {"dram_bytes_per_launch": r["dram_read"] + r["dram_write"], "time_us": r["time"],
                           "dram_read": r["dram_read"], "dram_write": r["dram_write"], "kernel": r["kernel"]}
    if "hessian" not in res and "hfirst" in raw and "hdet" in raw:  # two-pass form
        a, b = raw["hfirst"], raw["hdet"]
        res["hessian"] = {"dram_bytes_per_launch": 0.5 * (a["dram_read"] + a["dram_write"] + b["dram_read"] + b["dram_write"]),
                          "time_us": 0.5 * (a["time"] + b["time"]),
                          "note": "mean of hess_first and hess_det (16 levels x 8 images each)"}
    out = {"about": "ncu --set full --clock-control none, one launch per kernel (32 images of 1920x1200 per launch, "
                    "cold cache between replays); dram_bytes_per_launch = dram__bytes_read.sum + "
                    f"dram__bytes_write.sum. Source: profiles/{tag}/ncu_full_summary.txt", "kernels": res}
    json.dump(out, open("profiles/ncu_summary.json", "w"), indent=1)
    os.makedirs(f"profiles/{tag}", exist_ok=True)
    json.dump(raw, open(f"profiles/{tag}/ncu_full_raw.json", "w"), indent=1)
    with open(f"profiles/{tag}/ncu_full_summary.txt", "w") as fh:
        for t, r in raw.items():
            fh.write(f"== {t}: {r['kernel']}\n")
            for k, v in r.items():
                if k != "kernel":
                    fh.write(f"   {k:16s} {v:,.3f}\n")


if __name__ == "__main__":
    main()
