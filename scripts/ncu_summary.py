#!/usr/bin/env python
"""Key metrics of `ncu --set full` reports: python scripts/ncu_summary.py rep1.ncu-rep [...] [--json out.json]"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__block_size", "block"),
    ("launch__grid_size", "grid"),
    ("smsp__inst_executed.sum", "warp_inst"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
    ("l1tex__t_sector_hit_rate.pct", "l1_hit_pct"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1_pct"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pct"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu_pct"),
]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3,
        "ns": 1e-3, "us": 1, "ms": 1e3, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def summarise(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u = rows[0], rows[1]
    out = []
    for v in rows[2:]:
        d = {"kernel": v[h.index("Kernel Name")][:90]}
        for key, short in KEYS:
            if key in h:
                i = h.index(key)
                try:
                    x = float(v[i].replace(",", ""))
                except ValueError:
                    continue
                d[short] = x * UNIT.get(u[i], 1) if short in ("time", "dram_read", "dram_write", "l2_bytes") else x
        out.append(d)
    return out


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    res = {}
    jpath = sys.argv[sys.argv.index("--json") + 1] if "--json" in sys.argv else None
    for rep in args:
        if rep == jpath:
            continue
        for d in summarise(rep):
            res[rep] = d
            print(f"== {rep}: {d['kernel']}")
            for k, v in d.items():
                if k != "kernel":
                    print(f"   {k:16s} {v:,.3f}")
    if jpath:
        json.dump(res, open(jpath, "w"), indent=1)
