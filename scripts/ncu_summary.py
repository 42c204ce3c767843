#!/usr/bin/env python
"""Summarise one `ncu --set full` capture (its --page raw --csv export) into
profiles/<round>/ncu_summary.json under a key, for bench.py's roofline
fields (DRAM traffic, on-chip binding unit) — so every number the bench line
quotes from ncu is reproducible from a committed file.

    python scripts/ncu_summary.py RAW_CSV KEY OUT_JSON [--compulsory BYTES]
"""

import csv
import json
import sys
from pathlib import Path

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1tex_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "lts_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "launch__registers_per_thread": "registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__inst_executed.sum": "instructions",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "smsp__warps_eligible.avg.per_cycle_active": "eligible_warps",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9,
         "us": 1e-6, "ms": 1e-3, "s": 1.0,
         "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}


def summarise(raw_csv: str) -> dict:
    rows = list(csv.reader(open(raw_csv)))
    head, units, vals = rows[0], rows[1], rows[2]
    out = {"kernel": vals[head.index("Kernel Name")].split("(")[0].strip()}
    for metric, key in METRICS.items():
        if metric not in head:
            continue
        i = head.index(metric)
        v = float(vals[i].replace(",", ""))
        u = units[i]
        if u in SCALE:
            v *= SCALE[u]
        out[key] = v
    out["dram_bytes"] = out.get("dram_read", 0.0) + out.get("dram_write", 0.0)
    out["dram_gbs"] = out["dram_bytes"] / out["duration"] / 1e9
    return out


def main():
    raw, key, dst = sys.argv[1:4]
    s = summarise(raw)
    if "--compulsory" in sys.argv:
        c = float(sys.argv[sys.argv.index("--compulsory") + 1])
        s["compulsory_bytes"] = c
        s["dram_over_compulsory"] = s["dram_bytes"] / c
    s["source"] = str(Path(raw).as_posix())
    p = Path(dst)
    data = json.loads(p.read_text()) if p.exists() else {}
    data[key] = s
    p.write_text(json.dumps(data, indent=1, sort_keys=True) + "\n")
    print(json.dumps(s, indent=1))


if __name__ == "__main__":
    main()
