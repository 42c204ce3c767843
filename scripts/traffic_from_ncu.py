#!/usr/bin/env python
"""Record one kernel's DRAM traffic from an ncu `--page raw --csv` export into
profiles/traffic.json (bench.py reports it as roofline.traffic).

  python scripts/traffic_from_ncu.py KEY RAW.csv UPDATES_PER_LAUNCH BYTES_PER_UPDATE [NOTE]
"""
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main():
    key, raw, n, bpu = sys.argv[1], Path(sys.argv[2]).resolve(), int(sys.argv[3]), int(sys.argv[4])
    note = sys.argv[5] if len(sys.argv) > 5 else ""
    rows = list(csv.reader(raw.open()))
    head = next(i for i, r in enumerate(rows) if "dram__bytes_read.sum" in r)
    h, units, vals = rows[head], rows[head + 1], rows[head + 2]
    d, u = dict(zip(h, vals)), dict(zip(h, units))
    rd = float(d["dram__bytes_read.sum"].replace(",", "")) * SCALE[u["dram__bytes_read.sum"]]
    wr = float(d["dram__bytes_write.sum"].replace(",", "")) * SCALE[u["dram__bytes_write.sum"]]
    p = ROOT / "profiles" / "traffic.json"
    table = json.loads(p.read_text()) if p.exists() else {}
    table[key] = {"source": f"{raw.relative_to(ROOT)} (ncu --set full, 1 launch){' ' + note if note else ''}",
                  "kernel": d.get("Kernel Name", "")[:80],
                  "dram_bytes_read": int(rd), "dram_bytes_write": int(wr),
                  "dram_bytes_per_launch": int(rd + wr), "updates_per_launch": n,
                  "algorithmic_bytes_per_launch": n * bpu}
    p.write_text(json.dumps(table, indent=2) + "\n")
    print(json.dumps(table[key], indent=1))


if __name__ == "__main__":
    main()
