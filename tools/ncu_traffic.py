#!/usr/bin/env python3
"""Extracts the per-launch DRAM traffic of the main rollout kernel from an
`ncu --set full` report (exported with `ncu -i REP --page raw --csv`) into
profiles/r2_traffic.json, which bench.py reports as roofline.traffic.

  python tools/ncu_traffic.py raw.csv CANDIDATES_PER_LAUNCH "source text"
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
units = rows[1]
data = [r for r in rows[2:] if any("pe_rollout_kernel" in c for c in r)]
assert data, "no pe_rollout_kernel row"
col = {h: i for i, h in enumerate(hdr)}
# the main launch: the longest captured pe_rollout_kernel (retries are short)
r = max(data, key=lambda x: float(x[col["gpu__time_duration.sum"]].replace(",", "")))


def val(name):
    x = float(r[col[name]].replace(",", ""))
    u = units[col[name]].lower()
    return x * {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "tbyte": 1e12}.get(u, 1)


out = {"source": sys.argv[3], "candidates": int(sys.argv[2]),
       "dram_bytes_read": val("dram__bytes_read.sum"), "dram_bytes_write": val("dram__bytes_write.sum"),
       "lts_t_bytes": val("lts__t_bytes.sum") if "lts__t_bytes.sum" in col else None,
       "duration_ms": float(r[col["gpu__time_duration.sum"]].replace(",", "")) *
       {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1, "second": 1e3}.get(units[col["gpu__time_duration.sum"]].lower(), 1)}
out["bytes_per_candidate"] = (out["dram_bytes_read"] + out["dram_bytes_write"]) / out["candidates"]
json.dump(out, open(os.path.join(ROOT, "profiles", "r2_traffic.json"), "w"), indent=1)
print(json.dumps(out))
