#!/usr/bin/env python3
"""Merges per-candidate fixture files (FIXTURE_PART_DIR runs of
tools/cfg4_oracle_fixture.py) into tests/golden/cfg4_oracle.json."""
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tests", "golden", "cfg4_oracle.json")
data = json.load(open(OUT)) if os.path.exists(OUT) else {"graph": "config 4", "cands": []}
for f in glob.glob(os.path.join(sys.argv[1], "*.json")):
    rec = json.load(open(f))
    data["cands"] = [c for c in data["cands"] if c["name"] != rec["name"]] + [rec]
json.dump(data, open(OUT, "w"), indent=1)
print([c["name"] for c in data["cands"]])
