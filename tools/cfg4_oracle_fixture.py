#!/usr/bin/env python3
"""Generates tests/golden/cfg4_oracle.json: the reference CPU path
(oracle/_ref: patched reference + SPEC cost restatement) on single-decision
candidates of config 4 (52,154 ops).  One candidate takes 30-60 minutes of
one core here, so the fixture holds a handful; the GPU test compares the
engine with them bit-exactly.  TEST INFRASTRUCTURE.

  python tools/cfg4_oracle_fixture.py NAME      (appends one candidate)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import helpers as H  # noqa: E402
from paper_2112_02958_b200 import capi, engine, modelgen  # noqa: E402

CANDS = {"w2": ("l47_w2", 0, "model", False), "x0": ("x0", 0, "batch", False),
         "qgrp": ("l0_wq", 1, "model", True), "g1grp": ("l23_g1", 0, "batch", True),
         "w1_47": ("l47_w1", 1, "model", False), "w2_45": ("l45_w2", 0, "model", False),
         "wo_47": ("l47_wo", 0, "model", False), "g2_47": ("l47_g2", 0, "model", False)}
OUT = os.path.join(ROOT, "tests", "golden", "cfg4_oracle.json")


def main():
    name = sys.argv[1]
    text = modelgen.config_program(4)
    g = engine.Graph(text)
    cfg = capi.default_search_config(group_scopes=1)
    v, d, ax, grp = CANDS[name]
    a = g.action(v, d, ax, group=grp)
    seq = [(a.value, a.dim, a.axis, a.kind)]
    t0 = time.time()
    r, _ = H.eval_batch("oracle", text, [seq], cfg=cfg)
    rec = {"name": name, "seq": seq, "oracle_seconds": time.time() - t0,
           "result": capi.result_dict(r[0])}
    if os.environ.get("FIXTURE_PART_DIR"):  # concurrent runs: one file each, merged later
        json.dump(rec, open(os.path.join(os.environ["FIXTURE_PART_DIR"], name + ".json"), "w"))
    else:
        data = json.load(open(OUT)) if os.path.exists(OUT) else {"graph": "config 4", "cands": []}
        data["cands"] = [c for c in data["cands"] if c["name"] != name] + [rec]
        json.dump(data, open(OUT, "w"), indent=1)
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
