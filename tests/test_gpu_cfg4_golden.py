"""Config 4 (52,154 ops) against the reference itself: single-decision
candidates the reference CPU path evaluated offline (30-60 minutes each on
one core; tools/cfg4_oracle_fixture.py -> tests/golden/cfg4_oracle.json).
The engine must reproduce every recorded field exactly."""
import json
import os

import pytest

from paper_2112_02958_b200 import capi, engine, modelgen

pytestmark = pytest.mark.gpu
FIX = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cfg4_oracle.json")


def test_config4_single_decisions_equal_the_reference():
    data = json.load(open(FIX))
    assert data["cands"]
    text = modelgen.config_program(4)
    eng = engine.Engine(engine.Graph(text), device=0, cfg=capi.default_search_config(group_scopes=1))
    res = eng.eval_batch([[tuple(a) for a in c["seq"]] for c in data["cands"]])
    for c, r in zip(data["cands"], res):
        got = capi.result_dict(r)
        for k, v in c["result"].items():
            if k in ("runtime_s", "reward"):
                assert abs(got[k] - v) <= 1e-6 * max(abs(v), 1e-300), (c["name"], k)
            else:
                assert got[k] == v, (c["name"], k, got[k], v)
