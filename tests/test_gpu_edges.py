"""GPU edge cases through the C-ABI, against the oracle: empty batches,
batches that are not a multiple of a warp, ragged prefixes (empty, Stop
mid-prefix, an illegal action mid-prefix, prefixes longer than
max_decisions) and a max_decisions small enough to truncate the action
output.  Bit-exact on every integer field, legal bitmasks and action lists."""
import os

import pytest

import helpers as H
from paper_2112_02958_b200 import capi, engine, modelgen

pytestmark = pytest.mark.gpu

NTHR = os.cpu_count() or 1


def test_empty_batches():
    eng = engine.Engine(engine.Graph(modelgen.linear()), device=0)
    assert eng.eval_batch([]) == []
    res, tr = eng.eval_batch([], trace_words=64)
    assert res == [] and tr == []
    res, seqs, legal = eng.rollout_batch([], [], legal=True)
    assert res == [] and seqs == []


@pytest.mark.parametrize("maxd", [1, 2, 32])
def test_ragged_prefixes_odd_batch(oracle_lib, maxd):
    text = modelgen.config_program(2)
    cfg = capi.default_search_config(group_scopes=1, max_decisions=maxd)
    eng = engine.Engine(engine.Graph(text), device=0, cfg=cfg)
    # root rollouts give legal decision sequences to cut prefixes from
    roots, seqs, _ = eng.rollout_batch([[]] * 64, list(range(64)))
    stop = (0, 0, 0, capi.PE_ACT_STOP)
    prefixes = [[]]
    for s in seqs:
        if not s:
            continue
        prefixes.append(s[:1])
        prefixes.append(s)
        prefixes.append(s[:1] + [stop] + s[1:])  # Stop ends the rollout there
        prefixes.append(s[:1] + s[:1])           # the same tile twice: illegal
        prefixes.append(s * 3)                   # longer than max_decisions
    prefixes = prefixes[:37]                     # not a multiple of 32
    assert len(prefixes) == 37
    seeds = [1000 + i for i in range(len(prefixes))]
    res, out, legal = eng.rollout_batch(prefixes, seeds, legal=True)
    ref, rout, rlegal = H.rollout_batch("oracle", text, prefixes, seeds, cfg,
                                        legal_words=eng.legal_words, threads=NTHR)
    assert out == rout
    assert legal == rlegal
    diffs = [(i, H.compare_results(a, b)) for i, (a, b) in enumerate(zip(res, ref))]
    assert not [d for d in diffs if d[1]], diffs[:3]
    assert all(len(o) <= maxd for o in out)
    # the illegal prefixes report ILLEGAL with the failing step, like the oracle
    assert any(r.status == capi.PE_CAND_ILLEGAL for r in res)
