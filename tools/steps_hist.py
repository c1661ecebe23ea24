"""Histogram of decisions per rollout (config 3 by default): how many
rollouts end within the scheduling trie's depth.  python tools/steps_hist.py"""
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2112_02958_b200 import capi, engine, modelgen  # noqa: E402

cfgno = int(os.environ.get("CFG", "3"))
n = int(os.environ.get("N", "20000"))
eng = engine.Engine(engine.Graph(modelgen.config_program(cfgno)),
                    cfg=capi.default_search_config(group_scopes=1))
res, seqs, _ = eng.rollout_batch([[]] * n, list(range(n)))
h = collections.Counter(r.n_steps for r in res)
acc = 0
for k in sorted(h):
    acc += h[k]
    print(f"{k:3d} decisions: {h[k] / n:6.1%}  (<= {k}: {acc / n:6.1%})")
