#!/usr/bin/env python3
"""Workload for compute-sanitizer (memcheck / synccheck / racecheck): every
kernel of the engine on small graphs -- scheduled and unscheduled root
rollouts (config 2; one batch beyond the resident slots so the SM-wide
blocks and the warp-chunked second wave run), prefix rollouts with legal
sets, the forced-overflow retry path, traced evaluations of random
programs, InferRest pauses/resumes, the prefix-state cache and pe_state
handles.  Exits non-zero if any result differs from the oracle sample it
checks (so a sanitizer run also proves the instrumented kernels computed the
same answers)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import fuzz_util as F  # noqa: E402
import helpers as H  # noqa: E402
from paper_2112_02958_b200 import capi, engine, modelgen  # noqa: E402

big = int(sys.argv[1]) if len(sys.argv) > 1 else 0
text = modelgen.config_program(2)
cfg = capi.default_search_config(group_scopes=1)
eng = engine.Engine(engine.Graph(text), device=0, cfg=cfg)
n = 2 * eng.slots() + 37 if big else 8192
seeds = np.arange(n, dtype=np.uint64) + np.uint64(5)
r, a, na = eng.rollout_roots_np(seeds)            # scheduled (trie) launch
print("root rollouts", n, "ok", flush=True)
res, seqs, legal = eng.rollout_batch([[]] * 256, list(range(256)), legal=True)
ref, rseqs, rlegal = H.rollout_batch("oracle", text, [[]] * 256, list(range(256)), cfg,
                                     legal_words=eng.legal_words, threads=os.cpu_count() or 1)
assert seqs == rseqs and legal == rlegal
assert all(not H.compare_results(x, y) for x, y in zip(res, ref))
pre = [s[:k] for s in seqs[:32] for k in range(1, len(s) + 1)]
eng.rollout_batch(pre, list(range(len(pre))), legal=True)
print("prefix rollouts ok", flush=True)
if not big:
    for i in range(4):
        mesh = F.MESHES[i % 3]
        t = modelgen.random_program(9100 + i, mesh)
        e2 = engine.Engine(engine.Graph(t), device=0)
        sq = F.legal_sequences(t, mesh, 77 + i, n_seqs=6)
        rr, tr = e2.eval_batch(sq, trace_words=16384)
        rf, rtr = H.eval_batch("oracle", t, sq, trace_words=16384)
        assert all(not H.compare_results(x, y) for x, y in zip(rr, rf))
        assert all(x[:x[0]] == y[:y[0]] for x, y in zip(tr, rtr))
    print("traced eval fuzz ok", flush=True)
    ci = capi.default_search_config(group_scopes=1, infer_rest_action=1)
    e3 = engine.Engine(engine.Graph(text), device=0, cfg=ci)
    r3, s3, _ = e3.rollout_batch([[]] * 512, list(range(512)))
    f3, fs3, _ = H.rollout_batch("oracle", text, [[]] * 512, list(range(512)), ci,
                                 threads=os.cpu_count() or 1)
    assert s3 == fs3 and all(not H.compare_results(x, y) for x, y in zip(r3, f3))
    print("infer-rest rollouts ok", flush=True)
    e4 = engine.Engine(engine.Graph(text), device=0, cfg=cfg)
    e4.set_prefix_cache(0.25)
    for d in (1, 2, 3):
        pp = [s[:d] for s in seqs if len(s) >= d]
        e4.rollout_batch(pp, list(range(len(pp))), legal=True)
    st = e4.state(seqs[0][:1]) if seqs[0] else None
    if st is not None:
        e4.eval_from_states([st, None], [[seqs[1][0]] if seqs[1] else [], []])
    print("prefix cache / states ok", e4.prefix_cache_stats(), flush=True)
    os.environ["PE_DEBUG_TIGHT_EM_CAP"] = "8"
    e5 = engine.Engine(engine.Graph(text), device=0, cfg=cfg)
    e5.rollout_batch([[]] * 128, list(range(128)))
    print("retry path ok", flush=True)
print("SANITIZE WORKLOAD DONE")
