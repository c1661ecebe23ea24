"""Stuck resurfacing in the worklist (pe.h
`resurface_stuck`; SPEC Worklist "plus stuck nodes resurfaced by
propagation", "deterministic order (argument order, then stuck discovery
order)"): after every decision the ops of the fixpoint's stuck list
(REF propagate.cc:412-454) join the worklist as TileValue(op result)
entries.  The host-compiled core must enumerate the same legal actions in
the same order as the oracle, so that rollouts pick identical actions,
including from MCTS prefixes that end on resurfaced actions."""
import helpers as H
import fuzz_util as F
from paper_2112_02958_b200 import capi, engine, modelgen, search


def _cfg(group):
    return capi.default_search_config(group_scopes=group, resurface_stuck=1)


def _n_args(text):
    return text.split("->")[0].count("%")


def _resurfaced(seq, n_args):
    return sum(1 for a in seq if a[3] == capi.PE_ACT_TILE and a[0] >= n_args)


def test_ordinals_extend_by_one_block_per_op(oracle_lib):
    text = modelgen.config_program(2)
    g = engine.Graph(text)
    for group in (0, 1):
        cfg = _cfg(group)
        ords = search.ordinal_actions(g, cfg)
        assert len(ords) - 1 == H.oracle_info(text, cfg)["n_ordinals"]
        static = H.oracle_info(text, capi.default_search_config(group_scopes=group))
        first_op = ords[static["n_ordinals"]]
        assert first_op.kind == capi.PE_ACT_TILE and first_op.value == g.n_args
        assert ords[-1].kind == capi.PE_ACT_STOP


def test_resurfacing_rollouts_match_oracle(oracle_lib, harness_lib):
    picked = 0
    for cfgno, group in ((1, 1), (2, 1), (2, 0)):
        text = modelgen.config_program(cfgno)
        cfg = _cfg(group)
        lw = (H.oracle_info(text, cfg)["n_ordinals"] + 63) // 64
        seeds = list(range(200))
        ro, so, lo = H.rollout_batch("oracle", text, [[]] * 200, seeds, cfg, legal_words=lw)
        rh, sh, lh = H.rollout_batch("harness", text, [[]] * 200, seeds, cfg, legal_words=lw)
        assert so == sh and lo == lh
        assert all(not H.compare_results(a, b) for a, b in zip(ro, rh))
        picked += sum(_resurfaced(s, _n_args(text)) for s in so)
    for i in range(120):
        mesh = F.MESHES[i % 3]
        text = modelgen.random_program(50000 + i, mesh)
        cfg = _cfg(0)
        lw = (H.oracle_info(text, cfg)["n_ordinals"] + 63) // 64
        ro, so, lo = H.rollout_batch("oracle", text, [[]] * 12, list(range(12)), cfg, legal_words=lw)
        rh, sh, lh = H.rollout_batch("harness", text, [[]] * 12, list(range(12)), cfg, legal_words=lw)
        assert so == sh and lo == lh
        assert all(not H.compare_results(a, b) for a, b in zip(ro, rh))
        picked += sum(_resurfaced(s, _n_args(text)) for s in so)
    assert picked > 200  # resurfaced entries are actually taken


def test_resurfacing_prefixes_match_oracle(oracle_lib, harness_lib):
    # prefixes ending on / containing resurfaced actions: the worklist must
    # depend only on the action sequence, not on where the prefix ends
    n_with = 0
    for i in range(60):
        mesh = F.MESHES[i % 3]
        text = modelgen.random_program(61000 + i, mesh)
        cfg = _cfg(0)
        lw = (H.oracle_info(text, cfg)["n_ordinals"] + 63) // 64
        _, seqs, _ = H.rollout_batch("oracle", text, [[]] * 8, list(range(8)), cfg, legal_words=lw)
        prefixes = [s[:k] for s in seqs for k in range(1, len(s) + 1)]
        if not prefixes:
            continue
        n_with += sum(1 for p in prefixes if _resurfaced(p, _n_args(text)))
        seeds = [900 + k for k in range(len(prefixes))]
        ro, so, lo = H.rollout_batch("oracle", text, prefixes, seeds, cfg, legal_words=lw)
        rh, sh, lh = H.rollout_batch("harness", text, prefixes, seeds, cfg, legal_words=lw)
        assert so == sh and lo == lh
        assert all(not H.compare_results(a, b) for a, b in zip(ro, rh))
        for p in prefixes[:3]:  # oracle's ordered legal list agrees with the bitmask
            legal = H.oracle_legal(text, p, cfg)
            _, _, lp = H.rollout_batch("harness", text, [p], [0], cfg, legal_words=lw)
            assert sorted(legal) == [o for o in range(lw * 64) if (lp[0][o // 64] >> (o % 64)) & 1]
    assert n_with > 20


def test_search_with_resurfacing_oracle_vs_core(oracle_lib, harness_lib):
    text = modelgen.build_transformer(2, mesh=(("model", 2),), **modelgen.TOY)
    g = engine.Graph(text)
    cfg = _cfg(1)
    cp = capi.default_cost_params()
    cp.memory_budget_bytes = int(0.6 * H.oracle_info(text, cfg)["baseline_bytes"])
    ords = search.ordinal_actions(g, cfg)
    lw = (len(ords) - 1 + 63) // 64
    plans = {}
    for which in ("oracle", "harness"):
        def ev(prefixes, seeds, which=which):
            return H.rollout_batch(which, text, prefixes, seeds, cfg, cp=cp, legal_words=lw)
        p = search.run_mcts(ev, len(ords) - 1, ords, episodes=120, seed=5, leaf_batch=16)
        plans[which] = (search.plan_actions(p), p.found_at_episode, p.result.reward)
    assert plans["oracle"] == plans["harness"]
