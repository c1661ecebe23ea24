"""MCTS with GPU leaf evaluation (pe_search): identical plan to the same
search driven by the CPU oracle, Megatron recovery (SPEC acceptance 3 and 9),
and the 24-layer GPT-2-medium configuration."""
import os

import pytest

import helpers as H
from paper_2112_02958_b200 import capi, engine, modelgen, search
from test_search import TWO_LAYER, evaluator, megatron, setup

pytestmark = pytest.mark.gpu


def _engine(text, cfg, cp):
    return engine.Engine(engine.Graph(text), device=0, cfg=cfg, cost=cp)


def test_gpu_search_equals_oracle_search(oracle_lib):
    text = modelgen.build_transformer(**TWO_LAYER)
    g, cfg, cp, ords, lw = setup(text)
    eng = _engine(text, cfg, cp)
    gp = search.mcts_search(eng, episodes=256, seed=7, leaf_batch=32)
    op = search.run_mcts(evaluator("oracle", text, cfg, cp, lw), len(ords) - 1, ords,
                         episodes=256, seed=7, leaf_batch=32)
    assert search.plan_actions(gp) == search.plan_actions(op)
    assert gp.found_at_episode == op.found_at_episode
    assert not H.compare_results(gp.result, op.result)


def test_gpu_search_with_resurfacing_equals_oracle_search(oracle_lib):
    # worklist with stuck resurfacing (pe.h resurface_stuck)
    text = modelgen.build_transformer(**TWO_LAYER)
    g = engine.Graph(text)
    cfg = capi.default_search_config(group_scopes=1, resurface_stuck=1)
    cp = capi.default_cost_params()
    cp.memory_budget_bytes = int(0.6 * H.oracle_info(text, cfg)["baseline_bytes"])
    ords = search.ordinal_actions(g, cfg)
    lw = (len(ords) - 1 + 63) // 64
    eng = _engine(text, cfg, cp)
    assert eng.n_ordinals == len(ords) - 1
    assert [(eng.ordinal_action(o).value, eng.ordinal_action(o).kind) for o in range(len(ords) - 1)] \
        == [(a.value, a.kind) for a in ords[:-1]]
    gp = search.mcts_search(eng, episodes=192, seed=9, leaf_batch=32)
    op = search.run_mcts(evaluator("oracle", text, cfg, cp, lw), len(ords) - 1, ords,
                         episodes=192, seed=9, leaf_batch=32)
    assert search.plan_actions(gp) == search.plan_actions(op)
    assert not H.compare_results(gp.result, op.result)


def test_gpu_megatron_recovery_20_seeds():
    # SPEC acceptance 3: >= 80% of 20 seeds at budget 500; 9: 2-20 decisions
    text = modelgen.build_transformer(**TWO_LAYER)
    g, cfg, cp, ords, lw = setup(text)
    eng = _engine(text, cfg, cp)
    hits = 0
    for seed in range(20):
        p = search.mcts_search(eng, episodes=500, seed=seed, leaf_batch=64)
        if megatron(p.result, 2):
            hits += 1
            assert 2 <= p.n_actions <= 20
    assert hits >= 16


def test_gpu_emit_plan_roundtrip():
    text = modelgen.build_transformer(**TWO_LAYER)
    g, cfg, cp, ords, lw = setup(text)
    eng = _engine(text, cfg, cp)
    p = search.mcts_search(eng, episodes=300, seed=1, leaf_batch=64)
    import json
    d = json.loads(search.emit_plan(eng, p))
    assert d["args"]["l0_wq"]["dims"][1] == "model"  # column-parallel q_proj
    assert d["cost"]["ar_cnt"][0] == 4 and d["cost"]["ag_cnt"][0] == 0
    # replay (SPEC emit_plan example): same CostReport
    again = eng.eval_batch([[capi.PeAction(*a, 0) for a in search.plan_actions(p)]])[0]
    assert not H.compare_results(again, p.result)


def test_gpu_gpt2_medium_24_layer_megatron():
    # config 3: 24-layer GPT-2-medium on [batch=4, model=2], model axis searched,
    # the batch axis left manual
    text = modelgen.config_program(3)
    g0 = engine.Graph(text)
    cfg = capi.default_search_config(group_scopes=1, scoped_only=1,
                                     auto_axes_mask=1 << g0.axis_index("model"))
    cp = capi.default_cost_params()
    base = engine.Engine(g0, cfg=cfg).baseline_bytes
    cp.memory_budget_bytes = int(0.6 * base)
    eng = _engine(text, cfg, cp)
    p = search.mcts_search(eng, episodes=1024, seed=0, leaf_batch=256)
    model = g0.axis_index("model")
    assert p.result.ar_cnt[model] == 48 and p.result.ag_cnt[model] == 0, search.plan_actions(p)


def test_gpu_searched_plan_preserves_semantics(oracle_lib):
    text = modelgen.build_transformer(**TWO_LAYER)
    g, cfg, cp, ords, lw = setup(text)
    eng = _engine(text, cfg, cp)
    p = search.mcts_search(eng, episodes=500, seed=4, leaf_batch=64)
    ok, diff, _ = H.oracle_check_equivalence(text, search.plan_actions(p), trials=3)
    assert ok, diff


def test_config1_mlp_search_seeds_equal_the_reference_search(oracle_lib):
    # BASELINE.json configs[0] / SURVEY.md §8(d) config 1: the 2-layer MLP on
    # {model=8}, MCTS with the SPEC defaults (memory + comm cost model, budget
    # 500 episodes), seeds 0-19 on the GPU engine; the same searches driven by
    # the reference CPU path (oracle evaluator) return identical plans
    text = modelgen.config_program(1)
    g = engine.Graph(text)
    cfg = capi.default_search_config(group_scopes=0)
    cp = capi.default_cost_params()
    ords = search.ordinal_actions(g, cfg)
    lw = (len(ords) - 1 + 63) // 64
    eng = _engine(text, cfg, cp)
    plans = [search.mcts_search(eng, episodes=500, seed=s, leaf_batch=64) for s in range(20)]
    assert all(p.result.status == capi.PE_CAND_OK and p.episodes == 500 for p in plans)
    for s in range(0, 20, 5):
        op = search.run_mcts(evaluator("oracle", text, cfg, cp, lw), len(ords) - 1, ords,
                             episodes=500, seed=s, leaf_batch=64)
        assert search.plan_actions(plans[s]) == search.plan_actions(op)
        assert not H.compare_results(plans[s].result, op.result)
