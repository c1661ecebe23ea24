"""InferRest as a legal rollout / MCTS action (pe.h infer_rest_action; SPEC
legal_actions "plus InferRest (if any argument untiled)", apply_action
"InferRest -> infer_rest"), evaluated on the device:
rollouts that draw it pause, every paused candidate's (argument x dim x axis)
trials run as one batched evaluation per inference round, and the rollouts
resume with their RNG streams advanced.  The oracle applies the reference's
own infer_rest (REF propagate.cc:484-544).  Bit-exact: action sequences,
legal bitmasks (InferRest's bit included) and every integer result field."""
import os

import pytest

import fuzz_util as F
import helpers as H
from paper_2112_02958_b200 import capi, engine, modelgen, search
from test_search import TWO_LAYER, evaluator

pytestmark = pytest.mark.gpu

NTHR = os.cpu_count() or 1
PROGRAMS = {
    "mlp3": lambda: modelgen.build_mlp(3, (16, 64, 64, 16), 8, (("model", 2),)),
    "t1": lambda: modelgen.config_program(2),
    "t2": lambda: modelgen.build_transformer(2, mesh=(("model", 2),), **modelgen.TOY),
    "t2x2": lambda: modelgen.build_transformer(2, mesh=(("batch", 2), ("model", 2)), **modelgen.TOY),
    "rand": lambda: modelgen.random_program(4321, F.MESHES[1]),
}


def _count_ir(seqs):
    return sum(1 for s in seqs for a in s if a[3] == capi.PE_ACT_INFER_REST)


@pytest.mark.parametrize("name", sorted(PROGRAMS))
@pytest.mark.parametrize("group", [0, 1])
def test_rollouts_with_infer_rest_device_vs_oracle(oracle_lib, name, group):
    text = PROGRAMS[name]()
    cfg = capi.default_search_config(group_scopes=group, infer_rest_action=1)
    eng = engine.Engine(engine.Graph(text), device=0, cfg=cfg)
    assert eng.n_ordinals == H.oracle_info(text, cfg)["n_ordinals"]
    assert eng.ordinal_action(eng.n_ordinals - 1).kind == capi.PE_ACT_INFER_REST
    n = 384
    seeds = [1000 + i for i in range(n)]
    res, seqs, legal = eng.rollout_batch([[]] * n, seeds, legal=True)
    ref, rseqs, rlegal = H.rollout_batch("oracle", text, [[]] * n, seeds, cfg,
                                         legal_words=eng.legal_words, threads=NTHR)
    assert seqs == rseqs
    assert legal == rlegal
    bad = [i for i, (a, b) in enumerate(zip(res, ref)) if H.compare_results(a, b)]
    assert not bad, (bad[:4], H.compare_results(res[bad[0]], ref[bad[0]]) if bad else None)
    assert _count_ir(seqs) > 20  # the batch really exercised InferRest
    # prefixes that end on / contain an (unexpanded) InferRest decision:
    # paused inside the prefix, expanded, resumed
    prefixes = [s[:k] for s in seqs if _count_ir([s]) for k in range(1, len(s) + 1)][:256]
    ps = [77 + k for k in range(len(prefixes))]
    res2, seqs2, legal2 = eng.rollout_batch(prefixes, ps, legal=True)
    ref2, rseqs2, rlegal2 = H.rollout_batch("oracle", text, prefixes, ps, cfg,
                                            legal_words=eng.legal_words, threads=NTHR)
    assert seqs2 == rseqs2 and legal2 == rlegal2
    assert all(not H.compare_results(a, b) for a, b in zip(res2, ref2))
    # replay of the recorded decisions (pe_eval_batch expands every InferRest
    # in batched rounds) equals the rollout's own result
    ev = eng.eval_batch(seqs[:128])
    assert all(not H.compare_results(a, b) for a, b in zip(ev, res[:128]))


def test_large_batch_with_infer_rest(oracle_lib):
    # a batch beyond one wave of pauses: thousands of paused candidates
    # expanded together, resumed, some pausing again
    text = PROGRAMS["t2"]()
    cfg = capi.default_search_config(group_scopes=1, infer_rest_action=1)
    eng = engine.Engine(engine.Graph(text), device=0, cfg=cfg)
    n = 16384
    seeds = [5_000_000 + i for i in range(n)]
    res, seqs, _ = eng.rollout_batch([[]] * n, seeds)
    assert all(r.status == capi.PE_CAND_OK for r in res)
    assert sum(1 for s in seqs if _count_ir([s]) >= 2) > 50  # repeated pauses
    idx = list(range(0, n, 64))
    ref, rseqs, _ = H.rollout_batch("oracle", text, [[]] * len(idx), [seeds[i] for i in idx], cfg,
                                    threads=NTHR)
    assert [seqs[i] for i in idx] == rseqs
    assert all(not H.compare_results(res[i], r) for i, r in zip(idx, ref))


def test_eval_batch_expands_infer_rest_decisions_in_batches(oracle_lib):
    # unexpanded InferRest anywhere in explicit sequences, several per
    # sequence, behind illegal actions too; fail_step names the caller's index
    text = PROGRAMS["t2x2"]()
    eng = engine.Engine(engine.Graph(text), device=0,
                        cfg=capi.default_search_config(group_scopes=0))
    g = eng.graph
    IR = (0, 0, 0, capi.PE_ACT_INFER_REST)
    seqs = []
    for a in range(g.n_args):
        for d in range(len(g.shapes[a])):
            for ax in range(g.n_axes):
                if g.shapes[a][d] % g.axis_sizes[ax] == 0:
                    seqs.append([(a, d, ax, 0), IR])
                    seqs.append([IR, (a, d, ax, 0), IR])
    seqs.append([(0, 0, 0, 0), IR, (0, 0, 0, 0), IR])  # illegal second tile of x
    res, tr = eng.eval_batch(seqs, trace_words=16384)
    ref, rtr = H.eval_batch("oracle", text, seqs, trace_words=16384, threads=NTHR)
    for a, b, x, y in zip(res, ref, tr, rtr):
        assert not H.compare_results(a, b)
        assert x[:x[0]] == y[:y[0]]
    assert res[-1].status == capi.PE_CAND_ILLEGAL and res[-1].fail_step == 2


def test_search_with_infer_rest_equals_oracle_search(oracle_lib):
    text = modelgen.build_transformer(**TWO_LAYER)
    g = engine.Graph(text)
    cfg = capi.default_search_config(group_scopes=1, scoped_only=1, infer_rest_action=1)
    cp = capi.default_cost_params()
    cp.memory_budget_bytes = int(0.6 * H.oracle_info(text, cfg)["baseline_bytes"])
    ords = search.ordinal_actions(g, cfg)
    lw = (len(ords) - 1 + 63) // 64
    eng = engine.Engine(g, device=0, cfg=cfg, cost=cp)
    assert eng.n_ordinals == len(ords) - 1
    gp = search.mcts_search(eng, episodes=256, seed=11, leaf_batch=32)
    op = search.run_mcts(evaluator("oracle", text, cfg, cp, lw), len(ords) - 1, ords,
                         episodes=256, seed=11, leaf_batch=32)
    assert search.plan_actions(gp) == search.plan_actions(op)
    assert not H.compare_results(gp.result, op.result)


def test_emitted_plan_with_infer_rest_replays(oracle_lib):
    # SPEC emit_plan: the plan file is replayable; an InferRest decision is
    # kept as a decision and re-expanded on replay
    text = PROGRAMS["t2"]()
    cfg = capi.default_search_config(group_scopes=1, infer_rest_action=1)
    eng = engine.Engine(engine.Graph(text), device=0, cfg=cfg)
    res, seqs, _ = eng.rollout_batch([[]] * 256, list(range(256)))
    k = next(i for i, sq in enumerate(seqs) if any(a[3] == capi.PE_ACT_INFER_REST for a in sq))
    plan = capi.PePlan()
    plan.n_actions = len(seqs[k])
    for i, a in enumerate(seqs[k]):
        plan.actions[i] = capi.PeAction(*a, 0)
    plan.result = res[k]
    import json
    d = search.emit_plan(eng, plan)
    assert any("infer_rest" in a for a in json.loads(d)["actions"])
    again = eng.eval_batch([search.plan_actions_from_json(eng, d)])[0]
    assert not H.compare_results(again, res[k])
