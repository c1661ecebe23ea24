"""Ranker pre-filter (SPEC ranker module): the SPEC
examples and properties, and the worklist filter it feeds
(pe_search_config.worklist_args) through the oracle and the host-compiled
core."""
import re

import numpy as np
import pytest

import helpers as H
from paper_2112_02958_b200 import capi, engine, modelgen, ranker, search


def oracle_evaluate(text, seqs, cp):
    return H.eval_batch("oracle", text, seqs, cp=cp)[0]


def test_featurize_linear_structure():
    enc = ranker.featurize(modelgen.linear())
    assert enc.n_nodes == 5 and enc.n_args == 3  # 3 args + 2 ops (PAPER Fig. 2)
    edges = set(zip(enc.agg_from.tolist(), enc.agg_to.tolist()))
    # dataflow x->dot, w->dot, dot->add, b->add (aggregated both ways)
    for p, c in ((0, 3), (1, 3), (3, 4), (2, 4)):
        assert (p, c) in edges and (c, p) in edges
    assert enc.x.shape[1] == ranker.N_FEATURES
    assert all(enc.x[a, ranker.ARG_SLOT] == 1 for a in range(3))
    assert enc.x[3, ranker.KINDS.index("dot")] == 1 and enc.x[4, ranker.KINDS.index("add")] == 1


def test_partitioned_axes_indicator_and_determinism():
    text = modelgen.linear()
    tiled = ranker.featurize(text, arg_axes=[[], [0], []])
    col = ranker.KIND_SLOTS + ranker.MAX_RANK + 1 + 0
    assert tiled.x[1, col] == 1 and tiled.x[0, col] == 0
    a, b = ranker.featurize(text), ranker.featurize(text)
    assert np.array_equal(a.x, b.x) and np.array_equal(a.agg_to, b.agg_to)
    # relabelling value ids (structure preserved) leaves encodings and scores unchanged
    renamed = text.replace("%w", "%weights").replace("%0", "%t0").replace("%1", "%t1")
    c = ranker.featurize(renamed)
    m = ranker.RankerModel(3)
    assert np.array_equal(a.x, c.x) and np.allclose(m.scores(a), m.scores(c))


def test_structural_edges_link_scope_siblings():
    text = modelgen.build_transformer(2, mesh=(("model", 2),), **modelgen.TOY)
    enc = ranker.featurize(text)
    names = enc.names
    e = set(zip(enc.agg_from.tolist(), enc.agg_to.tolist()))
    assert (names.index("l0_wq"), names.index("l1_wq")) in e
    assert (names.index("l0_wq"), names.index("l1_wk")) not in e


def test_gradient_check_every_block():
    # analytic vs central finite differences (eps 1e-4), within 1e-4 relative
    rng = np.random.default_rng(0)
    text = modelgen.build_transformer(1, mesh=(("model", 2),), **modelgen.TOY)
    enc = ranker.featurize(text)
    data = [(enc, [1, 5])]
    m = ranker.RankerModel(7)
    for k in m.p:
        m.p[k] = m.p[k] + rng.normal(0, 0.3, m.p[k].shape)
    _, g = ranker.loss_and_grad(m, data)
    eps = 1e-4
    for k in ranker.RankerModel.BLOCKS:
        flat = m.p[k].reshape(-1)
        for idx in rng.choice(flat.size, size=min(6, flat.size), replace=False):
            old = flat[idx]
            flat[idx] = old + eps
            lp = ranker.loss_and_grad(m, data)[0]
            flat[idx] = old - eps
            lm = ranker.loss_and_grad(m, data)[0]
            flat[idx] = old
            num = (lp - lm) / (2 * eps)
            ana = g[k].reshape(-1)[idx]
            assert abs(num - ana) <= 1e-4 * max(1.0, abs(num), abs(ana)), (k, idx, num, ana)


def test_training_converges_and_zero_epochs_is_identity():
    enc = ranker.featurize(modelgen.linear())
    data = [(enc, [1])]
    m0 = ranker.RankerModel(1)
    same = ranker.train(data, epochs=0, seed=1)
    assert all(np.array_equal(same.p[k], m0.p[k]) for k in m0.p)
    m = ranker.train(data, epochs=200, seed=1)
    assert m.final_loss < 0.1  # SPEC: 1 example, 200 epochs -> loss < 0.1
    assert ranker.score_and_filter(enc, m, 1) == [1]


def test_score_and_filter_k():
    enc = ranker.featurize(modelgen.config_program(2))
    m = ranker.RankerModel(2)
    assert ranker.score_and_filter(enc, m, 100) == list(range(enc.n_args))
    big = modelgen.build_training_step(4, mesh=(("m", 2),), **modelgen.TOY)
    e2 = ranker.featurize(big)
    assert e2.n_args > 25 and len(ranker.score_and_filter(e2, m, 25)) == 25


def test_model_file_roundtrip(tmp_path):
    m = ranker.RankerModel(4)
    path = tmp_path / "r.txt"
    ranker.save_model(m, str(path))
    assert open(path).readline().strip() == ranker.MODEL_MAGIC
    m2 = ranker.load_model(str(path))
    enc = ranker.featurize(modelgen.config_program(2))
    assert np.array_equal(m.scores(enc), m2.scores(enc))


def test_labels_and_dataset_reproducible(oracle_lib):
    # SPEC: n=1 on `linear` -> label {%w}; same seed twice -> identical dataset
    assert ranker.label_program(modelgen.linear(), oracle_evaluate) == {1}
    a = ranker.generate_dataset(3, seed=0, evaluate=oracle_evaluate)
    b = ranker.generate_dataset(3, seed=0, evaluate=oracle_evaluate)
    assert len(a) == 3
    assert [lab for _, lab in a] == [lab for _, lab in b]
    assert all(np.array_equal(x.x, y.x) for (x, _), (y, _) in zip(a, b))


@pytest.mark.parametrize("group", [0, 1])
def test_worklist_filter_matches_oracle(oracle_lib, harness_lib, group):
    text = modelgen.build_transformer(2, mesh=(("model", 2),), **modelgen.TOY)
    g = engine.Graph(text)
    keep = [g.value_index("l0_wq"), g.value_index("l1_w1"), g.value_index("x")]
    cfg = capi.default_search_config(group_scopes=group).restrict_worklist(keep)
    full = H.oracle_info(text, capi.default_search_config(group_scopes=group))["n_ordinals"]
    n_ord = H.oracle_info(text, cfg)["n_ordinals"]
    assert 0 < n_ord < full
    lw = (n_ord + 63) // 64
    ro, so, lo = H.rollout_batch("oracle", text, [[]] * 100, list(range(100)), cfg, legal_words=lw)
    rh, sh, lh = H.rollout_batch("harness", text, [[]] * 100, list(range(100)), cfg, legal_words=lw)
    assert so == sh and lo == lh
    assert all(not H.compare_results(a, b) for a, b in zip(ro, rh))
    # only kept entries are ever decided
    if group:
        groups = {gi for gi, mem in enumerate(g.groups) if set(mem) & set(keep)}
        assert all(a[0] in groups for s in so for a in s if a[3] == capi.PE_ACT_TILE_GROUP)
    else:
        assert all(a[0] in keep for s in so for a in s)


def test_filtered_config_feeds_search(oracle_lib, harness_lib):
    text = modelgen.build_transformer(2, mesh=(("model", 2),), **modelgen.TOY)
    m = ranker.RankerModel(0)
    cfg = ranker.filtered_config(text, m, capi.default_search_config(group_scopes=0), k=4)
    assert cfg.n_worklist_args == 4
    ords = search.ordinal_actions(engine.Graph(text), cfg)
    # Python ordinal decoding follows the filtered worklist too
    assert len(ords) - 1 == H.oracle_info(text, cfg)["n_ordinals"]
