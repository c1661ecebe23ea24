"""Differential fuzz of the engine's rewrite automaton (host-compiled test
harness of paper_2112_02958_b200/csrc/pe_core.cuh) against the oracle:
random programs over all 18 base kinds x legal action sequences on three
meshes; every integer field and the whole SPMD trace must be bit-identical.
The device build is checked against the same oracle in test_gpu_parity.py."""
import helpers as H
import fuzz_util as F
import pytest
from paper_2112_02958_b200 import capi, modelgen


@pytest.mark.parametrize("seed0", [0, 5000])
def test_random_programs_match_oracle(oracle_lib, harness_lib, seed0):
    n_bad = 0
    for i in range(120):
        mesh = F.MESHES[i % 3]
        text = modelgen.random_program(seed0 + i, mesh)
        seqs = F.legal_sequences(text, mesh, seed0 * 31 + i)
        ro, to = H.eval_batch("oracle", text, seqs, trace_words=8192)
        rh, th = H.eval_batch("harness", text, seqs, trace_words=8192)
        for a, b, x, y in zip(ro, rh, to, th):
            if H.compare_results(a, b) or F.first_trace_diff(x, y) >= 0:
                n_bad += 1
    assert n_bad == 0


def test_non_power_of_two_meshes_match_oracle(oracle_lib, harness_lib):
    n_bad = n_tiled = 0
    for i in range(150):
        mesh = F.ODD_MESHES[i % 3]
        text = modelgen.random_program(31000 + i, mesh, dims=F.ODD_DIMS)
        seqs = F.legal_sequences(text, mesh, 31000 + i)
        ro, to = H.eval_batch("oracle", text, seqs, trace_words=8192)
        rh, th = H.eval_batch("harness", text, seqs, trace_words=8192)
        for a, b, x, y in zip(ro, rh, to, th):
            n_tiled += a.n_steps > 0 and a.status == 0
            if H.compare_results(a, b) or F.first_trace_diff(x, y) >= 0:
                n_bad += 1
    assert n_bad == 0 and n_tiled > 100


def test_illegal_and_unordered_actions_match(oracle_lib, harness_lib):
    bad = 0
    for text, mesh, seqs in F.corpus(150, 777):
        ro, to = H.eval_batch("oracle", text, seqs, trace_words=8192)
        rh, th = H.eval_batch("harness", text, seqs, trace_words=8192)
        for a, b, x, y in zip(ro, rh, to, th):
            bad += bool(H.compare_results(a, b)) or F.first_trace_diff(x, y) >= 0
    assert bad == 0


@pytest.mark.parametrize("cfgno,group", [(1, 1), (2, 1), (2, 0)])
def test_rollouts_match_oracle(oracle_lib, harness_lib, cfgno, group):
    text = modelgen.config_program(cfgno)
    cfg = capi.default_search_config(group_scopes=group)
    lw = (H.oracle_info(text, cfg)["n_ordinals"] + 63) // 64
    seeds = list(range(200))
    ro, so, lo = H.rollout_batch("oracle", text, [[]] * 200, seeds, cfg, legal_words=lw)
    rh, sh, lh = H.rollout_batch("harness", text, [[]] * 200, seeds, cfg, legal_words=lw)
    assert so == sh and lo == lh
    assert all(not H.compare_results(a, b) for a, b in zip(ro, rh))


def test_megatron_two_layer_and_reshape_hazard(oracle_lib, harness_lib):
    text = modelgen.build_transformer(2, mesh=(("model", 2),), **modelgen.TOY)
    names = modelgen.program_values(text)[0]
    seq = [(names.index(f"l{l}_{w}"), d, 0, 0) for l in range(2)
           for w, d in (("wq", 1), ("w1", 1))]
    ro, to = H.eval_batch("oracle", text, [seq], trace_words=16384)
    rh, th = H.eval_batch("harness", text, [seq], trace_words=16384)
    assert not H.compare_results(ro[0], rh[0]) and to == th
    assert sum(rh[0].ar_cnt) == 4 and rh[0].reduction_bytes == 1024


def test_training_step_graphs_match_oracle(oracle_lib, harness_lib):
    # config-4 family (forward + reverse-mode gradients + Adam) at toy size:
    # rollouts, legal sets and full SPMD traces identical
    # (the last two: config 4's own generator -- MHLO-granularity ops,
    # stable softmax, GELU, dropout, clipped Adam, gradient accumulation)
    for layers, mesh, kw in ((1, (("m", 2),), {}), (2, (("batch", 2), ("model", 2)), {}),
                             (1, (("m", 2),), dict(detailed=True, microbatches=2)),
                             (1, (("batch", 2), ("model", 2)), dict(detailed=True, microbatches=2))):
        text = modelgen.build_training_step(layers, mesh=mesh, **kw, **modelgen.TOY)
        cfg = capi.default_search_config(group_scopes=0)
        lw = (H.oracle_info(text, cfg)["n_ordinals"] + 63) // 64
        n = 60
        ro, so, lo = H.rollout_batch("oracle", text, [[]] * n, list(range(n)), cfg, legal_words=lw,
                                     threads=8)
        rh, sh, lh = H.rollout_batch("harness", text, [[]] * n, list(range(n)), cfg, legal_words=lw)
        assert so == sh and lo == lh
        assert all(not H.compare_results(a, b) for a, b in zip(ro, rh))
        e1, t1 = H.eval_batch("oracle", text, so, trace_words=1 << 16, threads=8)
        e2, t2 = H.eval_batch("harness", text, so, trace_words=1 << 16)
        assert all(x[:x[0]] == y[:y[0]] for x, y in zip(t1, t2))
