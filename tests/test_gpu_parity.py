"""GPU parity: the sm_100a engine (libpe_b200.so, through the C-ABI) against
the oracle (patched reference + SPEC restatement) — bit-exact on every
integer field and on the full SPMD trace; runtime/reward within 1e-6
relative (north_star tolerance)."""
import os

import pytest

import fuzz_util as F
import helpers as H
from paper_2112_02958_b200 import capi, engine, modelgen

pytestmark = pytest.mark.gpu

TW = 16384


def _engine(text, cfg=None):
    return engine.Engine(engine.Graph(text), device=0, cfg=cfg)


def test_fig3_and_megatron_on_device(oracle_lib):
    text = modelgen.linear()
    eng = _engine(text)
    seqs = [[], [(1, 1, 0, 0)], [(1, 0, 0, 0)], [(0, 0, 0, 0)]]
    res, tr = eng.eval_batch(seqs, trace_words=TW)
    ref, rtr = H.eval_batch("oracle", text, seqs, trace_words=TW)
    assert res[0].peak_bytes == 10752 and res[0].flops == 16896
    assert res[2].reduction_bytes == 2048
    for a, b, x, y in zip(res, ref, tr, rtr):
        assert not H.compare_results(a, b)
        assert x[:x[0]] == y[:y[0]]
    assert eng.launch_count() >= 2


def test_random_programs_device_vs_oracle(oracle_lib):
    bad = []
    total = 0
    for i in range(48):
        # every fourth program on a non-power-of-two mesh (32-bit division)
        if i % 4 == 3:
            mesh = F.ODD_MESHES[i % 3]
            text = modelgen.random_program(9000 + i, mesh, dims=F.ODD_DIMS)
        else:
            mesh = F.MESHES[i % 3]
            text = modelgen.random_program(9000 + i, mesh)
        seqs = F.legal_sequences(text, mesh, 4242 + i, n_seqs=6)
        seqs += [modelgen.random_actions(31 * i + k, text, mesh) for k in range(4)]
        eng = _engine(text)
        res, tr = eng.eval_batch(seqs, trace_words=TW)
        ref, rtr = H.eval_batch("oracle", text, seqs, trace_words=TW)
        for k, (a, b, x, y) in enumerate(zip(res, ref, tr, rtr)):
            total += 1
            d = H.compare_results(a, b)
            if d or F.first_trace_diff(x, y) >= 0:
                bad.append((i, k, d))
    assert total == 48 * 10
    assert not bad, bad[:5]


@pytest.mark.parametrize("cfgno,group", [(1, 1), (2, 1), (2, 0)])
def test_rollouts_device_vs_oracle(oracle_lib, cfgno, group):
    text = modelgen.config_program(cfgno)
    cfg = capi.default_search_config(group_scopes=group)
    eng = _engine(text, cfg)
    n = 512
    seeds = [77 + i for i in range(n)]
    prefixes = [[] for _ in range(n)]
    res, seqs, legal = eng.rollout_batch(prefixes, seeds, legal=True)
    ref, rseqs, rlegal = H.rollout_batch("oracle", text, prefixes, seeds, cfg,
                                         legal_words=eng.legal_words, threads=os.cpu_count() or 1)
    assert seqs == rseqs
    assert legal == rlegal
    assert all(not H.compare_results(a, b) for a, b in zip(res, ref))


def test_resurfacing_rollouts_device_vs_oracle(oracle_lib):
    # stuck resurfacing (pe.h resurface_stuck; tests/test_resurface.py):
    # rollouts from the root and from prefixes that contain resurfaced
    # TileValue(op result) actions, legal bitmasks included
    nthr = os.cpu_count() or 1
    picked = 0
    for i in range(24):
        if i < 2:
            text = modelgen.config_program(2)
            cfg = capi.default_search_config(group_scopes=i, resurface_stuck=1)
        else:
            mesh = F.MESHES[i % 3]
            text = modelgen.random_program(70000 + i, mesh)
            cfg = capi.default_search_config(group_scopes=0, resurface_stuck=1)
        n_args = text.split("->")[0].count("%")
        eng = _engine(text, cfg)
        seeds = list(range(64))
        res, seqs, legal = eng.rollout_batch([[]] * 64, seeds, legal=True)
        ref, rseqs, rlegal = H.rollout_batch("oracle", text, [[]] * 64, seeds, cfg,
                                             legal_words=eng.legal_words, threads=nthr)
        assert seqs == rseqs and legal == rlegal
        assert all(not H.compare_results(a, b) for a, b in zip(res, ref))
        picked += sum(1 for s in seqs for a in s if a[3] == capi.PE_ACT_TILE and a[0] >= n_args)
        prefixes = [s[:k] for s in seqs[:8] for k in range(1, len(s) + 1)]
        if prefixes:
            ps = [500 + k for k in range(len(prefixes))]
            res, seqs2, legal = eng.rollout_batch(prefixes, ps, legal=True)
            ref, rseqs2, rlegal = H.rollout_batch("oracle", text, prefixes, ps, cfg,
                                                  legal_words=eng.legal_words, threads=nthr)
            assert seqs2 == rseqs2 and legal == rlegal
            assert all(not H.compare_results(a, b) for a, b in zip(res, ref))
    assert picked > 50


@pytest.mark.parametrize("cfgno,reuse", [(2, 0), (2, 4), (3, 0), (3, 4)])
def test_trie_scheduling_preserves_results(oracle_lib, monkeypatch, cfgno, reuse):
    # prefix-trie scheduling (pe.h pe_engine_sched_nodes) only reorders
    # candidates, and prefix-state reuse (pe_engine_set_state_reuse) starts
    # them from saved prefix states: acts, legal sets and results equal an
    # unscheduled engine's, call after call while the trie grows
    text = modelgen.config_program(cfgno)
    cfg = capi.default_search_config(group_scopes=1)
    sched = _engine(text, cfg)
    if reuse:
        sched.set_state_reuse(reuse)
    monkeypatch.setenv("PE_SCHED_DEPTH", "0")
    plain = _engine(text, cfg)
    n = 8192
    for call in range(4):
        seeds = [call * 100_000 + i for i in range(n)]
        legal = not reuse  # (legal-set output turns state reuse off)
        r1, s1, l1 = sched.rollout_batch([[]] * n, seeds, legal=legal)
        r2, s2, l2 = plain.rollout_batch([[]] * n, seeds, legal=legal)
        assert s1 == s2 and l1 == l2
        assert all(not H.compare_results(a, b) for a, b in zip(r1, r2))
    assert sched.sched_nodes() > 1 and plain.sched_nodes() == 0
    if cfgno == 2:
        ref, rseqs, _ = H.rollout_batch("oracle", text, [[]] * 256, seeds[:256], cfg,
                                        threads=os.cpu_count() or 1)
        assert rseqs == s1[:256]
        assert all(not H.compare_results(a, b) for a, b in zip(r1[:256], ref))


def test_l2_persist_window_preserves_results(oracle_lib, monkeypatch):
    # PE_L2_PERSIST=1 launches the main rollout kernel with the graph image
    # as a persisting L2 window (a cache hint only): same actions and results
    text = modelgen.config_program(2)
    cfg = capi.default_search_config(group_scopes=1)
    plain = _engine(text, cfg)
    monkeypatch.setenv("PE_L2_PERSIST", "1")
    hinted = _engine(text, cfg)
    n = 8192
    seeds = list(range(n))
    r1, s1, _ = hinted.rollout_batch([[]] * n, seeds)
    r2, s2, _ = plain.rollout_batch([[]] * n, seeds)
    assert s1 == s2
    assert all(not H.compare_results(a, b) for a, b in zip(r1, r2))
    ref, rseqs, _ = H.rollout_batch("oracle", text, [[]] * 256, seeds[:256], cfg,
                                    threads=os.cpu_count() or 1)
    assert rseqs == s1[:256]
    assert all(not H.compare_results(a, b) for a, b in zip(r1[:256], ref))


def test_gpt2_medium_24_layer_rollouts(oracle_lib):
    # config 3: 24-layer GPT-2-medium graph on [batch=4, model=2]
    text = modelgen.config_program(3)
    cfg = capi.default_search_config(group_scopes=1)
    eng = _engine(text, cfg)
    n = 24
    seeds = [5 + i for i in range(n)]
    res, seqs, _ = eng.rollout_batch([[]] * n, seeds)
    ref, _, _ = H.rollout_batch("oracle", text, [[]] * n, seeds, cfg, threads=os.cpu_count() or 1)
    ev_ref, _ = H.eval_batch("oracle", text, seqs, threads=os.cpu_count() or 1)
    for a, b, c in zip(res, ref, ev_ref):
        assert not H.compare_results(a, b)
        assert not H.compare_results(a, c)


def test_gpt2_medium_grouped_megatron_dp(oracle_lib):
    # grouped q_proj -> w1 -> x batch plan; 48 all_reduce(model),
    # 48 all_gather(batch) of 1,207,959,552 B.
    text = modelgen.config_program(3)
    eng = _engine(text)
    g = eng.graph
    seq = [g.action("l0_wq", 1, "model", group=True), g.action("l0_w1", 1, "model", group=True),
           g.action("x", 0, "batch")]
    res, tr = eng.eval_batch([seq], trace_words=1 << 16)
    ref, rtr = H.eval_batch("oracle", text, [seq], trace_words=1 << 16)
    assert not H.compare_results(res[0], ref[0])
    assert tr[0][:tr[0][0]] == rtr[0][:rtr[0][0]]
    r = res[0]
    assert r.ar_cnt[1] == 48 and r.ar_bytes[1] == 1610612736
    assert r.ag_cnt[0] == 48 and r.ag_bytes[0] == 1207959552


def test_capacity_retry_path(oracle_lib, monkeypatch):
    # force the tight arena to overflow: every candidate must take the retry
    # kernel (full-size arena) and still match the oracle exactly
    monkeypatch.setenv("PE_DEBUG_TIGHT_EM_CAP", "8")
    text = modelgen.config_program(2)
    cfg = capi.default_search_config(group_scopes=1)
    eng = _engine(text, cfg)
    n = 256
    res, seqs, _ = eng.rollout_batch([[]] * n, list(range(n)))
    ref, rseqs, _ = H.rollout_batch("oracle", text, [[]] * n, list(range(n)), cfg)
    assert seqs == rseqs
    assert all(r.status == 0 for r in res)
    assert all(not H.compare_results(a, b) for a, b in zip(res, ref))


INFER_PROGRAMS = {
    "mlp2": lambda: modelgen.build_mlp(2, (16, 64, 16), 8, (("model", 2),)),
    "mlp3": lambda: modelgen.build_mlp(3, (16, 64, 64, 16), 8, (("model", 2),)),
    "t1": lambda: modelgen.config_program(2),
    "t2": lambda: modelgen.build_transformer(2, mesh=(("model", 2),), **modelgen.TOY),
}


@pytest.mark.parametrize("cfgno", sorted(INFER_PROGRAMS))
def test_infer_rest_device_vs_reference(oracle_lib, cfgno):
    # a6: the engine's batched infer_rest expansion vs the reference's own
    # infer_rest after every single first decision (t1 / t2 / mlp3 include
    # prefixes where inference changes the state)
    text = INFER_PROGRAMS[cfgno]()
    eng = _engine(text)
    names, shapes = modelgen.program_values(text)
    seqs = []
    for a in range(eng.graph.n_args):
        for d in range(len(shapes[a])):
            if shapes[a][d] % eng.graph.axis_sizes[0] == 0:
                seqs.append([(a, d, 0, 0), (0, 0, 0, 2)])
    seqs.append([(0, 0, 0, 2)])  # InferRest first: nothing tiled -> no-op
    res, tr = eng.eval_batch(seqs, trace_words=TW)
    ref, rtr = H.eval_batch("oracle", text, seqs, trace_words=TW)
    for a, b, x, y in zip(res, ref, tr, rtr):
        assert not H.compare_results(a, b)
        assert x[:x[0]] == y[:y[0]]
    # the explicit API returns prefix + expanded marker + inferred tiles whose
    # evaluation equals evaluating the unexpanded InferRest decision
    for s in seqs[:6]:
        prefix = [capi.PeAction(*s[0], 0)]
        exp = eng.infer_rest(prefix)
        assert exp[0].value == prefix[0].value and exp[1].kind == capi.PE_ACT_INFER_REST
        assert all(x.kind == capi.PE_ACT_TILE and x.pad == capi.PE_ACT_FLAG_INFERRED
                   for x in exp[2:])
        a = eng.eval_batch([exp])[0]
        b = eng.eval_batch([s])[0]
        assert not H.compare_results(a, b)


@pytest.mark.parametrize("detailed,group", [(False, 0), (True, 0), (True, 1)])
def test_training_step_device_vs_oracle(oracle_lib, detailed, group):
    # the config-4 generator at toy size (detailed: MHLO granularity with
    # 4-way gradient accumulation, as config 4 itself)
    kw = dict(detailed=True, microbatches=4) if detailed else {}
    n = 128 if detailed else 256
    text = modelgen.build_training_step(2, mesh=(("batch", 2), ("model", 2)), **kw, **modelgen.TOY)
    cfg = capi.default_search_config(group_scopes=group)
    eng = _engine(text, cfg)
    res, seqs, legal = eng.rollout_batch([[]] * n, list(range(n)), legal=True)
    ref, rseqs, rlegal = H.rollout_batch("oracle", text, [[]] * n, list(range(n)), cfg,
                                         legal_words=eng.legal_words, threads=os.cpu_count() or 1)
    assert seqs == rseqs and legal == rlegal
    assert all(not H.compare_results(a, b) for a, b in zip(res, ref))
    ev, tr = eng.eval_batch(seqs[:64], trace_words=1 << 16)
    _, rtr = H.eval_batch("oracle", text, seqs[:64], trace_words=1 << 16,
                          threads=os.cpu_count() or 1)
    assert all(x[:x[0]] == y[:y[0]] for x, y in zip(tr, rtr))


def test_calibrated_arena_preserves_results(oracle_lib, monkeypatch):
    # arena calibration (automatic when the budget limits
    # slots, forced here): tighter caps, overflow through the retry path,
    # identical results
    text = modelgen.config_program(3)
    cfg = capi.default_search_config(group_scopes=1)
    plain = _engine(text, cfg)
    monkeypatch.setenv("PE_CALIBRATE", "2")
    calib = _engine(text, cfg)
    assert calib.arena_bytes() < plain.arena_bytes()
    n = 8192
    seeds = [123_000 + i for i in range(n)]
    r1, s1, _ = calib.rollout_batch([[]] * n, seeds)
    r2, s2, _ = plain.rollout_batch([[]] * n, seeds)
    assert s1 == s2
    assert all(not H.compare_results(a, b) for a, b in zip(r1, r2))
    ref, rseqs, _ = H.rollout_batch("oracle", text, [[]] * 64, seeds[:64], cfg,
                                    threads=os.cpu_count() or 1)
    assert rseqs == s1[:64]
    assert all(not H.compare_results(a, b) for a, b in zip(r1[:64], ref))


def test_config4_training_step_runs():
    # config 4 at full size (48 layers, 52,154 ops, 1,156 arguments): every
    # rollout evaluates (tight arena or retry), no failures
    text = modelgen.config_program(4)
    eng = _engine(text, capi.default_search_config(group_scopes=1))
    assert eng.graph.n_ops == 52154 and eng.graph.n_args == 1156
    res, seqs, _ = eng.rollout_batch([[]] * 256, list(range(256)))
    assert all(r.status == 0 for r in res)
    assert all(r.n_spmd_ops >= eng.graph.n_ops for r in res)
