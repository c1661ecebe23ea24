"""Incremental evaluation (§8(b) pe_state handles; MCTS leaves as parent
state + 1 action): results from saved states are
bit-identical to evaluating the whole sequence from the untiled graph, and
the prefix-state cache never changes a rollout's actions or result."""
import os

import pytest

import helpers as H
from paper_2112_02958_b200 import capi, engine, modelgen

pytestmark = pytest.mark.gpu
TW = 1 << 16


def _legal_actions(eng, seq):
    res, seqs, legal = eng.rollout_batch([seq + [(0, 0, 0, capi.PE_ACT_STOP)]], [0], legal=True)
    out = []
    for o in range(eng.n_ordinals):
        if (legal[0][o // 64] >> (o % 64)) & 1:
            a = eng.ordinal_action(o)
            out.append((a.value, a.dim, a.axis, a.kind))
    return out


@pytest.mark.parametrize("cfgno", [2, 3])
def test_parent_plus_one_action_equals_full_replay(oracle_lib, cfgno):
    text = modelgen.config_program(cfgno)
    cfg = capi.default_search_config(group_scopes=1)
    eng = engine.Engine(engine.Graph(text), device=0, cfg=cfg)
    _, seqs, _ = eng.rollout_batch([[]] * 64, list(range(300, 364)))
    parents = [s[:2] for s in seqs if len(s) >= 2][:6] + [[]]
    cands, ps = [], []
    for p in parents:
        st = eng.state(p) if p else None
        if st is not None:
            full = eng.eval_batch([p])[0]
            assert not H.compare_results(st.result(), full)
            # pe_state_specs equals the header of the parity trace
            _, tr = eng.eval_batch([p], trace_words=TW)
            args, res_spec, stuck = st.specs()
            A = tr[0][1]
            assert args == [x & 0xFFFFFFFF for x in tr[0][2:2 + A]]
            assert res_spec == tr[0][2 + A] & 0xFFFFFFFF
            assert len(stuck) == tr[0][3 + A]
        for a in _legal_actions(eng, p)[:12]:
            cands.append((st, p, a))
    res = eng.eval_from_states([c[0] for c in cands], [[c[2]] for c in cands])
    full = eng.eval_batch([c[1] + [c[2]] for c in cands])
    assert all(not H.compare_results(a, b) for a, b in zip(res, full))
    ref, _ = H.eval_batch("oracle", text, [c[1] + [c[2]] for c in cands[:48]],
                          threads=os.cpu_count() or 1)
    assert all(not H.compare_results(a, b) for a, b in zip(res, ref))


@pytest.mark.parametrize("tight", [None, "8"])
def test_prefix_cache_preserves_rollouts(oracle_lib, monkeypatch, tight):
    # MCTS-like traffic: prefixes growing one action at a time; the cached
    # engine starts each from its longest cached prefix, also when the tight
    # arena is forced to overflow and candidates take the retry path.
    if tight:
        monkeypatch.setenv("PE_DEBUG_TIGHT_EM_CAP", tight)
    text = modelgen.config_program(2)
    cfg = capi.default_search_config(group_scopes=0)
    cached = engine.Engine(engine.Graph(text), device=0, cfg=cfg)
    cached.set_prefix_cache(1.0)
    monkeypatch.delenv("PE_DEBUG_TIGHT_EM_CAP", raising=False)
    plain = engine.Engine(engine.Graph(text), device=0, cfg=cfg)
    _, seqs, _ = plain.rollout_batch([[]] * 128, list(range(128)))
    for depth in range(1, 5):
        prefixes = [s[:depth] for s in seqs if len(s) >= depth]
        seeds = [depth * 1000 + i for i in range(len(prefixes))]
        r1, s1, l1 = cached.rollout_batch(prefixes, seeds, legal=True)
        r2, s2, l2 = plain.rollout_batch(prefixes, seeds, legal=True)
        assert s1 == s2 and l1 == l2
        assert all(not H.compare_results(a, b) for a, b in zip(r1, r2))
    # (with the SPMD-op cap forced down, lowering overflows after the prefix
    # state was saved: the retry path re-evaluates from the untiled graph)
    stats = cached.prefix_cache_stats()
    assert stats["hits"] > 0 and stats["saved"] > 0
