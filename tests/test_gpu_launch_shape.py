"""GPU parity of the exact launch shape bench.py times.

A bench step is 1,048,576 root rollouts (round 1: 262,144), about seven
times the engine's resident slots (148 SMs x 1024 = 151,552).  That launch
takes paths small batches never reach: SM-wide 1024-thread blocks at 32
candidates per warp (pe_engine.cu launch geometry), the warp-chunked later
waves claimed from the work counter (__activemask + __shfl_sync), and arena
reuse by later candidates inside one launch.  Every candidate of such a launch
must equal the same seed evaluated in single-wave launches (8,192 candidates:
two per warp, one-warp blocks), and a strided sample must equal the oracle (the patched reference's
propagate / lower_to_spmd / collective_stats + the SPEC cost and rollout
restatement) bit-exactly on every integer field.
"""
import os

import numpy as np
import pytest

import helpers as H
from paper_2112_02958_b200 import capi, engine, modelgen

pytestmark = pytest.mark.gpu

N_FULL = 1048576  # bench.py --batch default
WAVE = 8192


def _rows_equal(a_res, a_acts, a_n, b_res, b_acts, b_n):
    """Indices where two rollout outputs differ (results byte-exact, action
    rows compared up to n_acts)."""
    bad = np.nonzero((a_n != b_n) | (a_res != b_res).any(axis=1))[0]
    maxd = a_acts.shape[1]
    mask = np.arange(maxd)[None, :] < a_n[:, None]
    diff = ((a_acts != b_acts).any(axis=2) & mask).any(axis=1)
    return np.union1d(bad, np.nonzero(diff)[0])


def _seqs(acts, n):
    return [[tuple(int(x) for x in acts[i, k]) for k in range(int(n[i]))] for i in range(len(n))]


@pytest.mark.parametrize("cfgno,n_oracle", [(2, 2048), (3, 128)])
def test_bench_launch_shape_equals_single_wave_and_oracle(oracle_lib, cfgno, n_oracle):
    text = modelgen.config_program(cfgno)
    cfg = capi.default_search_config(group_scopes=1)
    eng = engine.Engine(engine.Graph(text), device=0, cfg=cfg)
    assert N_FULL > eng.slots(), (N_FULL, eng.slots())
    seeds = np.arange(N_FULL, dtype=np.uint64) + np.uint64(1_000_003)
    # warm-up call grows the scheduling trie as the bench's warm-up steps do
    eng.rollout_roots_np(seeds[:N_FULL // 2] + np.uint64(9_999_999))
    r_full, a_full, n_full = eng.rollout_roots_np(seeds)
    st_off = capi.PeResult.status.offset // 4
    assert (r_full.view(np.int32)[:, st_off] == 0).all()  # every candidate evaluated OK

    # the same seeds as 32 single-wave launches of 8,192
    parts = [eng.rollout_roots_np(seeds[i:i + WAVE]) for i in range(0, N_FULL, WAVE)]
    r_w = np.concatenate([p[0] for p in parts])
    a_w = np.concatenate([p[1] for p in parts])
    n_w = np.concatenate([p[2] for p in parts])
    bad = _rows_equal(r_full, a_full, n_full, r_w, a_w, n_w)
    assert bad.size == 0, (bad.size, bad[:8])

    # strided sample against the oracle
    idx = np.arange(0, N_FULL, N_FULL // n_oracle)[:n_oracle]
    ref, rseqs, _ = H.rollout_batch("oracle", text, [[]] * len(idx), [int(s) for s in seeds[idx]],
                                    cfg, threads=os.cpu_count() or 1)
    assert _seqs(a_full[idx], n_full[idx]) == rseqs
    mism = [i for i, k in enumerate(idx)
            if H.compare_results(capi.PeResult.from_buffer_copy(r_full[k].tobytes()), ref[i])]
    assert not mism, mism[:8]


def test_config4_multi_wave_launch_equals_single_wave():
    # config 4 (52,154 ops) is slot-limited by its arena: a launch of
    # 2 x slots + 37 candidates runs second and third waves through the work
    # counter; every candidate equals its evaluation in launches of at most
    # one wave.  (The reference CPU path needs well over 30 minutes per
    # candidate here -- profiles/r2_cfg4_cpu_baseline.json -- so the oracle
    # parity of this generator is checked at toy size in test_gpu_parity.py
    # and tests/test_core_fuzz.py.)
    text = modelgen.config_program(4)
    cfg = capi.default_search_config(group_scopes=1)
    eng = engine.Engine(engine.Graph(text), device=0, cfg=cfg)
    slots = eng.slots()
    n = 2 * slots + 37
    seeds = np.arange(n, dtype=np.uint64) + np.uint64(77_000)
    r_full, a_full, n_full = eng.rollout_roots_np(seeds)
    wave = min(slots, 4096)
    parts = [eng.rollout_roots_np(seeds[i:i + wave]) for i in range(0, n, wave)]
    r_w = np.concatenate([p[0] for p in parts])
    a_w = np.concatenate([p[1] for p in parts])
    n_w = np.concatenate([p[2] for p in parts])
    bad = _rows_equal(r_full, a_full, n_full, r_w, a_w, n_w)
    assert bad.size == 0, (bad.size, bad[:8])
    st_off = capi.PeResult.status.offset // 4
    assert (r_full.view(np.int32)[:, st_off] == 0).all()
