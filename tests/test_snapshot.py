"""Prefix-state reuse: a rollout resumed from the saved
state after its own first d decisions equals the rollout from the root
(actions, every result field), here on the host-compiled core against the
oracle; the device path is checked against an unscheduled engine in
test_gpu_parity.py::test_trie_scheduling_preserves_results."""
import ctypes as C

import pytest

import helpers as H
import fuzz_util as F
from paper_2112_02958_b200 import capi, modelgen
from paper_2112_02958_b200.capi import PeAction, PeResult, PeSearchConfig, PeCostParams


def resumed(text, cfg, seeds, d):
    lib = C.CDLL(H.build_harness())
    f = lib.harness_resume_rollouts
    f.restype = C.c_int
    f.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(PeSearchConfig), C.POINTER(PeCostParams),
                  C.c_void_p, C.c_uint32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                  C.c_char_p, C.c_size_t]
    b = text.encode()
    n = len(seeds)
    maxd = cfg.max_decisions
    sd = (C.c_uint64 * n)(*seeds)
    aout = (PeAction * (n * maxd))()
    nout = (C.c_uint32 * n)()
    out = (PeResult * n)()
    err = C.create_string_buffer(256)
    cp = capi.default_cost_params()
    assert f(b, len(b), C.byref(cfg), C.byref(cp), sd, n, d, aout, nout, out, err, 256) == 0
    seqs = [[(aout[i * maxd + k].value, aout[i * maxd + k].dim, aout[i * maxd + k].axis,
              aout[i * maxd + k].kind) for k in range(nout[i])] for i in range(n)]
    return list(out), seqs


@pytest.mark.parametrize("d", [1, 2, 3])
def test_resumed_rollouts_equal_oracle(oracle_lib, harness_lib, d):
    cases = [(modelgen.config_program(2), 1), (modelgen.config_program(2), 0),
             (modelgen.config_program(1), 1)]
    cases += [(modelgen.random_program(81000 + i, F.MESHES[i % 3]), 0) for i in range(30)]
    for text, group in cases:
        cfg = capi.default_search_config(group_scopes=group)
        seeds = list(range(40))
        ro, so, _ = H.rollout_batch("oracle", text, [[]] * 40, seeds, cfg)
        rr, sr = resumed(text, cfg, seeds, d)
        assert so == sr
        assert all(not H.compare_results(a, b) for a, b in zip(ro, rr))
