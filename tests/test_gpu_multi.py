"""Root-parallel search with the GPU engine as the
evaluator: the native NCCL entry point (pe.h pe_search_multi: root
statistics all-reduced on the device) and 2 ranks on the test GPU merging
through gloo.  The ranks' kernels never wait on each other (the merge is a
host-side collective between launches), so one GPU stands in legitimately;
no 8-GPU scaling curve is claimed from this."""
import os

import pytest
import torch.multiprocessing as mp

import helpers as H
from paper_2112_02958_b200 import engine, modelgen, search
from test_search import TWO_LAYER, evaluator, setup

pytestmark = pytest.mark.gpu


def test_nccl_search_single_rank_equals_pe_search(oracle_lib):
    text = modelgen.build_transformer(**TWO_LAYER)
    g, cfg, cp, ords, lw = setup(text)
    eng = engine.Engine(g, device=0, cfg=cfg, cost=cp)
    comm = search.NcclComm(1, 0, 0)
    try:
        a = search.mcts_search_multi(eng, comm, episodes=256, seed=7, leaf_batch=32, merge_every=64)
    finally:
        comm.close()
    b = search.mcts_search(eng, episodes=256, seed=7, leaf_batch=32)
    assert search.plan_actions(a) == search.plan_actions(b)
    assert not H.compare_results(a.result, b.result)
    assert a.winner_rank == 0


def _rank_main(rank, world, port, text, out):
    import sys

    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    g, cfg, cp, ords, lw = setup(text)
    eng = engine.Engine(g, device=0, cfg=cfg, cost=cp)
    merge = search.TorchMerge(device="cpu")
    p = search.mcts_search(eng, episodes=256, seed=5, leaf_batch=16, merge=merge, merge_every=64,
                           rank=rank)
    # the same root-parallel search with the host-compiled core as evaluator
    hm = search.TorchMerge(device="cpu")
    q = search.run_mcts(evaluator("harness", text, cfg, cp, lw), len(ords) - 1, ords,
                        episodes=256, seed=5, leaf_batch=16, merge=hm, merge_every=64, rank=rank)
    out[rank] = (search.plan_actions(p), p.winner_rank, p.result.reward, merge.calls,
                 search.plan_actions(q), q.winner_rank)
    dist.destroy_process_group()


def test_two_ranks_gloo_merge_with_gpu_engines(harness_lib):
    text = modelgen.build_transformer(**TWO_LAYER)
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = 31500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, text, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    a, b = out[0], out[1]
    assert a[0] == b[0] and a[1] == b[1] and a[2] == b[2]  # one winning plan on every rank
    assert a[3] == b[3] == 256 // 64 + 3
    assert a[0] == a[4] and a[1] == a[5]  # = the CPU-evaluated root-parallel search
