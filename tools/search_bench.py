#!/usr/bin/env python3
"""Search time to the Megatron plan (BASELINE.json metric #2).

Config 3: the 24-layer GPT-2-medium graph on [batch=4, model=2], model axis
searched (parameters only, scope groups), memory budget 0.6 x the replicated
peak.  The same deterministic MCTS (pe_mcts_run) runs
  * on the GPU engine (pe_search: one rollout launch per leaf batch), and
  * on the reference CPU path (oracle/_ref: patched reference + SPEC
    restatement) with every host core evaluating the leaf batch,
and both report the wall-clock until the best plan carries the Megatron
signature (2 all_reduce / layer on `model`, 0 all_gather on `model`).

Multi-GPU (root-parallel): launch with torchrun; every rank searches its own
tree (seed + rank) and root statistics are all-reduced over NCCL every
--merge-every episodes; the first rank to hold a Megatron plan defines the
time (max over ranks of the search wall time is reported).

  python tools/search_bench.py [--episodes 1024] [--cpu]
  torchrun --nproc-per-node N tools/search_bench.py
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_2112_02958_b200 import capi, engine, modelgen, search  # noqa: E402


def setup(layers=24):
    if layers == 24:
        text = modelgen.config_program(3)
    else:
        text = modelgen.build_transformer(layers, mesh=(("batch", 4), ("model", 2)),
                                          **modelgen.GPT2_MEDIUM)
    g = engine.Graph(text)
    model = g.axis_index("model")
    cfg = capi.default_search_config(group_scopes=1, scoped_only=1, auto_axes_mask=1 << model)
    return text, g, cfg, model


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--episodes", type=int, default=1024)
    ap.add_argument("--leaf-batch", type=int, default=256)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--merge-every", type=int, default=256)
    ap.add_argument("--cpu", action="store_true", help="also time the reference CPU search")
    ap.add_argument("--layers", type=int, default=24)
    args = ap.parse_args()
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    merge = None
    if ws > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
        merge = search.TorchMerge()
    text, g, cfg, model = setup(args.layers)
    base = engine.Engine(g, device=local, cfg=cfg).baseline_bytes
    cp = capi.default_cost_params()
    cp.memory_budget_bytes = int(0.6 * base)
    eng = engine.Engine(g, device=local, cfg=cfg, cost=cp)
    layers = args.layers

    def run(episodes):
        t0 = time.perf_counter()
        p = search.mcts_search(eng, episodes=episodes, seed=args.seed + rank,
                               leaf_batch=args.leaf_batch, merge=merge,
                               merge_every=args.merge_every, rank=rank)
        return p, time.perf_counter() - t0

    search.mcts_search(eng, episodes=args.leaf_batch, seed=12345, leaf_batch=args.leaf_batch)
    plan, dt = run(args.episodes)
    ok = search.megatron_signature(plan.result, model, layers)
    # deterministic: re-run with the budget that first reached the plan
    found = plan.found_at_episode + 1
    budget = ((found + args.leaf_batch - 1) // args.leaf_batch) * args.leaf_batch
    p2, t_found = run(budget)
    same = search.plan_actions(p2) == search.plan_actions(plan)
    out = {"metric": "search time to Megatron plan", "config": "gpt2-medium-24L [batch=4, model=2]",
           "gpus": ws, "episodes_budget": args.episodes, "leaf_batch": args.leaf_batch,
           "megatron_found": bool(ok), "found_at_episode": plan.found_at_episode,
           "episodes_to_found": budget, "gpu_search_s_to_megatron": t_found,
           "gpu_search_s_full_budget": dt, "gpu_episodes_per_s": args.episodes / dt,
           "replay_identical": bool(same), "plan": search.plan_actions(plan),
           "ar_model": plan.result.ar_cnt[model], "ag_model": plan.result.ag_cnt[model]}
    if args.cpu and rank == 0:
        import helpers as H
        ords = search.ordinal_actions(g, cfg)
        lw = (len(ords) - 1 + 63) // 64
        threads = os.cpu_count() or 1

        def ev(prefixes, seeds):
            return H.rollout_batch("oracle", text, prefixes, seeds, cfg, cp=cp, legal_words=lw,
                                   threads=threads)
        t0 = time.perf_counter()
        cpu_plan = search.run_mcts(ev, len(ords) - 1, ords, episodes=budget, seed=args.seed,
                                   leaf_batch=args.leaf_batch)
        t_cpu = time.perf_counter() - t0
        out.update({"cpu_search_s_to_megatron": t_cpu, "cpu_threads": threads,
                    "cpu_plan_identical": search.plan_actions(cpu_plan) == search.plan_actions(plan)
                    if ws == 1 else None,
                    "speedup_time_to_megatron": t_cpu / t_found})
    if rank == 0:
        print(json.dumps(out))
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
