#!/usr/bin/env python3
"""bench.py — partition candidates evaluated / s on B200.

Workload (BASELINE.json configs[2], the north_star's "24-layer transformer
graph"): the 24-layer GPT-2-medium-shaped forward graph (d=1024, H=16,
F=4096, S=1024, B=8; 1032 ops, 145 arguments) on the 2-axis mesh
[batch=4, model=2], scope-grouped worklist, auto axes {batch, model}.  A
candidate = one MCTS rollout from the root under the SPEC rollout policy
(uniform over legal TileValue actions, Stop weight 2 after the first
decision, <= 32 decisions), each action followed by propagate, then
lower_to_spmd + collective_stats + cost model + reward.  One step = one
launch over a batch of candidates with fresh seeds.

  python bench.py [--gpus N --steps K --warmup W]        engine (this repo)
  python bench.py --impl reference ...                    reference CPU path

Under torchrun every rank evaluates its own candidate stream (seeds offset by
rank; weak scaling, no data-path collective); timing is max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

METRIC = "partition candidates evaluated/sec"
UNIT = "candidates/s"
WORKLOAD = "gpt2-medium-24L rollouts, mesh [batch=4, model=2], grouped worklist"


def _config(batch, extra=None):
    c = {"workload": WORKLOAD, "graph": "24-layer GPT-2-medium forward (1032 ops, 145 args)",
         "mesh": "[batch=4, model=2]", "candidates_per_step": batch,
         "candidate": "SPEC rollout from root: uniform legal TileValue, Stop w=2 after 1st, <=32",
         "auto_axes": ["batch", "model"], "group_scopes": True,
         "infer_rest_in_action_space": False, "rng": "splitmix64 per candidate (both arms)"}
    if extra:
        c.update(extra)
    return c


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, device=0):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > i + 2 and s[i + 2].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws > 1:
        import torch.distributed as dist
        if not dist.is_initialized():
            backend = "nccl"
            import torch
            if not torch.cuda.is_available():
                backend = "gloo"
            dist.init_process_group(backend)
        return dist, dist.get_rank(), ws
    return None, 0, 1


def _max_over_ranks(dist, x: float, device=None) -> float:
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------- CPU baseline
def _cpu_model() -> str:
    """The host CPU the reference arm ran on (state it)."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_reference(text, n_cand, seed0, threads):
    """The reference's own CPU path (oracle/_ref: patched REF propagate /
    lower_to_spmd / collective_stats + SPEC cost/rollout restatement) on
    `threads` host cores.  Returns (cand/s, seconds)."""
    import helpers as H
    from paper_2112_02958_b200 import capi
    cfg = capi.default_search_config(group_scopes=1)
    t0 = time.perf_counter()
    H.rollout_batch("oracle", text, [[]] * n_cand, [seed0 + i for i in range(n_cand)], cfg,
                    threads=threads)
    dt = time.perf_counter() - t0
    return n_cand / dt, dt


def run_reference(args):
    dist, rank, ws = _dist()
    if rank != 0:
        return 0
    from paper_2112_02958_b200 import modelgen
    text = modelgen.config_program(3)
    threads = os.cpu_count() or 1
    # ~2 s of CPU work per step on this path; 8 rollouts per thread so one
    # long rollout does not leave the other threads idle for most of the step
    per_step = 8 * threads
    for w in range(args.warmup):
        cpu_reference(text, per_step, 10_000_000 + w * per_step, threads)
    total = 0.0
    n = 0
    for s in range(args.steps):
        _, dt = cpu_reference(text, per_step, 20_000_000 + s * per_step, threads)
        total += dt
        n += per_step
    v = n / total
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic", "config": _config(per_step, {"parallelism": f"{threads} host threads"}),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "cpu": _cpu_model(), "kind": "reference",
                             "sample": f"{args.steps} x {per_step} rollouts of the bench workload"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def _parity_sample(text, cfg, seeds, acts_out, nacts, res, B, maxd, n_sample):
    """Oracle check of a strided sample of one timed batch: returns
    {"n", "mismatches", "stride", "kind"} or None without the oracle."""
    import ctypes as C

    import numpy as np

    import helpers as H
    from paper_2112_02958_b200 import capi
    if not os.path.exists(H.ORACLE_SO):
        return {"n": 0, "mismatches": None, "note": "oracle/_ref not built on this host"}
    stride = max(1, B // n_sample)
    idx = np.arange(0, B, stride)[:n_sample]
    a = acts_out.view(B, maxd, 8).cpu().numpy()[idx]
    na = nacts.cpu().numpy().astype(np.int64)[idx]
    rr = res.view(B, C.sizeof(capi.PeResult)).cpu().numpy()[idx]
    ref, rseqs, _ = H.rollout_batch("oracle", text, [[]] * len(idx), [int(x) for x in seeds[idx]],
                                    cfg, threads=os.cpu_count() or 1)
    bad = 0
    for j in range(len(idx)):
        v = a[j].view(np.uint32)[:, 0]
        seq = [(int(v[k]), int(a[j, k, 4]), int(a[j, k, 5]), int(a[j, k, 6])) for k in range(na[j])]
        r = capi.PeResult.from_buffer_copy(rr[j].tobytes())
        if seq != rseqs[j] or H.compare_results(r, ref[j]):
            bad += 1
    return {"n": int(len(idx)), "mismatches": bad, "stride": int(stride),
            "kind": "oracle/_ref (patched reference + SPEC restatement), last timed step"}


# ------------------------------------------------------------- engine
def run_engine(args):
    import ctypes as C

    import torch

    from paper_2112_02958_b200 import capi, engine, modelgen

    dist, rank, ws = _dist()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    text = modelgen.config_program(3)
    cfg = capi.default_search_config(group_scopes=1)
    g = engine.Graph(text)
    eng = engine.Engine(g, device=local, cfg=cfg)
    B = args.batch
    K, W = args.steps, args.warmup
    maxd = cfg.max_decisions
    lib = g.lib
    stream = torch.cuda.current_stream(dev)
    sp = C.c_void_p(stream.cuda_stream)

    # inputs resident in HBM before timing: per-step seeds, empty prefixes
    base = 1_000_003 * (rank + 1)
    seeds = (torch.arange((K + W) * B, dtype=torch.int64, device=dev) + base).view(K + W, B)
    poff = torch.zeros(B + 1, dtype=torch.int32, device=dev)
    acts_out = torch.empty(B * maxd * 8, dtype=torch.uint8, device=dev)
    nacts = torch.empty(B, dtype=torch.int32, device=dev)
    res = torch.empty(B * C.sizeof(capi.PeResult), dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def step(i):
        # prefix = NULL: every prefix is empty (root rollouts; pe.h)
        eng.rollout_batch_device(None, poff.data_ptr(), seeds[i].data_ptr(), B,
                                 acts_out.data_ptr(), nacts.data_ptr(), res.data_ptr(),
                                 stream=sp)

    for i in range(W):
        flush.zero_()
        step(K + i)
    torch.cuda.synchronize(dev)
    launches0 = eng.launch_count()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    stops = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    eng.kernel_times(True)  # engine-side events around each main launch
    with ClockSampler(local) as clk:
        for i in range(K):
            flush.zero_()  # L2 flushed between timed iterations (outside the events)
            starts[i].record(stream)
            step(i)
            stops[i].record(stream)
        torch.cuda.synchronize(dev)
    kern_ms = eng.kernel_times(False)
    if dist:
        dist.barrier()
    launches = eng.launch_count() - launches0
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, stops)]
    total_ms = _max_over_ranks(dist, sum(step_ms), dev)
    value = ws * K * B / (total_ms / 1e3)

    # sanity: every candidate evaluated OK (numpy views of the pe_result
    # fields; no per-candidate Python objects, whose garbage collection
    # could land in the e2e timing below)
    import gc

    import numpy as np
    host = res.view(B, C.sizeof(capi.PeResult)).cpu().numpy()

    def field(name):
        f = getattr(capi.PeResult, name)
        return np.frombuffer(host[:, f.offset:f.offset + 4].tobytes(), dtype=np.int32)
    bad = int((field("status") != 0).sum())
    mean_steps = float(field("n_steps").mean())
    mean_ops = float(field("n_spmd_ops").mean())
    del host

    # parity sample: a strided sample of the LAST timed step's candidates
    # re-evaluated by the oracle (test infrastructure, off the timed path):
    # same seeds -> same action sequences and bit-exact results
    parity = None
    if rank == 0 and not args.no_parity_sample:
        parity = _parity_sample(text, cfg, seeds[K - 1].cpu().numpy(), acts_out, nacts, res, B,
                                maxd, args.parity_n)
    # the round-1 step size, same timing rules, device-timed only (after the
    # parity sample: it overwrites the output buffers): keeps the
    # number comparable across rounds (DESIGN.md §8 batch-size table)
    also = None
    B2 = args.also_batch
    if 0 < B2 < B:
        poff2 = poff[:B2 + 1]
        ms2 = []
        for i in range(W + K):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            eng.rollout_batch_device(None, poff2.data_ptr(), seeds[i].data_ptr(), B2,
                                     acts_out.data_ptr(), nacts.data_ptr(), res.data_ptr(), stream=sp)
            e1.record(stream)
            ms2.append((e0, e1))
        torch.cuda.synchronize(dev)
        t2 = _max_over_ranks(dist, sum(a.elapsed_time(b) for a, b in ms2[W:]), dev)
        also = {"candidates_per_step": B2, "value": ws * K * B2 / (t2 / 1e3), "ms_per_step": t2 / K,
                "note": "round-1 step size; device-timed, L2 flushed between steps"}

    gc.collect()

    # e2e: the public C-ABI with HOST buffers (pinned), copies inside the region
    e2e_k = max(1, min(K, 5))
    # each call's seeds prepared in pinned host memory before the region
    # (the inputs a caller hands over); the H2D copy is inside it
    pin_seeds_all = [(torch.arange(B, dtype=torch.int64) + base + 7_000_000 * (i + 1)).pin_memory()
                     for i in range(e2e_k)] + [torch.empty(B, dtype=torch.int64).pin_memory()]
    pin_poff = torch.zeros(B + 1, dtype=torch.int32).pin_memory()
    pin_acts = torch.empty(B * maxd * 8, dtype=torch.uint8).pin_memory()
    pin_nacts = torch.empty(B, dtype=torch.int32).pin_memory()
    pin_res = torch.empty(B * C.sizeof(capi.PeResult), dtype=torch.uint8).pin_memory()
    err = capi.PeError()
    h2d = B * 8 + pin_poff.numel() * 4
    d2h = None  # counted after the calls: the engine copies back only the action columns used

    def host_step(i):
        pin_seeds = pin_seeds_all[min(i, e2e_k)]
        rc = lib.pe_rollout_batch(eng.h, None, C.c_void_p(pin_poff.data_ptr()),
                                  C.c_void_p(pin_seeds.data_ptr()), B, C.c_void_p(pin_acts.data_ptr()),
                                  C.c_void_p(pin_nacts.data_ptr()), C.c_void_p(pin_res.data_ptr()),
                                  None, 0, sp, C.byref(err))
        assert rc == 0, err.message
        _ = pin_res[:8].numpy().tobytes()  # host read of the step's result

    pin_seeds_all[e2e_k].copy_(torch.arange(B, dtype=torch.int64) + base + 6_000_000)
    host_step(e2e_k)  # untimed warm-up: the engine's host-mode staging buffers are allocated
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for i in range(e2e_k):
        host_step(i)
    e2e_s = _max_over_ranks(dist, time.perf_counter() - t0, dev)
    kmax = int(pin_nacts.max().item())
    d2h = B * kmax * 8 + pin_nacts.numel() * 4 + pin_res.numel()  # acts columns, counts, results
    e2e = ws * e2e_k * B / e2e_s

    # roofline: algorithmic bytes per candidate
    A, N = g.n_args, g.n_ops
    s_graph = eng.graph_bytes()
    s_state = 8 * (A + N)
    s_io = C.sizeof(capi.PeResult) + 8 * maxd + 4 + 8 + 4
    b_cand = s_graph + 2 * s_state + s_io
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    # the dominant kernel's own duration: CUDA events the engine records
    # around its main rollout launch on the launching stream (pe.h
    # pe_engine_set_kernel_timing), averaged over the timed steps
    kern_s = sum(kern_ms) / 1e3 / K if kern_ms else sum(step_ms) / 1e3 / K
    achieved = b_cand * B / kern_s / 1e9
    # DRAM traffic of that kernel per launch, from the committed ncu --set
    # full capture of the same launch (tools/ncu_traffic.py); only when it
    # was captured at this batch size and engine build
    traffic, traffic_src = None, None
    tf = os.path.join(ROOT, "profiles", "r2_traffic.json")
    if os.path.exists(tf):
        try:
            t = json.load(open(tf))
            if int(t.get("candidates", -1)) == B:
                traffic = t["dram_bytes_read"] + t["dram_bytes_write"]
                traffic_src = t.get("source")
        except Exception:
            traffic = None

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        import helpers as H
        if os.path.exists(H.ORACLE_SO):
            threads = os.cpu_count() or 1
            n_cpu = 48 * threads  # ~12 s of reference CPU work on this path
            v_cpu, dt = cpu_reference(text, n_cpu, 30_000_000, threads)
            cpu = {"value": v_cpu, "unit": UNIT, "cores": threads, "cpu": _cpu_model(), "kind": "reference",
                   "sample": f"{n_cpu} rollouts of the bench workload ({dt:.1f} s)"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": K,
                "warmup": W, "ms_per_step": total_ms / K, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
                "config": _config(B, {"parallelism": f"candidate-parallel x{ws}",
                                      "l2": "256 MB flush between timed steps",
                                      "mean_decisions": round(mean_steps, 3),
                                      "mean_spmd_ops": round(mean_ops, 1),
                                      "arena_bytes": eng.arena_bytes(), "slots": eng.slots(),
                                      "failed_candidates": bad}),
                "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": d2h},
                "gpu_launches": launches,
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                             "frac": achieved / peak, "traffic": traffic,
                             "algorithmic_bytes_per_candidate": b_cand,
                             "kernel": "pe_rollout_kernel (main launch; engine-side CUDA events)",
                             "kernel_ms_per_launch": 1e3 * kern_s, "traffic_source": traffic_src,
                             "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback"},
                "cpu_baseline": cpu,
                "parity_sample": parity,
                "clocks": clk.summary(),
                "also_measured": also}
        print(json.dumps(line))
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


# ------------------------------------------------------------- search metric
SEARCH_METRIC = "search time to Megatron plan"


def _search_setup(layers=24):
    from paper_2112_02958_b200 import capi, engine, modelgen
    text = modelgen.config_program(3) if layers == 24 else modelgen.build_transformer(
        layers, mesh=(("batch", 4), ("model", 2)), **modelgen.GPT2_MEDIUM)
    g = engine.Graph(text)
    model = g.axis_index("model")
    # SURVEY.md §8(d) config 3 / DESIGN.md §5: model axis searched over the
    # parameters (scope groups), the batch axis a manual decision, memory
    # budget 0.6 x the replicated peak (the paper's regime)
    cfg = capi.default_search_config(group_scopes=1, scoped_only=1, auto_axes_mask=1 << model)
    return text, g, cfg, model


def _search_config(args, leaf_batch, episodes_to_found):
    return {"workload": "MCTS on gpt2-medium-24L [batch=4, model=2], model axis searched, "
                        "grouped parameters, budget 0.6 x replicated peak",
            "leaf_batch": leaf_batch, "seed": args.seed, "episodes_to_megatron": episodes_to_found,
            "megatron": "48 all_reduce / 0 all_gather on the model axis"}


def run_search(args):
    """BASELINE.json metric #2: wall-clock of the deterministic MCTS until its
    best plan carries the Megatron signature, on the GPU engine (pe_search;
    root-parallel pe_search_multi over NCCL under torchrun), next to the same
    search on the reference CPU path (oracle/_ref evaluating every leaf batch
    on all host threads).  Time = a re-run with the episode budget that first
    reached the plan (the search is deterministic per seed)."""
    from paper_2112_02958_b200 import capi, engine, search
    dist, rank, ws = _dist()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    text, g, cfg, model = _search_setup()
    lb = args.leaf_batch
    if args.impl == "reference":
        if rank != 0:
            return 0
        import helpers as H
        cp = capi.default_cost_params()
        cp.memory_budget_bytes = int(0.6 * H.oracle_info(text, cfg)["baseline_bytes"])
        ords = search.ordinal_actions(g, cfg)
        lw = (len(ords) - 1 + 63) // 64
        threads = os.cpu_count() or 1

        def ev(prefixes, seeds):
            return H.rollout_batch("oracle", text, prefixes, seeds, cfg, cp=cp, legal_words=lw,
                                   threads=threads)
        t0 = time.perf_counter()
        p = search.run_mcts(ev, len(ords) - 1, ords, episodes=args.search_episodes, seed=args.seed,
                            leaf_batch=lb)
        t_budget = time.perf_counter() - t0
        ok = search.megatron_signature(p.result, model, 24)
        budget = ((p.found_at_episode + lb) // lb) * lb
        t0 = time.perf_counter()
        search.run_mcts(ev, len(ords) - 1, ords, episodes=budget, seed=args.seed, leaf_batch=lb)
        t = time.perf_counter() - t0
        line = {"impl": "reference", "metric": SEARCH_METRIC, "value": t, "unit": "s",
                "n_gpus": args.gpus, "steps": 1, "warmup": 0, "ms_per_step": 1e3 * t,
                "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
                "dtype": "int64", "data": "synthetic",
                "config": _search_config(args, lb, budget), "megatron_found": bool(ok),
                "plan": search.plan_actions(p), "search_s_full_budget": t_budget,
                "cpu_baseline": {"value": t, "unit": "s", "cores": threads, "cpu": _cpu_model(), "kind": "reference",
                                 "sample": f"the full search to the plan ({budget} episodes)"},
                "e2e": {"value": t, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return 0
    import torch
    torch.cuda.set_device(local)
    base = engine.Engine(g, device=local, cfg=cfg).baseline_bytes
    cp = capi.default_cost_params()
    cp.memory_budget_bytes = int(0.6 * base)
    eng = engine.Engine(g, device=local, cfg=cfg, cost=cp)
    comm = search.NcclComm(ws, rank, local, dist) if ws > 1 else None
    launches0 = eng.launch_count()

    def run(episodes, seed):
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        if comm is not None:
            p = search.mcts_search_multi(eng, comm, episodes=episodes, seed=seed, leaf_batch=lb,
                                         merge_every=args.merge_every)
        else:
            p = search.mcts_search(eng, episodes=episodes, seed=seed, leaf_batch=lb)
        return p, _max_over_ranks(dist, time.perf_counter() - t0,
                                  torch.device("cuda", local) if dist else None)

    for w in range(args.warmup):  # warm-up searches (other seeds)
        run(lb, 10_000 + w)
    with ClockSampler(local) as clk:
        plan, t_budget = run(args.search_episodes, args.seed)
        ok = search.megatron_signature(plan.result, model, 24)
        budget = ((plan.found_at_episode + lb) // lb) * lb
        p2, t = run(budget, args.seed)
    same = search.plan_actions(p2) == search.plan_actions(plan)
    hits = eng.prefix_cache_stats()
    cpu = None
    if rank == 0 and not args.no_cpu_baseline and ws == 1:
        import helpers as H
        if os.path.exists(H.ORACLE_SO):
            ords = search.ordinal_actions(g, cfg)
            lw = (len(ords) - 1 + 63) // 64
            threads = os.cpu_count() or 1

            def ev(prefixes, seeds):
                return H.rollout_batch("oracle", text, prefixes, seeds, cfg, cp=cp,
                                       legal_words=lw, threads=threads)
            t0 = time.perf_counter()
            cp_plan = search.run_mcts(ev, len(ords) - 1, ords, episodes=budget, seed=args.seed,
                                      leaf_batch=lb)
            tc = time.perf_counter() - t0
            cpu = {"value": tc, "unit": "s", "cores": threads, "cpu": _cpu_model(), "kind": "reference",
                   "sample": f"the same search ({budget} episodes, leaf batch {lb})",
                   "plan_identical": search.plan_actions(cp_plan) == search.plan_actions(plan)}
    if comm is not None:
        comm.close()
    if rank == 0:
        line = {"metric": SEARCH_METRIC, "value": t, "unit": "s", "n_gpus": ws, "steps": 1,
                "warmup": args.warmup, "ms_per_step": 1e3 * t, "higher_is_better": False,
                "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
                "config": dict(_search_config(args, lb, budget),
                               parallelism=f"root-parallel x{ws} (NCCL merge every "
                                           f"{args.merge_every} episodes)" if ws > 1 else "1 tree"),
                "megatron_found": bool(ok), "replay_identical": bool(same),
                "plan": search.plan_actions(plan), "found_at_episode": plan.found_at_episode,
                "search_s_full_budget": t_budget, "episodes_per_s_full_budget":
                    args.search_episodes / t_budget,
                "prefix_cache": hits, "gpu_launches": eng.launch_count() - launches0,
                "e2e": {"value": t, "unit": "s", "h2d_bytes_per_step": None,
                        "d2h_bytes_per_step": None,
                        "note": "the search API is host-level: every leaf batch's prefixes and "
                                "seeds go H2D and results D2H inside the timed search"},
                "cpu_baseline": cpu, "clocks": clk.summary()}
        print(json.dumps(line))
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


# ------------------------------------------------------------- config 4 sweep
def _cpu_worker(text, k, seed0, q):
    import helpers as H
    from paper_2112_02958_b200 import capi
    cfg = capi.default_search_config(group_scopes=1)
    i = 0
    while True:
        H.rollout_batch("oracle", text, [[]], [seed0 + k * 1_000_000 + i], cfg, threads=1)
        q.put(k)
        i += 1


def cpu_capped(text, cap_s, threads, seed0):
    """Reference CPU rollouts, one candidate stream per host core (one
    process each), stopped hard after `cap_s` seconds (SURVEY.md §8(d):
    time-capped; a config-4 candidate takes longer than any bounded sample on
    this path).  Returns (completed candidates, seconds)."""
    import multiprocessing as mpr
    ctx = mpr.get_context("fork")
    q = ctx.Queue()
    procs = [ctx.Process(target=_cpu_worker, args=(text, k, seed0, q), daemon=True)
             for k in range(threads)]
    t0 = time.perf_counter()
    for p in procs:
        p.start()
    done = 0
    while time.perf_counter() - t0 < cap_s:
        try:
            q.get(timeout=max(0.05, cap_s - (time.perf_counter() - t0)))
            done += 1
        except Exception:
            pass
    dt = time.perf_counter() - t0
    for p in procs:
        p.kill()
        p.join()
    return done, dt


def run_sweep(args):
    """BASELINE.json configs[3] / SURVEY.md §8(d) config 4: batched
    candidate evaluation at 1K..1M candidates per launch on the 48-layer
    training-step graph (52,154 ops, 1,156 arguments), mesh [batch=4,
    model=2], grouped worklist.  One JSON line; `value` is the largest size's
    device-timed rate, `sweep` has every size."""
    import ctypes as C

    import torch

    from paper_2112_02958_b200 import capi, engine, modelgen
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    text = modelgen.config_program(4)
    cfg = capi.default_search_config(group_scopes=1)
    g = engine.Graph(text)
    eng = engine.Engine(g, device=0, cfg=cfg)
    maxd = cfg.max_decisions
    st = torch.cuda.current_stream(dev)
    sp = C.c_void_p(st.cuda_stream)
    b_cand = eng.graph_bytes() + 2 * 8 * (g.n_args + g.n_ops) + C.sizeof(capi.PeResult) + 8 * maxd + 16
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    sizes = [int(x) for x in args.sizes.split(",")]
    rows = []
    base = 40_000_000
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    with ClockSampler(0) as clk:
        for B in sizes:
            seeds = torch.arange(B, dtype=torch.int64, device=dev)
            poff = torch.zeros(B + 1, dtype=torch.int32, device=dev)
            acts = torch.empty(B * maxd * 8, dtype=torch.uint8, device=dev)
            na = torch.empty(B, dtype=torch.int32, device=dev)
            res = torch.empty(B * C.sizeof(capi.PeResult), dtype=torch.uint8, device=dev)
            ms = []
            for rep in range(args.warmup + args.steps):
                seeds.add_(base)  # fresh candidates every call
                base += B
                flush.zero_()
                torch.cuda.synchronize(dev)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                eng.rollout_batch_device(None, poff.data_ptr(), seeds.data_ptr(), B, acts.data_ptr(),
                                         na.data_ptr(), res.data_ptr(), stream=sp)
                e1.record(st)
                torch.cuda.synchronize(dev)
                if rep >= args.warmup:
                    ms.append(e0.elapsed_time(e1))
            t = sum(ms) / len(ms)
            cps = B / t * 1e3
            import numpy as np
            host = res.view(B, C.sizeof(capi.PeResult)).cpu().numpy().view(np.int32)
            f = lambda name: host[:, getattr(capi.PeResult, name).offset // 4]  # noqa: E731
            rows.append({"candidates": B, "ms_per_launch": t, "cand_per_s": cps,
                         "roofline_frac": cps * b_cand / 1e9 / peak,
                         "failed": int((f("status") != 0).sum()),
                         "mean_decisions": float(f("n_steps").mean()),
                         "mean_spmd_ops": float(f("n_spmd_ops").mean())})
            print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
    top = rows[-1]
    # second variant: MCTS leaf evaluation = a
    # parent state + 1 action.  Parents: 2-decision prefixes of the last
    # batch's rollouts, held as pe_state handles; candidates: every legal
    # action of every parent, evaluated from the parent's state
    # (pe_eval_from_states) and, for comparison, by full replay from the
    # untiled graph (pe_eval_batch); the two must agree bit-for-bit.
    import numpy as np
    a_host = acts.view(sizes[-1], maxd, 8).cpu().numpy()
    n_host = na.cpu().numpy()
    parents, seen = [], set()
    for i in range(sizes[-1]):
        if n_host[i] >= 3:
            v = a_host[i].view(np.uint32)[:, 0]
            pre = tuple((int(v[k]), int(a_host[i, k, 4]), int(a_host[i, k, 5]), int(a_host[i, k, 6]))
                        for k in range(2))
            if pre not in seen:
                seen.add(pre)
                parents.append(list(pre))
        if len(parents) >= args.p1_parents:
            break
    cands_p, cands_a = [], []
    for pre in parents:
        st = eng.state(pre)
        _, _, legal = eng.rollout_batch([pre + [(0, 0, 0, capi.PE_ACT_STOP)]], [0], legal=True)
        for o in range(eng.n_ordinals):
            if (legal[0][o // 64] >> (o % 64)) & 1:
                a = eng.ordinal_action(o)
                cands_p.append(st)
                cands_a.append([(a.value, a.dim, a.axis, a.kind)])
    eng.eval_from_states(cands_p[:64], cands_a[:64])  # warm-up
    t0 = time.perf_counter()
    inc = eng.eval_from_states(cands_p, cands_a)
    t_inc = time.perf_counter() - t0
    t0 = time.perf_counter()
    full = eng.eval_batch([p.seq + a for p, a in zip(cands_p, cands_a)])
    t_full = time.perf_counter() - t0
    import helpers as H
    p1 = {"parents": len(parents), "candidates": len(cands_a),
          "cand_per_s_from_parent_state": len(cands_a) / t_inc,
          "cand_per_s_full_replay": len(cands_a) / t_full,
          "mismatches_vs_full_replay": sum(1 for x, y in zip(inc, full) if H.compare_results(x, y)),
          "timing": "host C-ABI calls (pe_eval_from_states / pe_eval_batch), copies included"}
    print(json.dumps(p1), file=sys.stderr, flush=True)
    # e2e: host buffers through the C-ABI at the largest size (copies timed)
    B = sizes[-1]
    t0 = time.perf_counter()
    eng.rollout_roots_np(__import__("numpy").arange(B, dtype="uint64") + base)
    e2e = B / (time.perf_counter() - t0)
    cpu = None
    if not args.no_cpu_baseline:
        import helpers as H
        if os.path.exists(H.ORACLE_SO):
            threads = os.cpu_count() or 1
            done, dt = cpu_capped(text, args.cpu_cap_s, threads, 90_000_000)
            cpu = {"value": done / dt, "unit": UNIT, "cores": threads, "cpu": _cpu_model(), "kind": "reference",
                   "sample": f"root rollouts, one stream per core, stopped hard at "
                             f"{args.cpu_cap_s:.0f} s: {done} completed in {dt:.0f} s",
                   "completed": done, "note": "an upper bound when 0 completed; see "
                   "profiles/r2_cfg4_cpu_baseline.json for the long capped run and its "
                   "extrapolation"}
    line = {"metric": METRIC, "value": top["cand_per_s"], "unit": UNIT, "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": top["ms_per_launch"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic",
            "config": {"workload": "config 4: 48-layer training step (52,154 ops, 1,156 args), "
                                   "mesh [batch=4, model=2], grouped worklist, root rollouts",
                       "graph_ops": g.n_ops, "graph_args": g.n_args, "sizes": sizes,
                       "arena_bytes": eng.arena_bytes(), "slots": eng.slots(),
                       "arena_caps": eng.arena_caps(),
                       "l2": "256 MB flush before every launch"},
            "sweep": rows, "parent_plus_one": p1,
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": B * 8 + (B + 1) * 4,
                    "d2h_bytes_per_step": B * (maxd * 8 + 4 + C.sizeof(capi.PeResult))},
            "roofline": {"bound": "hbm", "achieved": top["cand_per_s"] * b_cand / 1e9, "peak": peak,
                         "unit": "GB/s", "frac": top["roofline_frac"], "traffic": None,
                         "algorithmic_bytes_per_candidate": b_cand, "kernel": "pe_rollout_kernel"},
            "cpu_baseline": cpu, "clocks": clk.summary()}
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    # >= the engine's resident slots (148 SMs x 32 warps x 32 lanes = 151,552)
    ap.add_argument("--batch", type=int, default=1048576,
                    help="rollouts per step (about 7 waves of the config-3 slots)")
    ap.add_argument("--also-batch", type=int, default=262144,
                    help="also time this step size (round 1's), device-timed; 0 = off")
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity-sample", action="store_true")
    ap.add_argument("--parity-n", type=int, default=128)
    ap.add_argument("--config", type=int, default=3,
                    help="3: the headline (GPT-2-medium 24L rollouts); 4: the 1K..1M sweep")
    ap.add_argument("--sizes", default="1024,4096,16384,65536",
                    help="config 4 sweep sizes (candidates per launch)")
    ap.add_argument("--p1-parents", type=int, default=64,
                    help="config 4: parent states of the parent + 1 action variant")
    ap.add_argument("--cpu-cap-s", type=float, default=60.0,
                    help="config 4: per-thread cap of the reference CPU sample")
    ap.add_argument("--metric", default="candidates", choices=["candidates", "search"],
                    help="candidates: cand/s (headline); search: search time to the Megatron plan")
    ap.add_argument("--leaf-batch", type=int, default=256)
    ap.add_argument("--search-episodes", type=int, default=2048)
    ap.add_argument("--merge-every", type=int, default=256)
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    if args.metric == "search":
        return run_search(args)
    if args.config == 4:
        if args.impl == "reference":
            print(json.dumps({"impl": "reference", "unavailable": "config 4 reference timing is the "
                              "capped run in profiles/r2_cfg4_cpu_baseline.json"}))
            return 0
        return run_sweep(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_engine(args)


if __name__ == "__main__":
    sys.exit(main())
