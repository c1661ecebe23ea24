#!/usr/bin/env python3
"""Config 4 (BASELINE.json configs[3]): batched candidate-evaluation sweep on
the 48-layer training-step graph (52,154 ops, 1,156 arguments), mesh
[batch=4, model=2], grouped worklist; batches of rollouts of increasing size,
device-timed, with the algorithmic-bytes roofline fraction.

  python tools/sweep_bench.py [--sizes 1024,4096,16384] [--cfg 4]
"""
import argparse
import ctypes as C
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2112_02958_b200 import capi, engine, modelgen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1024,4096,16384")
    ap.add_argument("--cfg", type=int, default=4)
    ap.add_argument("--reps", type=int, default=3,
                    help="calls per size; the last is reported (the scheduling trie warms up)")
    args = ap.parse_args()
    text = modelgen.config_program(args.cfg)
    g = engine.Graph(text)
    eng = engine.Engine(g, cfg=capi.default_search_config(group_scopes=1))
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    maxd = 32
    b_cand = eng.graph_bytes() + 2 * 8 * (g.n_args + g.n_ops) + 192 + 8 * maxd + 16
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream()
    sp = C.c_void_p(st.cuda_stream)
    out = {"config": args.cfg, "ops": g.n_ops, "args": g.n_args, "slots": eng.slots(),
           "arena_bytes_per_candidate": eng.arena_bytes(), "algorithmic_bytes_per_candidate": b_cand,
           "rows": []}
    for B in [int(x) for x in args.sizes.split(",")]:
        seeds = torch.arange(B, dtype=torch.int64, device=dev) + 777
        poff = torch.zeros(B + 1, dtype=torch.int32, device=dev)
        acts = torch.empty(B * maxd * 8, dtype=torch.uint8, device=dev)
        na = torch.empty(B, dtype=torch.int32, device=dev)
        res = torch.empty(B * 192, dtype=torch.uint8, device=dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for rep in range(args.reps):
            seeds += B  # fresh candidates every call
            torch.cuda.synchronize()
            e0.record(st)
            eng.rollout_batch_device(None, poff.data_ptr(), seeds.data_ptr(), B, acts.data_ptr(),
                                     na.data_ptr(), res.data_ptr(), stream=sp)
            e1.record(st)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
        host = res.view(B, 192).cpu().numpy()
        rs = [capi.PeResult.from_buffer_copy(host[i].tobytes()) for i in range(B)]
        cps = B / ms * 1e3
        out["rows"].append({"candidates": B, "ms": ms, "cand_per_s": cps,
                            "achieved_GBps": cps * b_cand / 1e9,
                            "roofline_frac": cps * b_cand / 1e9 / peak,
                            "failed": sum(r.status != 0 for r in rs),
                            "mean_decisions": sum(r.n_steps for r in rs) / B,
                            "mean_spmd_ops": sum(r.n_spmd_ops for r in rs) / B})
        print(json.dumps(out["rows"][-1]), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
