"""mcts_search / emit_plan (SPEC search module) over the engine's C-ABI.

* ``mcts_search(engine, ...)``      leaf-parallel MCTS on one GPU (pe_search):
                                     every leaf batch is one rollout launch.
* root-parallel over N GPUs: each rank runs ``mcts_search`` with its own
  engine and ``merge=TorchMerge()``; root visit / value statistics (int64 N,
  2^-32 fixed-point W) are all-reduced every ``merge_every`` episodes through
  torch.distributed (NCCL over NVLink on GPUs, gloo in the CPU tests).  No
  other data crosses ranks.
* ``run_mcts(evaluate, ...)``       the same search loop (pe_mcts_run) over any
                                     evaluator callback — used by the tests to
                                     run the search on the CPU oracle.
* ``emit_plan``                      the SPEC plan JSON (args / output specs,
                                     actions, cost, seed, episodes).
"""
from __future__ import annotations

import ctypes as C
import json

from . import capi
from .capi import PeAction, PeError, PeMctsParams, PePlan


class TorchMerge:
    """pe_merge_fn over torch.distributed: op 0 = SUM, op 1 = MAX."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        if device is None:
            device = ("cuda" if dist.get_backend(group) == "nccl" else "cpu")
        self.device = device
        self.torch = torch
        self.calls = 0

        def _merge(_user, values, n, op):
            try:
                t = self.torch.tensor([values[i] for i in range(n)], dtype=self.torch.int64,
                                      device=self.device)
                red = self.dist.ReduceOp.SUM if op == 0 else self.dist.ReduceOp.MAX
                self.dist.all_reduce(t, op=red, group=self.group)
                host = t.cpu().tolist()
                for i in range(n):
                    values[i] = host[i]
                self.calls += 1
                return 0
            except Exception:  # pragma: no cover - reported as a status
                return 1

        self.fn = capi.MERGE_FN(_merge)


def _null_merge():
    return C.cast(None, capi.MERGE_FN)


def mcts_search(engine, episodes=500, seed=0, leaf_batch=8192, uct_c=1.414, merge=None,
                merge_every=0, rank=0) -> PePlan:
    cfg = capi.PeSearchConfig()
    C.memmove(C.byref(cfg), C.byref(engine.cfg), C.sizeof(cfg))
    cfg.episodes = episodes
    cfg.seed = seed
    cfg.leaf_batch = leaf_batch
    cfg.uct_c = uct_c
    plan = PePlan()
    err = PeError()
    mfn = merge.fn if merge is not None else _null_merge()
    rc = engine.lib.pe_search(engine.h, C.byref(cfg), merge_every if merge else 0, rank, mfn, None,
                              C.byref(plan), C.byref(err))
    if rc != capi.PE_OK:
        from .engine import _raise
        _raise(rc, err)
    return plan


class NcclComm:
    """An NCCL communicator made by the engine library (pe_nccl_comm_create):
    rank 0's unique id travels over `dist` (any torch.distributed backend),
    or no exchange at all when nranks == 1."""

    def __init__(self, nranks: int, rank: int, device: int, dist=None):
        self.lib = capi.load()
        uid = (C.c_uint8 * 128)()
        err = PeError()
        if rank == 0:
            rc = self.lib.pe_nccl_unique_id(uid, C.byref(err))
            if rc != capi.PE_OK:
                raise RuntimeError(err.message.decode())
        if nranks > 1:
            import torch
            t = torch.tensor(list(uid), dtype=torch.uint8)
            if dist.get_backend() == "nccl":
                t = t.cuda()
            dist.broadcast(t, 0)
            for i, x in enumerate(t.cpu().tolist()):
                uid[i] = x
        h = C.c_void_p()
        rc = self.lib.pe_nccl_comm_create(uid, nranks, rank, device, C.byref(h), C.byref(err))
        if rc != capi.PE_OK:
            raise RuntimeError(err.message.decode())
        self.h = h

    def close(self):
        if self.h:
            self.lib.pe_nccl_comm_destroy(self.h)
            self.h = None


def mcts_search_multi(engine, comm: NcclComm, episodes=500, seed=0, leaf_batch=8192, uct_c=1.414,
                      merge_every=256) -> PePlan:
    """Root-parallel mcts_search over NCCL (pe.h pe_search_multi): the root
    statistics are all-reduced on the device every `merge_every` episodes."""
    cfg = capi.PeSearchConfig()
    C.memmove(C.byref(cfg), C.byref(engine.cfg), C.sizeof(cfg))
    cfg.episodes = episodes
    cfg.seed = seed
    cfg.leaf_batch = leaf_batch
    cfg.uct_c = uct_c
    plan = PePlan()
    err = PeError()
    rc = engine.lib.pe_search_multi(engine.h, C.byref(cfg), merge_every, comm.h, C.byref(plan),
                                    C.byref(err))
    if rc != capi.PE_OK:
        from .engine import _raise
        _raise(rc, err)
    return plan


def run_mcts(evaluate, n_ordinals, ordinal_actions, episodes=500, seed=0, leaf_batch=256,
             uct_c=1.414, max_decisions=32, merge=None, merge_every=0, rank=0, lib=None) -> PePlan:
    """pe_mcts_run with a Python evaluator.  `evaluate(prefixes, seeds)`
    returns (results, action_seqs, legal_bitmasks) like Engine.rollout_batch."""
    lib = lib or capi.load()
    lw = (n_ordinals + 63) // 64

    def _eval(_user, prefix, poff, seeds, n, acts_out, nacts_out, out, legal_out):
        try:
            po = C.cast(poff, C.POINTER(C.c_uint32))
            pa = C.cast(prefix, C.POINTER(PeAction))
            sd = C.cast(seeds, C.POINTER(C.c_uint64))
            prefixes = [[(pa[k].value, pa[k].dim, pa[k].axis, pa[k].kind)
                         for k in range(po[i], po[i + 1])] for i in range(n)]
            res, seqs, legal = evaluate(prefixes, [sd[i] for i in range(n)])
            ao = C.cast(acts_out, C.POINTER(PeAction))
            no = C.cast(nacts_out, C.POINTER(C.c_uint32))
            ro = C.cast(out, C.POINTER(capi.PeResult))
            lo = C.cast(legal_out, C.POINTER(C.c_uint64))
            for i in range(n):
                ro[i] = res[i]
                no[i] = len(seqs[i])
                for k, a in enumerate(seqs[i]):
                    ao[i * max_decisions + k] = PeAction(*a, 0) if len(a) == 4 else a
                for w in range(lw):
                    lo[i * lw + w] = legal[i][w]
            return 0
        except Exception:  # pragma: no cover
            import traceback
            traceback.print_exc()
            return 1

    efn = capi.ROLLOUT_FN(_eval)
    p = PeMctsParams(n_ordinals, max_decisions, episodes, leaf_batch,
                     merge_every if merge else 0, rank, seed, uct_c)
    ords = (PeAction * (n_ordinals + 1))(*ordinal_actions)
    plan = PePlan()
    err = PeError()
    mfn = merge.fn if merge is not None else _null_merge()
    rc = lib.pe_mcts_run(C.byref(p), efn, None, mfn, None, ords, C.byref(plan), C.byref(err))
    if rc != capi.PE_OK:
        raise RuntimeError(f"pe_mcts_run failed rc={rc}: {err.message.decode()}")
    return plan


def ordinal_actions(graph, cfg) -> list:
    """Decode every TileValue ordinal (entry x dim x auto axis) plus Stop,
    exactly as pe_engine_ordinal_action does (no device needed)."""
    auto = [a for a in range(graph.n_axes) if (cfg.auto_axes_mask >> a) & 1]
    if cfg.group_scopes:  # (action value, members): group index
        entries = list(enumerate(graph.groups))
    else:                 # argument index
        entries = [(a, [a]) for a in range(graph.n_args)]
    if cfg.scoped_only:
        entries = [(v, m) for v, m in entries if graph.scopes[m[0]]]
    if cfg.worklist_args:  # ranker top-k (pe.h worklist_args)
        keep = {cfg.worklist_args[i] for i in range(cfg.n_worklist_args)}
        entries = [(v, m) for v, m in entries if keep & set(m)]
    kind = capi.PE_ACT_TILE_GROUP if cfg.group_scopes else capi.PE_ACT_TILE
    out = []
    for val, _mem in entries:
        for d in range(capi.PE_MAX_RANK):
            for ax in auto:
                out.append(PeAction(val, d, ax, kind, 0))
    if getattr(cfg, "resurface_stuck", 0):
        # one block per op for stuck nodes that resurface: TileValue(op result)
        for o in range(graph.n_ops):
            for d in range(capi.PE_MAX_RANK):
                for ax in auto:
                    out.append(PeAction(graph.n_args + o, d, ax, capi.PE_ACT_TILE, 0))
    if getattr(cfg, "infer_rest_action", 0):
        # InferRest follows every TileValue ordinal (pe.h infer_rest_action)
        out.append(PeAction(0, 0, 0, capi.PE_ACT_INFER_REST, 0))
    out.append(PeAction(0, 0, 0, capi.PE_ACT_STOP, 0))
    return out


def plan_actions(plan: PePlan):
    return [(plan.actions[k].value, plan.actions[k].dim, plan.actions[k].axis,
             plan.actions[k].kind) for k in range(plan.n_actions)]


def _spec_json(word: int, rank: int, axes):
    dims = []
    for d in range(rank):
        a = (word >> (4 * d)) & 0xF
        dims.append(axes[a - 1] if a else None)
    pend = [axes[i] for i in range(len(axes)) if (word >> (16 + i)) & 1]
    return {"dims": dims, "pending_sum": pend}


def emit_plan(engine, plan: PePlan) -> str:
    """SPEC emit_plan: {"args": {id: spec}, "output": spec, "actions": [...],
    "cost": {...}, "seed", "episodes"} — specs from the engine's own trace of
    the plan (the exact lowering the cost was computed on)."""
    g = engine.graph
    axes = g.axis_names
    acts = [PeAction(*a, 0) for a in plan_actions(plan)]
    (res,), (tr,) = engine.eval_batch([acts], trace_words=1 << 16)
    n_args = tr[1]
    args = {}
    for i in range(n_args):
        args[g.names[i]] = _spec_json(tr[2 + i], len(g.shapes[i]), axes)
    out_word = tr[2 + n_args]
    actions = []
    for a in acts:
        if a.kind == capi.PE_ACT_TILE_GROUP:
            members = [g.names[m] for m in g.groups[a.value]]
            actions.append({"tile_group": members, "dim": a.dim, "axis": axes[a.axis]})
        elif a.kind == capi.PE_ACT_TILE:
            actions.append({"tile": g.names[a.value], "dim": a.dim, "axis": axes[a.axis]})
        elif a.kind == capi.PE_ACT_INFER_REST:
            actions.append({"infer_rest": True})
    d = {"args": args, "output": _spec_json(out_word, (out_word >> 24) & 7, axes),
         "actions": actions, "cost": capi.result_dict(res, g.n_axes), "seed": plan.seed,
         "episodes": plan.episodes, "found_at_episode": plan.found_at_episode}
    return json.dumps(d, sort_keys=True)


def plan_actions_from_json(engine, text: str) -> list:
    """The action sequence of an emitted plan (SPEC: "replayable"): the
    inverse of emit_plan's "actions" list, for pe_eval_batch."""
    g = engine.graph
    out = []
    for a in json.loads(text)["actions"]:
        if "infer_rest" in a:
            out.append(PeAction(0, 0, 0, capi.PE_ACT_INFER_REST, 0))
        elif "tile_group" in a:
            grp = g.group_of(g.value_index(a["tile_group"][0]))
            out.append(PeAction(grp, a["dim"], g.axis_index(a["axis"]), capi.PE_ACT_TILE_GROUP, 0))
        else:
            out.append(PeAction(g.value_index(a["tile"]), a["dim"], g.axis_index(a["axis"]),
                                capi.PE_ACT_TILE, 0))
    return out


def megatron_signature(res, model_axis: int, layers: int) -> bool:
    """2 all_reduce on the model axis per layer, 0 all_gather
    on the model axis."""
    return res.ar_cnt[model_axis] == 2 * layers and res.ag_cnt[model_axis] == 0
