"""Host-side mirror of the reference interface for the candidate-evaluation
path, over the C-ABI of include/pe.h.

Reference API (REF = /root/reference/proj)        this module
------------------------------------------------   ---------------------------
parse_program(text)          parser.h:28           Graph(text)
apply_tile_action(p,v,d,ax)  rewrite.h:33-34       action tuples (value, dim, axis)
propagate(p)                 propagate.h:54        } applied after every action
lower_to_spmd(p)             spmd.h:67             } inside Engine.eval_batch,
collective_stats(sp)         spmd.h:87             } batched on the GPU
peak_liveness/comm_cost/runtime_estimate/reward    (SPEC cost module)
MCTS rollouts                (SPEC mcts_search)    Engine.rollout_batch
Errors: Error/ParseError/ValidationError/IllegalActionError/InternalError
(error.h:25-60) are raised with the same names; per-candidate
IllegalActionError/InternalError become a status in the result record.

The engine is GPU-only: constructing an Engine without a CUDA device raises
NoDeviceError — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C

from . import capi
from .capi import PeAction, PeError, PeResult


class Error(RuntimeError):
    pass


class ParseError(Error):
    def __init__(self, msg, line=0, column=0):
        super().__init__(msg)
        self.line = line
        self.column = column


class ValidationError(Error):
    pass


class IllegalActionError(Error):
    pass


class InternalError(Error):
    pass


class NoDeviceError(Error):
    pass


def _raise(rc: int, err: PeError):
    msg = err.message.decode(errors="replace")
    if rc == capi.PE_ERR_PARSE:
        raise ParseError(msg, err.line, err.column)
    if rc == capi.PE_ERR_VALIDATION:
        raise ValidationError(msg)
    if rc == capi.PE_ERR_ILLEGAL:
        raise IllegalActionError(msg)
    if rc == capi.PE_ERR_NO_DEVICE:
        raise NoDeviceError(msg)
    if rc == capi.PE_ERR_INTERNAL:
        raise InternalError(msg)
    raise Error(f"pe error {rc}: {msg}")


class Graph:
    """A parsed, validated and compiled program (parse_program)."""

    def __init__(self, text: str | None, _handle=None):
        self.lib = capi.load()
        self.text = text
        if _handle is None:
            b = text.encode()
            h = C.c_void_p()
            err = PeError()
            rc = self.lib.pe_graph_create(b, len(b), C.byref(h), C.byref(err))
            if rc != capi.PE_OK:
                _raise(rc, err)
        else:
            h = _handle
        self.h = h
        L = self.lib
        self.n_args = L.pe_graph_num_args(h)
        self.n_ops = L.pe_graph_num_ops(h)
        self.n_axes = L.pe_graph_num_axes(h)
        buf = C.create_string_buffer(1024)
        self.names = []
        self.shapes = []
        dims = (C.c_int64 * 4)()
        for v in range(self.n_args + self.n_ops):
            L.pe_graph_value_name(h, v, buf, 1024)
            self.names.append(buf.value.decode())
            r = L.pe_graph_value_shape(h, v, dims)
            self.shapes.append([dims[i] for i in range(r)])
        self.axis_sizes = [L.pe_graph_axis_size(h, a) for a in range(self.n_axes)]
        self.scopes = []
        for a in range(self.n_args):
            L.pe_graph_arg_scope(h, a, buf, 1024)
            self.scopes.append(buf.value.decode())
        self.axis_names = []
        for a in range(self.n_axes):
            L.pe_graph_axis_name(h, a, buf, 1024)
            self.axis_names.append(buf.value.decode())
        self.groups = [[L.pe_graph_group_member(h, g, i) for i in range(L.pe_graph_group_size(h, g))]
                       for g in range(L.pe_graph_num_groups(h))]
        self._index = {n: i for i, n in enumerate(self.names)}

    @classmethod
    def from_arrays(cls, name, axes, args, ops, result):
        """Structured construction (pe_graph_create_from_arrays): `axes` =
        [(name, size)], `args` = [(id, shape, scope)], `ops` = [dict(id, kind,
        shape, operands, batch=([],[]), contract=([],[]), dims=[], start=[],
        limit=[], dim=-1, value=0.0, scope="")], `result` = value index."""
        lib = capi.load()
        keep = []
        names = (C.c_char_p * max(1, len(axes)))(*[a[0].encode() for a in axes])
        sizes = (C.c_int64 * max(1, len(axes)))(*[a[1] for a in axes])
        ad = (capi.PeArgDesc * max(1, len(args)))()
        for i, (aid, shape, scope) in enumerate(args):
            ad[i].id = aid.encode()
            ad[i].scope = scope.encode() if scope else None
            ad[i].rank = len(shape)
            for d, x in enumerate(shape):
                ad[i].shape[d] = x
        od = (capi.PeOpDesc * max(1, len(ops)))()
        for i, o in enumerate(ops):
            d = od[i]
            d.id = o["id"].encode()
            d.kind = o["kind"]
            d.rank = len(o["shape"])
            for k, x in enumerate(o["shape"]):
                d.shape[k] = x
            opn = (C.c_int32 * max(1, len(o["operands"])))(*o["operands"])
            keep.append(opn)
            d.n_operands = len(o["operands"])
            d.operands = C.cast(opn, C.POINTER(C.c_int32))
            lb, rb = o.get("batch", ([], []))
            lc, rc_ = o.get("contract", ([], []))
            d.n_batch, d.n_contract = len(lb), len(lc)
            for k in range(len(lb)):
                d.lhs_batch[k], d.rhs_batch[k] = lb[k], rb[k]
            for k in range(len(lc)):
                d.lhs_contract[k], d.rhs_contract[k] = lc[k], rc_[k]
            dims = o.get("dims", [])
            d.n_dims = len(dims)
            for k, x in enumerate(dims):
                d.dims[k] = x
            for k, x in enumerate(o.get("start", [])):
                d.start[k] = x
            for k, x in enumerate(o.get("limit", [])):
                d.limit[k] = x
            d.dim = o.get("dim", -1)
            d.value = o.get("value", 0.0)
            d.scope = o["scope"].encode() if o.get("scope") else None
        h = C.c_void_p()
        err = PeError()
        rc = lib.pe_graph_create_from_arrays(name.encode(), len(axes), names, sizes, len(args),
                                             ad, len(ops), od, result, C.byref(h), C.byref(err))
        if rc != capi.PE_OK:
            _raise(rc, err)
        return cls(None, _handle=h)

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.lib.pe_graph_destroy(h)
            self.h = None

    def value_index(self, name: str) -> int:
        return self._index[name]

    def axis_index(self, name: str) -> int:
        i = self.lib.pe_graph_axis_index(self.h, name.encode())
        if i < 0:
            raise IllegalActionError(f'axis "{name}" is not declared')
        return i

    def group_of(self, arg: int) -> int:
        for g, m in enumerate(self.groups):
            if arg in m:
                return g
        raise KeyError(arg)

    def action(self, value, dim: int, axis, group: bool = False) -> PeAction:
        v = value if isinstance(value, int) else self.value_index(value)
        ax = axis if isinstance(axis, int) else self.axis_index(axis)
        if group:
            return PeAction(self.group_of(v), dim, ax, capi.PE_ACT_TILE_GROUP, 0)
        return PeAction(v, dim, ax, capi.PE_ACT_TILE, 0)

    def actions(self, seq, group: bool = False):
        return [self.action(*a, group=group) if not isinstance(a, PeAction) else a for a in seq]


class Engine:
    """Per-device batched candidate evaluator."""

    def __init__(self, graph: Graph, device: int = 0, cfg=None, cost=None):
        self.lib = graph.lib
        self.graph = graph
        self.cfg = cfg if cfg is not None else capi.default_search_config()
        self.cost = cost if cost is not None else capi.default_cost_params()
        h = C.c_void_p()
        err = PeError()
        rc = self.lib.pe_engine_create(graph.h, C.byref(self.cfg), C.byref(self.cost), device,
                                       C.byref(h), C.byref(err))
        if rc != capi.PE_OK:
            _raise(rc, err)
        self.h = h
        self.device = device
        self.n_ordinals = self.lib.pe_engine_num_ordinals(h)
        self.legal_words = self.lib.pe_engine_legal_words(h)
        self.baseline_bytes = self.lib.pe_engine_baseline_bytes(h)

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.lib.pe_engine_destroy(h)
            self.h = None

    def launch_count(self) -> int:
        return int(self.lib.pe_engine_launch_count(self.h))

    def sched_nodes(self) -> int:
        """Prefix states in the scheduling trie (pe.h pe_engine_sched_nodes)."""
        return int(self.lib.pe_engine_sched_nodes(self.h))

    def set_state_reuse(self, budget_gb: float) -> None:
        """Opt into prefix-state reuse (pe.h pe_engine_set_state_reuse)."""
        rc = self.lib.pe_engine_set_state_reuse(self.h, float(budget_gb))
        if rc != capi.PE_OK:
            raise Error(f"pe_engine_set_state_reuse failed rc={rc}")

    def set_prefix_cache(self, budget_gb: float) -> None:
        """Incremental leaf evaluation (pe.h pe_engine_set_prefix_cache)."""
        rc = self.lib.pe_engine_set_prefix_cache(self.h, float(budget_gb))
        if rc != capi.PE_OK:
            raise Error(f"pe_engine_set_prefix_cache failed rc={rc}")

    def prefix_cache_stats(self):
        h, s, n = C.c_uint64(), C.c_uint64(), C.c_int64()
        self.lib.pe_engine_prefix_cache_stats(self.h, C.byref(h), C.byref(s), C.byref(n))
        return {"hits": h.value, "saved": s.value, "entries": n.value}

    def state(self, seq) -> "State":
        """A propagated state after `seq` (pe_state_create)."""
        return State(self, seq)

    def eval_from_states(self, parents, seqs):
        """candidate c = parents[c] (State or None) + seqs[c] (pe_eval_from_states)."""
        acts, off = capi.actions_array(seqs)
        n = len(seqs)
        ps = (C.c_void_p * max(1, n))(*[p.h if p is not None else None for p in parents])
        out = (PeResult * n)()
        err = PeError()
        rc = self.lib.pe_eval_from_states(self.h, ps, acts, off, n, out, None, C.byref(err))
        if rc != capi.PE_OK:
            _raise(rc, err)
        return list(out)

    def graph_bytes(self) -> int:
        return int(self.lib.pe_engine_graph_bytes(self.h))

    def arena_bytes(self) -> int:
        return int(self.lib.pe_engine_arena_bytes(self.h))

    def kernel_times(self, on: bool):
        """Main-launch durations (ms) since the last call, then timing on/off
        (pe_engine_set_kernel_timing / pe_engine_kernel_times)."""
        buf = (C.c_float * 4096)()
        n = self.lib.pe_engine_kernel_times(self.h, buf, 4096)
        self.lib.pe_engine_set_kernel_timing(self.h, 1 if on else 0)
        return [buf[i] for i in range(min(n, 4096))]

    def arena_caps(self) -> dict:
        c = (C.c_int32 * 5)()
        self.lib.pe_engine_arena_caps(self.h, c)
        return dict(zip(("values", "loops", "front", "spmd_ops", "operand_refs"), list(c)))

    def slots(self) -> int:
        return int(self.lib.pe_engine_slots(self.h))

    def ordinal_action(self, ordinal: int) -> PeAction:
        a = PeAction()
        rc = self.lib.pe_engine_ordinal_action(self.h, ordinal, C.byref(a))
        if rc:
            raise IndexError(ordinal)
        return a

    # ---- host-buffer entry points (the e2e path) ----
    def eval_batch(self, seqs, trace_words: int = 0):
        acts, off = capi.actions_array(seqs)
        n = len(seqs)
        out = (PeResult * n)()
        tr = (C.c_int32 * (n * trace_words))() if trace_words else None
        err = PeError()
        rc = self.lib.pe_eval_batch(self.h, acts, off, n, out, tr, trace_words, 0, None,
                                    C.byref(err))
        if rc != capi.PE_OK:
            _raise(rc, err)
        res = list(out)
        if trace_words:
            return res, [list(tr[i * trace_words:(i + 1) * trace_words]) for i in range(n)]
        return res

    def rollout_batch(self, prefixes, seeds, legal: bool = False):
        acts, off = capi.actions_array(prefixes)
        n = len(prefixes)
        maxd = self.cfg.max_decisions
        sd = (C.c_uint64 * n)(*seeds)
        aout = (PeAction * (n * maxd))()
        nout = (C.c_uint32 * n)()
        out = (PeResult * n)()
        lg = (C.c_uint64 * (n * self.legal_words))() if legal else None
        err = PeError()
        rc = self.lib.pe_rollout_batch(self.h, acts, off, sd, n, aout, nout, out, lg, 0, None,
                                       C.byref(err))
        if rc != capi.PE_OK:
            _raise(rc, err)
        seqs = [[(aout[i * maxd + k].value, aout[i * maxd + k].dim, aout[i * maxd + k].axis,
                  aout[i * maxd + k].kind) for k in range(nout[i])] for i in range(n)]
        lgl = None
        if legal:
            lgl = [list(lg[i * self.legal_words:(i + 1) * self.legal_words]) for i in range(n)]
        return list(out), seqs, lgl

    def rollout_roots_np(self, seeds):
        """Root rollouts (every prefix empty) for a large batch, through the
        host-buffer C-ABI, returned as numpy arrays: results (n, 192) uint8
        (raw pe_result records), actions (n, max_decisions, 4) uint32 as
        (value, dim, axis, kind) and n_acts (n,) uint32.  Action rows past
        n_acts are unspecified (pe.h)."""
        import numpy as np
        seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
        n = int(seeds.shape[0])
        maxd = self.cfg.max_decisions
        poff = np.zeros(n + 1, dtype=np.uint32)
        aout = np.zeros((n, maxd, 8), dtype=np.uint8)
        nout = np.zeros(n, dtype=np.uint32)
        out = np.zeros((n, C.sizeof(PeResult)), dtype=np.uint8)
        err = PeError()
        p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        rc = self.lib.pe_rollout_batch(self.h, None, p(poff), p(seeds), n, p(aout), p(nout),
                                       p(out), None, 0, None, C.byref(err))
        if rc != capi.PE_OK:
            _raise(rc, err)
        v = aout.view(np.uint32)[..., 0]
        acts = np.stack([v, aout[..., 4], aout[..., 5], aout[..., 6]], axis=-1).astype(np.uint32)
        return out, acts, nout

    def infer_rest(self, prefix):
        """infer_rest (REF propagate.cc:484-544) after `prefix`: returns
        prefix + [INFER_REST marker] + inferred TILE actions."""
        acts, _ = capi.actions_array([prefix])
        cap = len(prefix) + 1 + self.graph.n_args
        out = (PeAction * cap)()
        n = C.c_uint32(0)
        err = PeError()
        rc = self.lib.pe_infer_rest(self.h, acts, len(prefix), out, cap, C.byref(n), C.byref(err))
        if rc != capi.PE_OK:
            _raise(rc, err)
        return [out[i] for i in range(n.value)]

    # ---- device-buffer entry points (inputs already resident in HBM) ----
    def rollout_batch_device(self, prefix_ptr, poff_ptr, seeds_ptr, n, acts_out_ptr,
                             nacts_out_ptr, out_ptr, legal_ptr=None, stream=None, sync=False):
        err = PeError()
        flags = capi.PE_MEM_DEVICE | (capi.PE_SYNC if sync else 0)
        rc = self.lib.pe_rollout_batch(self.h, prefix_ptr, poff_ptr, seeds_ptr, n, acts_out_ptr,
                                       nacts_out_ptr, out_ptr, legal_ptr, flags, stream,
                                       C.byref(err))
        if rc != capi.PE_OK:
            _raise(rc, err)

    def eval_batch_device(self, acts_ptr, off_ptr, n, out_ptr, stream=None, sync=False):
        err = PeError()
        flags = capi.PE_MEM_DEVICE | (capi.PE_SYNC if sync else 0)
        rc = self.lib.pe_eval_batch(self.h, acts_ptr, off_ptr, n, out_ptr, None, 0, flags, stream,
                                    C.byref(err))
        if rc != capi.PE_OK:
            _raise(rc, err)


class State:
    """A propagated partitioning state held on the device (pe.h pe_state):
    the decisions, their evaluation, per-argument / result specs and the
    stuck list (pe_state_specs)."""

    def __init__(self, eng: Engine, seq):
        self.eng = eng
        self.lib = eng.lib
        acts, _ = capi.actions_array([seq])
        h = C.c_void_p()
        err = PeError()
        rc = self.lib.pe_state_create(eng.h, acts, len(seq), C.byref(h), C.byref(err))
        if rc != capi.PE_OK:
            _raise(rc, err)
        self.h = h
        self.seq = list(seq)

    def result(self) -> PeResult:
        r = PeResult()
        self.lib.pe_state_result(self.h, C.byref(r))
        return r

    def specs(self):
        """(arg spec words, result spec word, [(op, reason)] stuck list)."""
        A = self.eng.graph.n_args
        args = (C.c_uint32 * max(1, A))()
        res = C.c_uint32()
        cap = 4 * (self.eng.graph.n_ops + 1)
        stk = (C.c_int32 * (2 * cap))()
        ns = C.c_uint32()
        err = PeError()
        rc = self.lib.pe_state_specs(self.h, args, C.byref(res), stk, cap, C.byref(ns), C.byref(err))
        if rc != capi.PE_OK:
            _raise(rc, err)
        return list(args)[:A], res.value, [(stk[2 * i], stk[2 * i + 1]) for i in range(ns.value)]

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.lib.pe_state_destroy(h)
            self.h = None


def describe(r: PeResult) -> str:
    return (f"status={r.status} peak={r.peak_bytes} ar={list(r.ar_cnt)}/{list(r.ar_bytes)} "
            f"ag={list(r.ag_cnt)}/{list(r.ag_bytes)} sbc={list(r.sbc_cnt)} steps={r.n_steps} "
            f"stuck={r.n_stuck} ops={r.n_spmd_ops} runtime={r.runtime_s:.6g} reward={r.reward:.9f}")
