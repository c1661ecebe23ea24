"""ctypes mirror of include/pe.h — the C-ABI structs and the product library
loader.

The product library is ``paper_2112_02958_b200/libpe_b200.so`` (built by
``__graft_entry__.build()`` with nvcc for sm_100a).  There is no CPU
fallback: if the library is missing, ``load()`` raises.
"""
from __future__ import annotations

import ctypes as C
import os

PE_MAX_AXES = 4
PE_MAX_RANK = 4

PE_OK = 0
PE_ERR_PARSE = 1
PE_ERR_VALIDATION = 2
PE_ERR_ILLEGAL = 3
PE_ERR_INVALID_ARGUMENT = 4
PE_ERR_CUDA = 5
PE_ERR_NO_DEVICE = 6
PE_ERR_CAPACITY = 7
PE_ERR_INTERNAL = 70

PE_ACT_TILE = 0
PE_ACT_TILE_GROUP = 1
PE_ACT_INFER_REST = 2
PE_ACT_STOP = 3

PE_CAND_OK = 0
PE_CAND_ILLEGAL = 1
PE_CAND_INTERNAL = 2
PE_CAND_CAPACITY = 3
PE_CAND_PAUSED = 4

PE_MEM_DEVICE = 1
PE_SYNC = 2

PE_ACT_FLAG_INFERRED = 1
PE_ACT_FLAG_EXPANDED = 2

TRACE_KIND_ALL_REDUCE = 22
TRACE_KIND_ALL_GATHER = 23
TRACE_KIND_SLICE_BY_COORD = 24


class PeError(C.Structure):
    _fields_ = [("code", C.c_int32), ("line", C.c_int32), ("column", C.c_int32),
                ("message", C.c_char * 500)]


class PeAction(C.Structure):
    _fields_ = [("value", C.c_uint32), ("dim", C.c_uint8), ("axis", C.c_uint8),
                ("kind", C.c_uint8), ("pad", C.c_uint8)]


class PeResult(C.Structure):
    _fields_ = [
        ("peak_bytes", C.c_int64), ("flops", C.c_int64),
        ("reduction_bytes", C.c_int64), ("baseline_bytes", C.c_int64),
        ("ar_bytes", C.c_int64 * PE_MAX_AXES), ("ag_bytes", C.c_int64 * PE_MAX_AXES),
        ("ar_cnt", C.c_int32 * PE_MAX_AXES), ("ag_cnt", C.c_int32 * PE_MAX_AXES),
        ("sbc_cnt", C.c_int32 * PE_MAX_AXES),
        ("n_spmd_ops", C.c_int32), ("n_stuck", C.c_int32), ("n_steps", C.c_int32),
        ("status", C.c_int32), ("fail_step", C.c_int32), ("feasible", C.c_int32),
        ("reserved", C.c_int32), ("reserved2", C.c_int32),
        ("runtime_s", C.c_double), ("reward", C.c_double),
    ]


class PeCostParams(C.Structure):
    _fields_ = [("memory_budget_bytes", C.c_int64), ("flops_per_second", C.c_double),
                ("bytes_per_second", C.c_double), ("collective_latency_s", C.c_double),
                ("w_mem", C.c_double), ("w_comm", C.c_double), ("w_steps", C.c_double)]


class PeSearchConfig(C.Structure):
    _fields_ = [("auto_axes_mask", C.c_uint32), ("max_decisions", C.c_uint32),
                ("group_scopes", C.c_uint32), ("episodes", C.c_uint32),
                ("seed", C.c_uint64), ("uct_c", C.c_double),
                ("leaf_batch", C.c_uint32), ("scoped_only", C.c_uint32),
                ("resurface_stuck", C.c_uint32),
                ("worklist_args", C.POINTER(C.c_uint32)), ("n_worklist_args", C.c_uint32),
                ("infer_rest_action", C.c_uint32)]

    def restrict_worklist(self, args) -> "PeSearchConfig":
        """Restrict the static worklist to these argument indices (ranker
        top-k); the array is kept alive by this config object."""
        arr = (C.c_uint32 * max(1, len(args)))(*args)
        self._worklist_keep = arr
        self.worklist_args = C.cast(arr, C.POINTER(C.c_uint32))
        self.n_worklist_args = len(args)
        return self


class PeArgDesc(C.Structure):
    _fields_ = [("id", C.c_char_p), ("scope", C.c_char_p), ("rank", C.c_int32),
                ("shape", C.c_int64 * PE_MAX_RANK)]


class PeOpDesc(C.Structure):
    _fields_ = [("id", C.c_char_p), ("kind", C.c_int32), ("rank", C.c_int32),
                ("shape", C.c_int64 * PE_MAX_RANK), ("n_operands", C.c_int32),
                ("operands", C.POINTER(C.c_int32)), ("n_batch", C.c_int32),
                ("n_contract", C.c_int32), ("lhs_batch", C.c_int32 * PE_MAX_RANK),
                ("rhs_batch", C.c_int32 * PE_MAX_RANK), ("lhs_contract", C.c_int32 * PE_MAX_RANK),
                ("rhs_contract", C.c_int32 * PE_MAX_RANK), ("n_dims", C.c_int32),
                ("dims", C.c_int32 * PE_MAX_RANK), ("start", C.c_int64 * PE_MAX_RANK),
                ("limit", C.c_int64 * PE_MAX_RANK), ("dim", C.c_int32), ("value", C.c_double),
                ("scope", C.c_char_p)]


PE_PLAN_MAX_ACTIONS = 64


class PePlan(C.Structure):
    _fields_ = [("actions", PeAction * PE_PLAN_MAX_ACTIONS), ("n_actions", C.c_uint32),
                ("episodes", C.c_uint32), ("found_at_episode", C.c_uint32),
                ("winner_rank", C.c_uint32), ("seed", C.c_uint64), ("result", PeResult)]


class PeMctsParams(C.Structure):
    _fields_ = [("n_ordinals", C.c_uint32), ("max_decisions", C.c_uint32),
                ("episodes", C.c_uint32), ("leaf_batch", C.c_uint32),
                ("merge_every", C.c_uint32), ("rank", C.c_uint32), ("seed", C.c_uint64),
                ("uct_c", C.c_double)]


MERGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_int64), C.c_uint32, C.c_int32)
ROLLOUT_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32,
                         C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p)

assert C.sizeof(PeAction) == 8
assert C.sizeof(PeResult) == 192, C.sizeof(PeResult)


def default_cost_params() -> PeCostParams:
    return PeCostParams(16 << 30, 1e14, 1e11, 1e-6, 0.1, 1.0, 0.01)


def default_search_config(**kw) -> PeSearchConfig:
    c = PeSearchConfig(0xFFFFFFFF, 32, 1, 500, 0, 1.414, 8192, 0, 0, None, 0, 0)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


# symbol -> (restype, argtypes) for every function include/pe.h declares
_P = C.c_void_p
SIGNATURES = {
    "pe_default_cost_params": (None, [C.POINTER(PeCostParams)]),
    "pe_default_search_config": (None, [C.POINTER(PeSearchConfig)]),
    "pe_graph_create": (C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(_P), C.POINTER(PeError)]),
    "pe_graph_create_from_arrays": (C.c_int, [C.c_char_p, C.c_int32, C.POINTER(C.c_char_p),
                                              C.POINTER(C.c_int64), C.c_int32,
                                              C.POINTER(PeArgDesc), C.c_int32,
                                              C.POINTER(PeOpDesc), C.c_int32, C.POINTER(_P),
                                              C.POINTER(PeError)]),
    "pe_graph_destroy": (None, [_P]),
    "pe_graph_axis_name": (C.c_int32, [_P, C.c_int32, C.c_char_p, C.c_int32]),
    "pe_graph_num_args": (C.c_int32, [_P]),
    "pe_graph_num_ops": (C.c_int32, [_P]),
    "pe_graph_num_axes": (C.c_int32, [_P]),
    "pe_graph_num_operands": (C.c_int32, [_P]),
    "pe_graph_axis_size": (C.c_int64, [_P, C.c_int32]),
    "pe_graph_value_index": (C.c_int32, [_P, C.c_char_p]),
    "pe_graph_axis_index": (C.c_int32, [_P, C.c_char_p]),
    "pe_graph_value_name": (C.c_int32, [_P, C.c_int32, C.c_char_p, C.c_int32]),
    "pe_graph_value_shape": (C.c_int32, [_P, C.c_int32, C.POINTER(C.c_int64)]),
    "pe_graph_arg_scope": (C.c_int32, [_P, C.c_int32, C.c_char_p, C.c_int32]),
    "pe_graph_num_groups": (C.c_int32, [_P]),
    "pe_graph_group_size": (C.c_int32, [_P, C.c_int32]),
    "pe_graph_group_member": (C.c_int32, [_P, C.c_int32, C.c_int32]),
    "pe_engine_create": (C.c_int, [_P, C.POINTER(PeSearchConfig), C.POINTER(PeCostParams),
                                   C.c_int32, C.POINTER(_P), C.POINTER(PeError)]),
    "pe_engine_destroy": (None, [_P]),
    "pe_eval_batch": (C.c_int, [_P, _P, _P, C.c_uint32, _P, _P, C.c_uint32, C.c_uint32, _P,
                                C.POINTER(PeError)]),
    "pe_rollout_batch": (C.c_int, [_P, _P, _P, _P, C.c_uint32, _P, _P, _P, _P, C.c_uint32, _P,
                                   C.POINTER(PeError)]),
    "pe_eval_batch_ex": (C.c_int, [_P, _P, _P, C.c_uint32, _P, _P, C.c_uint32, _P, C.c_uint32,
                                   _P, C.POINTER(PeError)]),
    "pe_infer_rest": (C.c_int, [_P, _P, C.c_uint32, _P, C.c_uint32, C.POINTER(C.c_uint32),
                                C.POINTER(PeError)]),
    "pe_engine_num_ordinals": (C.c_uint32, [_P]),
    "pe_engine_legal_words": (C.c_uint32, [_P]),
    "pe_engine_ordinal_action": (C.c_int, [_P, C.c_uint32, C.POINTER(PeAction)]),
    "pe_engine_baseline_bytes": (C.c_int64, [_P]),
    "pe_engine_arena_bytes": (C.c_int64, [_P]),
    "pe_engine_slots": (C.c_uint32, [_P]),
    "pe_engine_arena_caps": (None, [_P, C.POINTER(C.c_int32)]),
    "pe_engine_set_kernel_timing": (None, [_P, C.c_int32]),
    "pe_engine_kernel_times": (C.c_uint32, [_P, C.POINTER(C.c_float), C.c_uint32]),
    "pe_engine_launch_count": (C.c_uint64, [_P]),
    "pe_engine_sched_nodes": (C.c_int64, [_P]),
    "pe_engine_set_state_reuse": (C.c_int, [_P, C.c_double]),
    "pe_engine_graph_bytes": (C.c_int64, [_P]),
    "pe_engine_set_prefix_cache": (C.c_int, [_P, C.c_double]),
    "pe_engine_prefix_cache_stats": (None, [_P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                            C.POINTER(C.c_int64)]),
    "pe_state_create": (C.c_int, [_P, _P, C.c_uint32, C.POINTER(_P), C.POINTER(PeError)]),
    "pe_state_destroy": (None, [_P]),
    "pe_state_num_decisions": (C.c_uint32, [_P]),
    "pe_state_result": (C.c_int, [_P, C.POINTER(PeResult)]),
    "pe_state_specs": (C.c_int, [_P, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                                 C.POINTER(C.c_int32), C.c_uint32, C.POINTER(C.c_uint32),
                                 C.POINTER(PeError)]),
    "pe_search_multi": (C.c_int, [_P, C.POINTER(PeSearchConfig), C.c_uint32, _P,
                                  C.POINTER(PePlan), C.POINTER(PeError)]),
    "pe_nccl_unique_id": (C.c_int, [_P, C.POINTER(PeError)]),
    "pe_nccl_comm_create": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, C.POINTER(_P),
                                      C.POINTER(PeError)]),
    "pe_nccl_comm_destroy": (None, [_P]),
    "pe_eval_from_states": (C.c_int, [_P, _P, _P, _P, C.c_uint32, _P, _P, C.POINTER(PeError)]),
    "pe_mcts_run": (C.c_int, [C.POINTER(PeMctsParams), ROLLOUT_FN, _P, MERGE_FN, _P, _P,
                              C.POINTER(PePlan), C.POINTER(PeError)]),
    "pe_search": (C.c_int, [_P, C.POINTER(PeSearchConfig), C.c_uint32, C.c_uint32, MERGE_FN,
                            _P, C.POINTER(PePlan), C.POINTER(PeError)]),
}

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpe_b200.so")
_lib = None


def load(path: str | None = None) -> C.CDLL:
    """Load the product library (nvcc-built, sm_100a).  Raises if missing."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or os.environ.get("PE_LIB") or LIB_PATH  # PE_LIB: a debug build
    if not os.path.exists(p):
        raise RuntimeError(
            f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the engine has no CPU fallback)")
    lib = C.CDLL(p)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def actions_array(seqs):
    """List of action lists -> (PeAction array, uint32 offsets array)."""
    flat = [a for s in seqs for a in s]
    acts = (PeAction * max(1, len(flat)))()
    for i, a in enumerate(flat):
        acts[i] = a if isinstance(a, PeAction) else PeAction(*a)
    off = (C.c_uint32 * (len(seqs) + 1))()
    n = 0
    for i, s in enumerate(seqs):
        off[i] = n
        n += len(s)
    off[len(seqs)] = n
    return acts, off


def result_dict(r: PeResult, n_axes: int = PE_MAX_AXES) -> dict:
    return {
        "peak_bytes": r.peak_bytes, "flops": r.flops, "reduction_bytes": r.reduction_bytes,
        "baseline_bytes": r.baseline_bytes,
        "ar_bytes": list(r.ar_bytes)[:n_axes], "ag_bytes": list(r.ag_bytes)[:n_axes],
        "ar_cnt": list(r.ar_cnt)[:n_axes], "ag_cnt": list(r.ag_cnt)[:n_axes],
        "sbc_cnt": list(r.sbc_cnt)[:n_axes], "n_spmd_ops": r.n_spmd_ops,
        "n_stuck": r.n_stuck, "n_steps": r.n_steps, "status": r.status,
        "fail_step": r.fail_step, "feasible": r.feasible, "runtime_s": r.runtime_s,
        "reward": r.reward,
    }
