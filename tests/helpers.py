"""Test-side loaders: the parity oracle (oracle/_ref/liboracle.so), the
host-compiled core harness (tests/native) and the product library.

TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's
baseline legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

from paper_2112_02958_b200 import capi
from paper_2112_02958_b200.capi import PeAction, PeResult, PeSearchConfig, PeCostParams

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "_ref",
                         "liboracle_asan.so" if os.environ.get("PE_ASAN") else "liboracle.so")
# PE_ASAN=1: AddressSanitizer + UBSan builds of the host harness (with arena
# bounds checks) and of the oracle (tests/test_asan.py runs them)
HARNESS_SO = os.path.join(ROOT, "tests", "native", "_build",
                          "libpe_host_harness_asan.so" if os.environ.get("PE_ASAN")
                          else "libpe_host_harness.so")
SAN_FLAGS = ["-fsanitize=address,undefined", "-fno-omit-frame-pointer", "-DPE_BOUNDS_CHECK"]

_P = C.c_void_p


def build_harness() -> str:
    src = [os.path.join(ROOT, "tests", "native", "pe_host_harness.cc"),
           os.path.join(ROOT, "paper_2112_02958_b200", "csrc", "pe_graph.cc"),
           os.path.join(ROOT, "paper_2112_02958_b200", "csrc", "pe_pir.cc")]
    hdrs = [os.path.join(ROOT, "paper_2112_02958_b200", "csrc", h)
            for h in ("pe_core.cuh", "pe_graph.h", "pe_graph_view.h", "pe_rules.h")]
    hdrs.append(os.path.join(ROOT, "include", "pe.h"))
    if os.path.exists(HARNESS_SO):
        t = os.path.getmtime(HARNESS_SO)
        if all(os.path.getmtime(f) < t for f in src + hdrs):
            return HARNESS_SO
    os.makedirs(os.path.dirname(HARNESS_SO), exist_ok=True)
    subprocess.check_call(["g++", "-std=c++17", "-O2", "-g", "-fPIC", "-shared",
                           *(SAN_FLAGS if os.environ.get("PE_ASAN") else []),
                           "-I", os.path.join(ROOT, "include"),
                           "-I", os.path.join(ROOT, "paper_2112_02958_b200", "csrc"),
                           *src, "-o", HARNESS_SO])
    return HARNESS_SO


def build_oracle() -> str:
    if not os.path.exists(ORACLE_SO):
        target = ["asan"] if os.environ.get("PE_ASAN") else []
        subprocess.check_call(["make", "-C", os.path.join(ROOT, "oracle"), "-j8", *target])
    return ORACLE_SO


_oracle = None
_harness = None


def oracle():
    global _oracle
    if _oracle is None:
        lib = C.CDLL(ORACLE_SO)
        lib.oracle_eval_batch.restype = C.c_int
        lib.oracle_eval_batch.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(PeSearchConfig),
                                          C.POINTER(PeCostParams), _P, _P, C.c_uint32, _P, _P,
                                          C.c_uint32, C.c_int, C.c_char_p, C.c_size_t]
        lib.oracle_rollout_batch.restype = C.c_int
        lib.oracle_rollout_batch.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(PeSearchConfig),
                                             C.POINTER(PeCostParams), _P, _P, _P, C.c_uint32,
                                             _P, _P, _P, _P, C.c_int, C.c_char_p, C.c_size_t]
        lib.oracle_info.restype = C.c_int
        lib.oracle_info.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(PeSearchConfig), _P,
                                    C.c_char_p, C.c_size_t]
        lib.oracle_legal.restype = C.c_int
        lib.oracle_legal.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(PeSearchConfig), _P,
                                     C.c_uint32, _P, C.c_uint32, _P, C.c_char_p, C.c_size_t]
        lib.oracle_check_equivalence.restype = C.c_int
        lib.oracle_check_equivalence.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(PeSearchConfig),
                                                 _P, C.c_uint32, C.c_int, C.c_uint64, _P, _P, _P,
                                                 C.c_char_p, C.c_size_t]
        lib.oracle_debug_text.restype = C.c_int
        lib.oracle_debug_text.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(PeSearchConfig), _P,
                                          C.c_uint32, C.c_char_p, C.c_size_t]
        _oracle = lib
    return _oracle


def harness():
    global _harness
    if _harness is None:
        lib = C.CDLL(build_harness())
        lib.harness_eval_batch.restype = C.c_int
        lib.harness_eval_batch.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(PeSearchConfig),
                                           C.POINTER(PeCostParams), _P, _P, C.c_uint32, _P, _P,
                                           C.c_uint32, C.c_char_p, C.c_size_t]
        lib.harness_rollout_batch.restype = C.c_int
        lib.harness_rollout_batch.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(PeSearchConfig),
                                              C.POINTER(PeCostParams), _P, _P, _P, C.c_uint32,
                                              _P, _P, _P, _P, C.c_char_p, C.c_size_t]
        _harness = lib
    return _harness


def _cfg(cfg):
    return cfg if cfg is not None else capi.default_search_config()


def eval_batch(which: str, text: str, seqs, cfg=None, cp=None, trace_words=0, threads=1):
    """Evaluate action sequences with 'oracle' or 'harness'.  Returns
    (list[PeResult], trace list or None)."""
    b = text.encode()
    acts, off = capi.actions_array(seqs)
    n = len(seqs)
    out = (PeResult * n)()
    tr = (C.c_int32 * (n * trace_words))() if trace_words else None
    err = C.create_string_buffer(512)
    cfg = _cfg(cfg)
    cp = cp if cp is not None else capi.default_cost_params()
    if which == "oracle":
        rc = oracle().oracle_eval_batch(b, len(b), C.byref(cfg), C.byref(cp), acts, off, n, out,
                                        tr, trace_words, threads, err, 512)
    else:
        rc = harness().harness_eval_batch(b, len(b), C.byref(cfg), C.byref(cp), acts, off, n, out,
                                          tr, trace_words, err, 512)
    if rc:
        raise RuntimeError(f"{which} eval failed rc={rc}: {err.value.decode()}")
    traces = None
    if tr is not None:
        traces = [list(tr[i * trace_words:(i + 1) * trace_words]) for i in range(n)]
    return list(out), traces


def rollout_batch(which: str, text: str, prefixes, seeds, cfg, cp=None, legal_words=0, threads=1):
    b = text.encode()
    acts, off = capi.actions_array(prefixes)
    n = len(prefixes)
    maxd = cfg.max_decisions
    sd = (C.c_uint64 * n)(*seeds)
    aout = (PeAction * (n * maxd))()
    nout = (C.c_uint32 * n)()
    out = (PeResult * n)()
    legal = (C.c_uint64 * (n * legal_words))() if legal_words else None
    err = C.create_string_buffer(512)
    cp = cp if cp is not None else capi.default_cost_params()
    if which == "oracle":
        rc = oracle().oracle_rollout_batch(b, len(b), C.byref(cfg), C.byref(cp), acts, off, sd, n,
                                           aout, nout, out, legal, threads, err, 512)
    else:
        rc = harness().harness_rollout_batch(b, len(b), C.byref(cfg), C.byref(cp), acts, off, sd,
                                             n, aout, nout, out, legal, err, 512)
    if rc:
        raise RuntimeError(f"{which} rollout failed rc={rc}: {err.value.decode()}")
    seqs = [[(aout[i * maxd + k].value, aout[i * maxd + k].dim, aout[i * maxd + k].axis,
              aout[i * maxd + k].kind) for k in range(nout[i])] for i in range(n)]
    legal_l = None
    if legal is not None:
        legal_l = [list(legal[i * legal_words:(i + 1) * legal_words]) for i in range(n)]
    return list(out), seqs, legal_l


def oracle_info(text: str, cfg=None):
    b = text.encode()
    out = (C.c_int64 * 4)()
    err = C.create_string_buffer(512)
    cfg = _cfg(cfg)
    rc = oracle().oracle_info(b, len(b), C.byref(cfg), out, err, 512)
    if rc:
        raise RuntimeError(err.value.decode())
    return {"baseline_bytes": out[0], "n_groups": out[1], "n_ordinals": out[2], "n_entries": out[3]}


def oracle_legal(text: str, seq, cfg=None):
    b = text.encode()
    acts, off = capi.actions_array([seq])
    ords = (C.c_uint32 * 65536)()
    n = C.c_uint32(0)
    err = C.create_string_buffer(512)
    cfg = _cfg(cfg)
    rc = oracle().oracle_legal(b, len(b), C.byref(cfg), acts, len(seq), ords, 65536, C.byref(n),
                               err, 512)
    if rc:
        raise RuntimeError(f"rc={rc} {err.value.decode()}")
    return list(ords[:n.value])


def oracle_check_equivalence(text: str, seq, trials=5, seed=0, cfg=None):
    """Reference interpreter check of the plan `seq` (REF interp.cc:640-678).
    Returns (pass, max_abs_diff, order_preserving)."""
    b = text.encode()
    acts, _ = capi.actions_array([seq])
    mx = C.c_double(0)
    ok = C.c_int(0)
    op = C.c_int(0)
    err = C.create_string_buffer(512)
    rc = oracle().oracle_check_equivalence(b, len(b), C.byref(_cfg(cfg)), acts, len(seq), trials,
                                           seed, C.byref(mx), C.byref(ok), C.byref(op), err, 512)
    if rc:
        raise RuntimeError(f"rc={rc} {err.value.decode()}")
    return bool(ok.value), mx.value, bool(op.value)


def oracle_debug(text: str, seq, cfg=None) -> str:
    b = text.encode()
    acts, off = capi.actions_array([seq])
    out = C.create_string_buffer(1 << 20)
    oracle().oracle_debug_text(b, len(b), C.byref(_cfg(cfg)), acts, len(seq), out, 1 << 20)
    return out.value.decode()


RESULT_INT_FIELDS = ("peak_bytes", "flops", "reduction_bytes", "baseline_bytes", "n_spmd_ops",
                     "n_stuck", "n_steps", "status", "fail_step", "feasible")


def compare_results(a: PeResult, b: PeResult, rtol=1e-6):
    """Bit-exact on integer fields; <= rtol relative on runtime and reward."""
    diffs = []
    for f in RESULT_INT_FIELDS:
        if getattr(a, f) != getattr(b, f):
            diffs.append((f, getattr(a, f), getattr(b, f)))
    for f in ("ar_bytes", "ag_bytes", "ar_cnt", "ag_cnt", "sbc_cnt"):
        if list(getattr(a, f)) != list(getattr(b, f)):
            diffs.append((f, list(getattr(a, f)), list(getattr(b, f))))
    for f in ("runtime_s", "reward"):
        x, y = getattr(a, f), getattr(b, f)
        if abs(x - y) > rtol * max(abs(x), abs(y), 1e-300):
            diffs.append((f, x, y))
    return diffs
