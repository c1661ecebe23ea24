"""The C-ABI library loads, exports every symbol include/pe.h declares, parses
and validates graphs on the host, and refuses to run without a device."""
import ctypes as C
import os
import re

import pytest

from paper_2112_02958_b200 import capi, engine, modelgen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "pe.h")).read()
    return sorted(set(re.findall(r"^\s*(?:pe_status|void|int32_t|int64_t|uint32_t|uint64_t)\s+(pe_\w+)\(",
                                 text, re.M)))


def test_every_header_symbol_is_exported():
    lib = capi.load()
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
        assert s in capi.SIGNATURES, s


def test_graph_parse_and_tables():
    g = engine.Graph(modelgen.config_program(2))
    assert g.n_args == 7 and g.n_ops == 43 and g.n_axes == 1
    assert g.names[0] == "x" and g.shapes[g.value_index("l0_wq")] == [8, 2, 4]
    assert len(g.groups) == 7


def test_parse_errors_map_to_reference_errors():
    with pytest.raises(engine.ParseError) as e:
        engine.Graph("func @f(%x: f32[4]) -> f32[4] { %y = dot(%x) : f32[4] return %y ")
    with pytest.raises(engine.ValidationError):
        engine.Graph("func @f(%x: f32[4]) -> f32[4] { %y = add(%x, %z) : f32[4]\n return %y }")
    with pytest.raises(engine.ValidationError):
        engine.Graph("func @f(%x: f32[8,64]) -> f32[8,65] { %y = reshape(%x) : f32[8,65]\n return %y }")
    g = engine.Graph("func @id(%x: f32[4]) -> f32[4] { return %x }")
    assert g.n_ops == 0
    # dims and axis sizes must fit int32 (the engine's value records)
    with pytest.raises(engine.Error, match="exceeds 2\\^31-1"):
        engine.Graph("func @f(%x: f32[4294967296]) -> f32[4294967296] { return %x }")


def test_engine_refuses_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    g = engine.Graph(modelgen.linear())
    with pytest.raises(engine.NoDeviceError):
        engine.Engine(g)
