"""The graph boundary (pe_graph_create / pe_graph_create_from_arrays,
replacing REF parse_program parser.h:28 + validate): both entry points give
the same compiled graph; syntax errors map to ParseError with a position,
shape errors to ValidationError (REF error.h:28-46)."""
import re

import pytest

import fuzz_util as F
import pir_arrays
from paper_2112_02958_b200 import engine, modelgen


def _programs():
    yield modelgen.linear()
    for c in (1, 2, 3):
        yield modelgen.config_program(c)
    yield modelgen.build_training_step(2, mesh=(("batch", 2), ("model", 2)), **modelgen.TOY)
    for i in range(12):
        yield modelgen.random_program(500 + i, F.MESHES[i % 3])


def _same(a, b):
    assert (a.n_args, a.n_ops, a.n_axes) == (b.n_args, b.n_ops, b.n_axes)
    assert a.names == b.names and a.shapes == b.shapes and a.scopes == b.scopes
    assert a.axis_names == b.axis_names and a.axis_sizes == b.axis_sizes
    assert a.groups == b.groups
    assert a.lib.pe_graph_num_operands(a.h) == b.lib.pe_graph_num_operands(b.h)


def test_text_and_arrays_build_the_same_graph():
    for text in _programs():
        g = engine.Graph(text)
        h = engine.Graph.from_arrays(*pir_arrays.to_arrays(text))
        _same(g, h)


def test_axis_names_come_from_the_library():
    g = engine.Graph(modelgen.config_program(3))
    assert g.axis_names == ["batch", "model"]
    buf = bytearray(8)
    assert g.lib.pe_graph_axis_name(g.h, 5, None, 0) == -1


@pytest.mark.parametrize("text,line,col", [
    ("func @f(%x: f32[4]) -> f32[4] {\n  %y = neg(%x) : f32[4]\n  return %y", 3, 12),
    ("func @f(%x: f32[4]) -> f32[4] {\n  %y = frob(%x) : f32[4]\n  return %y }", 2, 8),
    ("func @f(%x: f32[4]) -> f32[4] { %y = neg(%x) : f64[4] return %y }", 1, 48),
    ("mesh { \"a\" = 2.5 }\nfunc @f(%x: f32[4]) -> f32[4] { return %x }", 1, 14),
    ("func @f(%x: f32[4]) -> f32[4] { %y = all_reduce(%x) : f32[4] return %y }", 1, 38),
    ("func @f(%x: f32[4]) -> f32[4] { return %x } trailing", 1, 45),
    ("func @f(%x: f32[4]) -> f32[4] { %y = neg(%x) {bogus=1} : f32[4] return %y }", 1, 47),
])
def test_syntax_errors_carry_positions(text, line, col):
    with pytest.raises(engine.ParseError) as e:
        engine.Graph(text)
    assert (e.value.line, e.value.column) == (line, col), str(e.value)


@pytest.mark.parametrize("text,frag", [
    ("func @f(%x: f32[4,8], %w: f32[4,8]) -> f32[4,8] { %y = dot(%x, %w) {contract=[[1],[1]], batch=[[],[]]} : f32[4,8] return %y }", "declared f32[4,8]"),
    ("func @f(%x: f32[4]) -> f32[4] { %y = add(%x, %x, %x) : f32[4] return %y }", "takes 2 operands"),
    ("func @f(%x: f32[4]) -> f32[4] { %x = neg(%x) : f32[4] return %x }", "defined twice"),
    ("func @f(%x: f32[4]) -> f32[4] { return %q }", "undefined"),
    ("func @f(%x: f32[4,4]) -> f32[4,4] { %y = transpose(%x) {perm=[0,0]} : f32[4,4] return %y }", "permutation"),
    ("func @f(%x: f32[4]) -> f32[4] { %y = slice(%x) {start=[2], limit=[1]} : f32[4] return %y }", "bounds"),
    ("mesh { \"a\" = 2, \"a\" = 2 }\nfunc @f(%x: f32[4]) -> f32[4] { return %x }", "declared twice"),
])
def test_shape_errors_are_validation_errors(text, frag):
    with pytest.raises(engine.ValidationError, match=re.escape(frag)):
        engine.Graph(text)


def test_tiled_dialect_is_refused_as_a_root():
    with pytest.raises(engine.Error, match="untiled"):
        engine.Graph('mesh { "a" = 2 }\nfunc @f(%x: f32[4]) -> f32[4] { %i = atomic { yield %x } : f32[4] return %i }')


def test_arrays_reject_forward_references():
    with pytest.raises(engine.Error, match="earlier value"):
        engine.Graph.from_arrays("f", [], [("x", [4], "")],
                                 [{"id": "y", "kind": 5, "shape": [4], "operands": [2]}], 1)


@pytest.mark.gpu
def test_arrays_graph_evaluates_identically():
    # the same candidates on engines over the text-built and the array-built
    # graph: identical actions and results (the compiled tables agree)
    import helpers as H
    from paper_2112_02958_b200 import capi
    for text in (modelgen.config_program(2), modelgen.random_program(777, F.MESHES[1])):
        cfg = capi.default_search_config(group_scopes=1)
        a = engine.Engine(engine.Graph(text), device=0, cfg=cfg)
        b = engine.Engine(engine.Graph.from_arrays(*pir_arrays.to_arrays(text)), device=0, cfg=cfg)
        seeds = list(range(512))
        ra, sa, la = a.rollout_batch([[]] * 512, seeds, legal=True)
        rb, sb, lb = b.rollout_batch([[]] * 512, seeds, legal=True)
        assert sa == sb and la == lb
        assert all(not H.compare_results(x, y) for x, y in zip(ra, rb))


def test_reader_accepts_the_grammar_variants():
    # comments, free whitespace, empty lists and attribute blocks, reals in
    # every spelling, scalar tensors, names with digits / dots / slashes
    text = """// leading comment
mesh {   "a"=2 ,"b" = 3 }   // trailing comment
func @f.v2 (%x0: f32[4,6] {scope="layer_0/in"}, %w/1: f32[6]) -> f32[4,6] {
  %c = constant() {value=-1.5e-3} : f32[]
  %cb = broadcast_in_dim(%c) {map=[]} : f32[4,6]
  %wb = broadcast_in_dim(%w/1) {map=[1]} : f32[4,6]
  %y = add(%x0, %cb) {} : f32[4,6]
  %z = mul(%y,%wb) : f32[4,6]
  return %z
}
"""
    g = engine.Graph(text)
    assert g.n_args == 2 and g.n_ops == 5 and g.axis_names == ["a", "b"]
    assert g.shapes[g.value_index("c")] == [] and g.scopes[0] == "layer_0/in"
    h = engine.Graph.from_arrays(*pir_arrays.to_arrays(text.replace("// leading comment\n", "")))
    assert h.names == g.names


@pytest.mark.parametrize("bad", [
    'mesh { "a" = 2 }\nfunc @f(%x: f32[4]) -> f32[4] { %y = neg(%x) : f32[4,] return %y }',
    'func @f(%x: f32[4]) -> f32[4] { %y = slice(%x) {start=[0], limit=[1.0]} : f32[1] return %y }',
    'func @f(%x: f32[4]) -> f32[4] { %y = neg(%x : f32[4] return %y }',
    'func @f(%x: f32[4]) -> f32[4] { %y = neg(%x) : f32[4] return y }',
    'func @f(%x: f32[4]) -> f32[4] { %y = neg(%x) : f32[99999999999999999999] return %y }',
    'func @f(%x: f32[4]) -> f32[4] { %y = constant() {value=} : f32[4] return %y }',
    'func @f(%x: f32[4] -> f32[4] { return %x }',
    'mesh { "a = 2 }',
])
def test_reader_rejects_malformed_text(bad):
    with pytest.raises(engine.ParseError):
        engine.Graph(bad)
