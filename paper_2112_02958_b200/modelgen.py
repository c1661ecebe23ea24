"""Deterministic `.pir` program builders (SPEC modelgen module; the reference's
src/modelgen.cc is listed in CMakeLists.txt:25 but not shipped).

* ``linear()``            — the golden Fig. 2 program (SPEC tensor_ir External
                            Interfaces).
* ``build_mlp``           — chain of dot + add + tanh (SPEC build_mlp).
* ``build_transformer``   — forward transformer with head-split weight layouts
                            (43 ops per layer;
                            Megatron = wq/wk/wv dim1, wo dim0, w1 dim1, w2 dim0).
* ``random_program``      — random valid programs over all 18 base kinds for
                            differential fuzzing.

All builders emit text; the engine and the oracle parse the same bytes.
"""
from __future__ import annotations

import random
from dataclasses import dataclass, field


def _ty(shape) -> str:
    return "f32[" + ",".join(str(d) for d in shape) + "]"


@dataclass
class ProgramBuilder:
    name: str
    mesh: list  # [(axis, size)]
    args: list = field(default_factory=list)   # (id, shape, scope)
    ops: list = field(default_factory=list)    # text lines
    shapes: dict = field(default_factory=dict)
    _n: int = 0

    def arg(self, name, shape, scope=None):
        self.args.append((name, list(shape), scope))
        self.shapes[name] = list(shape)
        return name

    def fresh(self, stem="v"):
        self._n += 1
        return f"{stem}{self._n}"

    def op(self, kind, operands, shape, attrs=None, name=None):
        name = name or self.fresh()
        a = ""
        if attrs:
            a = " {" + ", ".join(f"{k}={v}" for k, v in attrs.items()) + "}"
        ops = ", ".join("%" + o for o in operands)
        self.ops.append(f"  %{name} = {kind}({ops}){a} : {_ty(shape)}")
        self.shapes[name] = list(shape)
        return name

    def const(self, value, shape, name=None):
        return self.op("constant", [], shape, {"value": repr(float(value))}, name)

    def text(self, result) -> str:
        lines = []
        if self.mesh:
            lines.append("mesh { " + ", ".join(f'"{a}" = {s}' for a, s in self.mesh) + " }")
        sig = []
        for n, s, sc in self.args:
            sig.append(f"%{n}: {_ty(s)}" + (f' {{scope="{sc}"}}' if sc else ""))
        lines.append(f"func @{self.name}(" + ", ".join(sig) + f") -> {_ty(self.shapes[result])} {{")
        lines.extend(self.ops)
        lines.append(f"  return %{result}")
        lines.append("}")
        return "\n".join(lines) + "\n"


def _list(xs):
    return "[" + ",".join(str(x) for x in xs) + "]"


def _pair(a, b):
    return "[" + _list(a) + "," + _list(b) + "]"


def linear(mesh=(("shard", 2),)) -> str:
    """Fig. 2 golden program: %x f32[8,16], %w f32[16,64] {scope="mlp/w"},
    %b f32[8,64]; dot then add (SPEC tensor_ir External Interfaces)."""
    b = ProgramBuilder("linear", list(mesh))
    b.arg("x", [8, 16])
    b.arg("w", [16, 64], "mlp/w")
    b.arg("b", [8, 64])
    d = b.op("dot", ["x", "w"], [8, 64], {"contract": _pair([1], [0]), "batch": _pair([], [])}, "0")
    r = b.op("add", [d, "b"], [8, 64], None, "1")
    return b.text(r)


def build_mlp(depth=2, widths=(16, 64, 16), batch=8, mesh=(("model", 8),)) -> str:
    """Chain of dot + add + tanh (SPEC build_mlp): arguments x[batch, w0],
    per layer i: w{i+1}[w_i, w_{i+1}], b{i+1}[batch, w_{i+1}]."""
    assert len(widths) == depth + 1
    b = ProgramBuilder("mlp", list(mesh))
    h = b.arg("x", [batch, widths[0]])
    for i in range(depth):
        b.arg(f"w{i + 1}", [widths[i], widths[i + 1]], f"mlp/w{i + 1}")
        b.arg(f"b{i + 1}", [batch, widths[i + 1]], f"mlp/b{i + 1}")
    for i in range(depth):
        d = b.op("dot", [h, f"w{i + 1}"], [batch, widths[i + 1]],
                 {"contract": _pair([len(b.shapes[h]) - 1], [0]), "batch": _pair([], [])})
        a = b.op("add", [d, f"b{i + 1}"], [batch, widths[i + 1]])
        h = b.op("tanh", [a], [batch, widths[i + 1]])
    return b.text(h)


def _layernorm(b: ProgramBuilder, x, B, S, D, tag):
    """14 ops: mean / centred / variance / rsqrt / scale."""
    s = b.op("reduce_sum", [x], [B, S], {"dims": "[2]"}, f"{tag}_sum")
    inv = b.const(1.0 / D, [B, S], f"{tag}_invd")
    mean = b.op("mul", [s, inv], [B, S], None, f"{tag}_mean")
    mb = b.op("broadcast_in_dim", [mean], [B, S, D], {"map": "[0,1]"}, f"{tag}_meanb")
    xc = b.op("sub", [x, mb], [B, S, D], None, f"{tag}_xc")
    sq = b.op("mul", [xc, xc], [B, S, D], None, f"{tag}_sq")
    vs = b.op("reduce_sum", [sq], [B, S], {"dims": "[2]"}, f"{tag}_vsum")
    inv2 = b.const(1.0 / D, [B, S], f"{tag}_invd2")
    var = b.op("mul", [vs, inv2], [B, S], None, f"{tag}_var")
    eps = b.const(1e-5, [B, S], f"{tag}_eps")
    ve = b.op("add", [var, eps], [B, S], None, f"{tag}_ve")
    rs = b.op("rsqrt", [ve], [B, S], None, f"{tag}_rstd")
    rb = b.op("broadcast_in_dim", [rs], [B, S, D], {"map": "[0,1]"}, f"{tag}_rstdb")
    return b.op("mul", [xc, rb], [B, S, D], None, f"{tag}_out")


def build_transformer(layers=1, batch=2, seq=4, d_model=8, heads=2, d_ff=32,
                      mesh=(("model", 2),), name="transformer") -> str:
    """Forward transformer, head-split weights:
    x[B,S,D]; per layer wq/wk/wv [D,H,Dh], wo [H,Dh,D], w1 [D,F], w2 [F,D]
    with scopes layer_i/attention/{q,k,v,o}_proj and layer_i/mlp/{w1,w2}.
    43 ops per layer."""
    B, S, D, H, F = batch, seq, d_model, heads, d_ff
    if D % H:
        raise ValueError("heads must divide d_model")
    Dh = D // H
    b = ProgramBuilder(name, list(mesh))
    x = b.arg("x", [B, S, D])
    for i in range(layers):
        for w in ("q", "k", "v"):
            b.arg(f"l{i}_w{w}", [D, H, Dh], f"layer_{i}/attention/{w}_proj")
        b.arg(f"l{i}_wo", [H, Dh, D], f"layer_{i}/attention/o_proj")
        b.arg(f"l{i}_w1", [D, F], f"layer_{i}/mlp/w1")
        b.arg(f"l{i}_w2", [F, D], f"layer_{i}/mlp/w2")
    for i in range(layers):
        t = f"l{i}"
        ln = _layernorm(b, x, B, S, D, f"{t}_ln1")
        proj = {}
        for w in ("q", "k", "v"):
            proj[w] = b.op("dot", [ln, f"{t}_w{w}"], [B, S, H, Dh],
                           {"contract": _pair([2], [0]), "batch": _pair([], [])}, f"{t}_{w}")
        sc = b.op("dot", [proj["q"], proj["k"]], [B, H, S, S],
                  {"contract": _pair([3], [3]), "batch": _pair([0, 2], [0, 2])}, f"{t}_scores")
        e = b.op("exp", [sc], [B, H, S, S], None, f"{t}_exp")
        z = b.op("reduce_sum", [e], [B, H, S], {"dims": "[3]"}, f"{t}_z")
        zb = b.op("broadcast_in_dim", [z], [B, H, S, S], {"map": "[0,1,2]"}, f"{t}_zb")
        p = b.op("div", [e, zb], [B, H, S, S], None, f"{t}_probs")
        ctx = b.op("dot", [p, proj["v"]], [B, H, S, Dh],
                   {"contract": _pair([3], [1]), "batch": _pair([0, 1], [0, 2])}, f"{t}_ctx")
        att = b.op("dot", [ctx, f"{t}_wo"], [B, S, D],
                   {"contract": _pair([1, 3], [0, 1]), "batch": _pair([], [])}, f"{t}_attn")
        r1 = b.op("add", [x, att], [B, S, D], None, f"{t}_res1")
        ln2 = _layernorm(b, r1, B, S, D, f"{t}_ln2")
        h = b.op("dot", [ln2, f"{t}_w1"], [B, S, F],
                 {"contract": _pair([2], [0]), "batch": _pair([], [])}, f"{t}_h")
        act = b.op("tanh", [h], [B, S, F], None, f"{t}_act")
        o = b.op("dot", [act, f"{t}_w2"], [B, S, D],
                 {"contract": _pair([2], [0]), "batch": _pair([], [])}, f"{t}_mlp")
        x = b.op("add", [r1, o], [B, S, D], None, f"{t}_out")
    return b.text(x)


GPT2_MEDIUM = dict(batch=8, seq=1024, d_model=1024, heads=16, d_ff=4096)
TOY = dict(batch=2, seq=4, d_model=8, heads=2, d_ff=32)


def config_program(cfg: int) -> str:
    """The BASELINE.json configurations."""
    if cfg == 1:
        return build_mlp(2, (16, 64, 16), 8, (("model", 8),))
    if cfg == 2:
        return build_transformer(1, mesh=(("model", 2),), **TOY)
    if cfg == 3:
        return build_transformer(24, mesh=(("batch", 4), ("model", 2)), name="gpt2_medium",
                                 **GPT2_MEDIUM)
    raise ValueError(cfg)


# ---------------------------------------------------------------- fuzzing
_DIMS = (2, 4, 8)
_BIN = ("add", "sub", "mul", "div", "maximum")
_UN = ("neg", "exp", "tanh", "rsqrt")


def random_program(seed: int, mesh=(("m", 2),), max_ops=15) -> str:
    """A random valid program over all 18 base kinds: rank
    1-3, dims in {2,4,8}, 2-4 arguments, 4-15 ops."""
    rng = random.Random(seed)
    b = ProgramBuilder(f"rand{seed}", list(mesh))
    vals = []
    for i in range(rng.randint(2, 4)):
        shape = [rng.choice(_DIMS) for _ in range(rng.randint(1, 3))]
        vals.append(b.arg(f"a{i}", shape))
    nw = 0
    last = None
    for _ in range(rng.randint(4, max_ops)):
        v = rng.choice(vals)
        s = b.shapes[v]
        r = len(s)
        kind = rng.choice(["bin", "un", "dot", "reduce", "transpose", "reshape",
                           "broadcast", "slice", "concat", "const"])
        out = None
        if kind == "bin":
            same = [w for w in vals if b.shapes[w] == s]
            other = rng.choice(same) if rng.random() < 0.7 else b.const(rng.choice([0.5, 2.0]), s)
            ops = [v, other] if rng.random() < 0.5 else [other, v]
            out = b.op(rng.choice(_BIN), ops, s)
        elif kind == "un":
            out = b.op(rng.choice(_UN), [v], s)
        elif kind == "dot" and 1 <= r <= 3:
            n = rng.choice(_DIMS)
            cd = rng.randrange(r)
            w = b.arg(f"w{nw}", [s[cd], n])
            nw += 1
            res = [d for i, d in enumerate(s) if i != cd] + [n]
            if rng.random() < 0.5:
                out = b.op("dot", [v, w], res, {"contract": _pair([cd], [0]), "batch": _pair([], [])})
            else:
                res2 = [n] + [d for i, d in enumerate(s) if i != cd]
                out = b.op("dot", [w, v], res2, {"contract": _pair([0], [cd]), "batch": _pair([], [])})
        elif kind == "reduce" and r >= 1:
            d = rng.randrange(r)
            out = b.op(rng.choice(["reduce_sum", "reduce_max"]), [v],
                       [x for i, x in enumerate(s) if i != d], {"dims": _list([d])})
        elif kind == "transpose" and r >= 2:
            perm = list(range(r))
            rng.shuffle(perm)
            out = b.op("transpose", [v], [s[p] for p in perm], {"perm": _list(perm)})
        elif kind == "reshape" and r >= 1:
            if r >= 2 and rng.random() < 0.5:
                d = rng.randrange(r - 1)
                ns = s[:d] + [s[d] * s[d + 1]] + s[d + 2:]
            else:
                cands = [i for i in range(r) if s[i] >= 4]
                if not cands or r >= 4:
                    continue
                d = rng.choice(cands)
                ns = s[:d] + [2, s[d] // 2] + s[d + 1:]
            out = b.op("reshape", [v], ns)
        elif kind == "broadcast" and r <= 3:
            pos = rng.randint(0, r)
            ns = s[:pos] + [rng.choice(_DIMS)] + s[pos:]
            mp = [i if i < pos else i + 1 for i in range(r)]
            out = b.op("broadcast_in_dim", [v], ns, {"map": _list(mp)})
        elif kind == "slice" and r >= 1:
            d = rng.randrange(r)
            start = [0] * r
            limit = list(s)
            if s[d] >= 2:
                if rng.random() < 0.5:
                    limit[d] = s[d] // 2
                else:
                    start[d] = s[d] // 2
            out = b.op("slice", [v], [limit[i] - start[i] for i in range(r)],
                       {"start": _list(start), "limit": _list(limit)})
        elif kind == "concat" and r >= 1:
            same = [w for w in vals if b.shapes[w] == s]
            d = rng.randrange(r)
            others = [rng.choice(same) for _ in range(rng.randint(1, 2))]
            ns = list(s)
            ns[d] = s[d] * (1 + len(others))
            if ns[d] > 64:
                continue
            out = b.op("concatenate", [v] + others, ns, {"dim": d})
        elif kind == "const":
            out = b.const(rng.choice([1.0, 3.0]), [rng.choice(_DIMS) for _ in range(rng.randint(1, 3))])
        if out is not None:
            vals.append(out)
            if kind != "const":
                last = out
    if last is None:
        last = b.op("neg", [vals[0]], b.shapes[vals[0]])
    return b.text(last)


def program_values(text: str):
    """(names, shapes) of args then ops, parsed from builder output."""
    import re
    names, shapes = [], []
    head = re.search(r"func @\w+\((.*?)\) ->", text, re.S).group(1)
    for m in re.finditer(r"%([\w./]+): f32\[([0-9,]*)\]", head):
        names.append(m.group(1))
        shapes.append([int(x) for x in m.group(2).split(",") if x])
    for m in re.finditer(r"^\s*%([\w./]+) = \w+\(.*?\).*?: f32\[([0-9,]*)\]\s*$", text, re.M):
        names.append(m.group(1))
        shapes.append([int(x) for x in m.group(2).split(",") if x])
    return names, shapes


def random_actions(seed: int, text: str, mesh, n_max=6, legal_bias=0.9):
    """Random tile actions on arguments or op values: (value, dim, axis, kind)."""
    rng = random.Random(seed)
    names, shapes = program_values(text)
    acts = []
    for _ in range(rng.randint(1, n_max)):
        v = rng.randrange(len(names))
        s = shapes[v]
        if not s:
            continue
        ax = rng.randrange(len(mesh))
        size = mesh[ax][1]
        dims = [d for d in range(len(s)) if s[d] % size == 0]
        if dims and rng.random() < legal_bias:
            d = rng.choice(dims)
        else:
            d = rng.randrange(len(s))
        acts.append((v, d, ax, 0))
    return acts
