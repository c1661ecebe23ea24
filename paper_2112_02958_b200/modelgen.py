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
    if cfg == 4:
        # 48-layer training step at MHLO granularity with 4-way gradient
        # accumulation: 52,154 ops, 1,156 arguments ("just over 50k
        # operations, and 1150 arguments")
        return build_training_step(48, mesh=(("batch", 4), ("model", 2)), detailed=True,
                                   microbatches=4, **GPT2_MEDIUM)
    if cfg == 40:  # the round-1 config-4 graph (coarser ops): 13,757 ops, 1,153 arguments
        return build_training_step(48, mesh=(("batch", 4), ("model", 2)), **GPT2_MEDIUM)
    raise ValueError(cfg)


# ---------------------------------------------------------------- training step
class Tape:
    """Structured op recorder over ProgramBuilder with reverse-mode gradients
    for the kinds the transformer uses (SPEC modelgen: "hand-derived gradient
    ops"; here derived mechanically per op kind)."""

    def __init__(self, b: ProgramBuilder):
        self.b = b
        self.rec = []  # (out, kind, ins, meta)

    def shape(self, v):
        return self.b.shapes[v]

    def _op(self, kind, ins, shape, attrs, meta, name=None):
        out = self.b.op(kind, ins, shape, attrs, name)
        self.rec.append((out, kind, list(ins), meta))
        return out

    def const(self, value, shape):
        if getattr(self, "scalar_consts", False):
            # MHLO style (what a JAX-lowered graph contains): a scalar
            # constant broadcast to the use's shape
            c = self.b.const(value, [])
            return self.b.op("broadcast_in_dim", [c], list(shape), {"map": "[]"})
        return self.b.const(value, shape)

    def ew(self, kind, *ins):
        return self._op(kind, ins, self.shape(ins[0]), None, {})

    def dot(self, a, b, lc, rc, lb=(), rb=()):
        sa, sb = self.shape(a), self.shape(b)
        used_a = set(lb) | set(lc)
        used_b = set(rb) | set(rc)
        shape = [sa[i] for i in lb] + [sa[i] for i in range(len(sa)) if i not in used_a] + \
                [sb[j] for j in range(len(sb)) if j not in used_b]
        attrs = {"contract": _pair(list(lc), list(rc)), "batch": _pair(list(lb), list(rb))}
        return self._op("dot", [a, b], shape, attrs,
                        {"lc": list(lc), "rc": list(rc), "lb": list(lb), "rb": list(rb)})

    def reduce_sum(self, a, dims):
        sa = self.shape(a)
        shape = [sa[i] for i in range(len(sa)) if i not in dims]
        return self._op("reduce_sum", [a], shape, {"dims": _list(sorted(dims))},
                        {"dims": sorted(dims)})

    def bcast(self, a, shape, mp):
        return self._op("broadcast_in_dim", [a], list(shape), {"map": _list(mp)}, {"map": list(mp)})

    def transpose(self, a, perm):
        sa = self.shape(a)
        return self._op("transpose", [a], [sa[p] for p in perm], {"perm": _list(perm)},
                        {"perm": list(perm)})

    def grads(self, loss, wrt):
        needs = set(wrt)
        for out, kind, ins, meta in self.rec:
            if any(i in needs for i in ins):
                needs.add(out)
        g = {loss: self.const(1.0, self.shape(loss))}

        def acc(x, gx):
            if x not in needs:
                return
            g[x] = gx if x not in g else self.ew("add", g[x], gx)

        for out, kind, ins, meta in reversed(self.rec):
            if out not in g:
                continue
            go = g[out]
            if kind == "add":
                acc(ins[0], go)
                acc(ins[1], go)
            elif kind == "sub":
                acc(ins[0], go)
                if ins[1] in needs:
                    acc(ins[1], self.ew("neg", go))
            elif kind == "mul":
                if ins[0] in needs:
                    acc(ins[0], self.ew("mul", go, ins[1]))
                if ins[1] in needs:
                    acc(ins[1], self.ew("mul", go, ins[0]))
            elif kind == "div":
                if ins[0] in needs:
                    acc(ins[0], self.ew("div", go, ins[1]))
                if ins[1] in needs:
                    acc(ins[1], self.ew("neg", self.ew("div", self.ew("mul", go, out), ins[1])))
            elif kind == "exp":
                acc(ins[0], self.ew("mul", go, out))
            elif kind == "tanh":
                one = self.const(1.0, self.shape(out))
                acc(ins[0], self.ew("mul", go, self.ew("sub", one, self.ew("mul", out, out))))
            elif kind == "rsqrt":
                c = self.const(-0.5, self.shape(out))
                cube = self.ew("mul", out, self.ew("mul", out, out))
                acc(ins[0], self.ew("mul", go, self.ew("mul", c, cube)))
            elif kind == "neg":
                acc(ins[0], self.ew("neg", go))
            elif kind == "reduce_sum":
                sa = self.shape(ins[0])
                keep = [i for i in range(len(sa)) if i not in meta["dims"]]
                acc(ins[0], self.bcast(go, sa, keep))
            elif kind == "broadcast_in_dim":
                so = self.shape(out)
                acc(ins[0], self.reduce_sum(go, [j for j in range(len(so)) if j not in meta["map"]]))
            elif kind == "transpose":
                perm = meta["perm"]
                inv = [perm.index(i) for i in range(len(perm))]
                acc(ins[0], self.transpose(go, inv))
            elif kind == "dot":
                self._dot_grads(out, ins, meta, go, acc, needs)
            else:
                raise NotImplementedError(kind)
        return g

    def _dot_grads(self, out, ins, meta, go, acc, needs):
        a, b = ins
        lb, rb, lc, rc = meta["lb"], meta["rb"], meta["lc"], meta["rc"]
        ra, rbk = len(self.shape(a)), len(self.shape(b))
        nb = len(lb)
        a_free = [i for i in range(ra) if i not in lb and i not in lc]
        b_free = [j for j in range(rbk) if j not in rb and j not in rc]
        naf = len(a_free)
        if a in needs:
            r = self.dot(go, b, [nb + naf + j for j in range(len(b_free))], b_free,
                         list(range(nb)), rb)
            dims = lb + a_free + [lc[rc.index(c)] for c in sorted(rc)]
            perm = [dims.index(i) for i in range(ra)]
            acc(a, r if perm == list(range(ra)) else self.transpose(r, perm))
        if b in needs:
            r = self.dot(a, go, a_free, [nb + i for i in range(naf)], lb, list(range(nb)))
            dims = rb + [rc[lc.index(c)] for c in sorted(lc)] + b_free
            perm = [dims.index(j) for j in range(rbk)]
            acc(b, r if perm == list(range(rbk)) else self.transpose(r, perm))


def build_training_step(layers=48, batch=8, seq=1024, d_model=1024, heads=16, d_ff=4096,
                        mesh=(("batch", 4), ("model", 2)), name="train_step",
                        detailed=False, microbatches=1) -> str:
    """One training step of the head-split transformer (SURVEY.md §8(d)
    config 4: "hand-derived backward plus optimiser state"): forward as
    build_transformer with learned layer-norm gains, loss = sum of the
    output, reverse-mode gradients of every parameter, and an Adam update
    (first/second moments are arguments with the parameter's scope); the
    function returns the sum of the updated parameters.

    detailed=True is the graph at the granularity a JAX/MHLO lowering has
    (a 24-layer GPT-3-style model with "just over 50k operations,
    and 1150 arguments"): scalar constants broadcast to shape, attention
    scaling and a max-subtracted softmax (the max under stop-gradient),
    dropout multipliers, the tanh-approximated GELU, and an Adam update with
    bias correction, decoupled weight decay and global-norm gradient
    clipping.  Same 8 parameters per layer (+ two moments each).
    microbatches=k: gradient accumulation over k data inputs x0..x{k-1}
    (one loss; each parameter's per-microbatch gradients are summed)."""
    B, S, D, H, F = batch, seq, d_model, heads, d_ff
    Dh = D // H
    bld = ProgramBuilder(name, list(mesh))
    t = Tape(bld)
    t.scalar_consts = detailed
    xs = [bld.arg("x", [B, S, D])] if microbatches == 1 else \
        [bld.arg(f"x{k}", [B, S, D]) for k in range(microbatches)]
    params = []
    for i in range(layers):
        for w, shp, sc in (("wq", [D, H, Dh], "attention/q_proj"), ("wk", [D, H, Dh], "attention/k_proj"),
                           ("wv", [D, H, Dh], "attention/v_proj"), ("wo", [H, Dh, D], "attention/o_proj"),
                           ("w1", [D, F], "mlp/w1"), ("w2", [F, D], "mlp/w2"),
                           ("g1", [D], "ln1/gain"), ("g2", [D], "ln2/gain")):
            params.append(bld.arg(f"l{i}_{w}", shp, f"layer_{i}/{sc}"))
    opt = {}
    for p in params:
        sc = [a[2] for a in bld.args if a[0] == p][0]
        opt[p] = (bld.arg(p + "_m", bld.shapes[p], sc + "/adam_m"),
                  bld.arg(p + "_v", bld.shapes[p], sc + "/adam_v"))

    def ln(v, gain):
        s = t.reduce_sum(v, [2])
        mean = t.ew("mul", s, t.const(1.0 / D, [B, S]))
        xc = t.ew("sub", v, t.bcast(mean, [B, S, D], [0, 1]))
        var = t.ew("mul", t.reduce_sum(t.ew("mul", xc, xc), [2]), t.const(1.0 / D, [B, S]))
        rs = t.ew("rsqrt", t.ew("add", var, t.const(1e-5, [B, S])))
        y = t.ew("mul", xc, t.bcast(rs, [B, S, D], [0, 1]))
        return t.ew("mul", y, t.bcast(gain, [B, S, D], [2]))

    def dropout(v):  # keep-probability multiplier (a splat mask)
        return t.ew("mul", v, t.const(0.9, t.shape(v))) if detailed else v

    def gelu(v):  # 0.5 x (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3)))
        sh = t.shape(v)
        x3 = t.ew("mul", t.ew("mul", v, v), v)
        inner = t.ew("mul", t.ew("add", v, t.ew("mul", x3, t.const(0.044715, sh))),
                     t.const(0.7978845608, sh))
        return t.ew("mul", t.ew("mul", v, t.const(0.5, sh)),
                    t.ew("add", t.const(1.0, sh), t.ew("tanh", inner)))

    def forward(h):
        for i in range(layers):
            P = lambda w: f"l{i}_{w}"  # noqa: E731
            a = ln(h, P("g1"))
            q = t.dot(a, P("wq"), [2], [0])
            k = t.dot(a, P("wk"), [2], [0])
            v = t.dot(a, P("wv"), [2], [0])
            if detailed:
                q = t.ew("mul", q, t.const(Dh ** -0.5, t.shape(q)))
            sc = t.dot(q, k, [3], [3], [0, 2], [0, 2])
            if detailed:
                # numerically stable softmax: the row max under stop-gradient
                # (recorded outside the tape, so no gradient flows through it)
                mx = bld.op("reduce_max", [sc], [B, H, S], {"dims": "[3]"})
                mxb = bld.op("broadcast_in_dim", [mx], [B, H, S, S], {"map": "[0,1,2]"})
                sc = t.ew("sub", sc, mxb)
            e = t.ew("exp", sc)
            z = t.bcast(t.reduce_sum(e, [3]), [B, H, S, S], [0, 1, 2])
            pr = dropout(t.ew("div", e, z))
            ctx = t.dot(pr, v, [3], [1], [0, 1], [0, 2])
            att = dropout(t.dot(ctx, P("wo"), [1, 3], [0, 1]))
            r1 = t.ew("add", h, att)
            m = ln(r1, P("g2"))
            u = t.dot(m, P("w1"), [2], [0])
            hh = gelu(u) if detailed else t.ew("tanh", u)
            h = t.ew("add", r1, dropout(t.dot(hh, P("w2"), [2], [0])))
        return h


    loss = None
    for x in xs:
        lk = t.reduce_sum(forward(x), [0, 1, 2])
        loss = lk if loss is None else t.ew("add", loss, lk)
    g = t.grads(loss, params)
    if detailed:
        # global-norm clipping: scale = clip * rsqrt(sum of squared grads + eps)
        norm2 = None
        for p in params:
            sq = t.reduce_sum(t.ew("mul", g[p], g[p]), list(range(len(bld.shapes[p]))))
            norm2 = sq if norm2 is None else t.ew("add", norm2, sq)
        scale = t.ew("mul", t.ew("rsqrt", t.ew("add", norm2, t.const(1e-6, []))), t.const(1.0, []))
    total = None
    for p in params:
        s = bld.shapes[p]
        m0, v0 = opt[p]
        gp = g[p]
        if detailed:
            gp = t.ew("mul", gp, t.bcast(scale, s, []))
        m1 = t.ew("add", t.ew("mul", m0, t.const(0.9, s)), t.ew("mul", gp, t.const(0.1, s)))
        v1 = t.ew("add", t.ew("mul", v0, t.const(0.999, s)),
                  t.ew("mul", t.ew("mul", gp, gp), t.const(0.001, s)))
        if detailed:  # bias correction (step 1) and decoupled weight decay
            mh = t.ew("div", m1, t.const(0.1, s))
            vh = t.ew("div", v1, t.const(0.001, s))
            upd = t.ew("add", t.ew("mul", mh, t.ew("rsqrt", t.ew("add", vh, t.const(1e-8, s)))),
                       t.ew("mul", p, t.const(0.01, s)))
        else:
            upd = t.ew("mul", m1, t.ew("rsqrt", t.ew("add", v1, t.const(1e-8, s))))
        p1 = t.ew("sub", p, t.ew("mul", upd, t.const(1e-3, s)))
        red = t.reduce_sum(p1, list(range(len(s))))
        total = red if total is None else t.ew("add", total, red)
    return bld.text(total)


# ---------------------------------------------------------------- fuzzing
_DIMS = (2, 4, 8)
_BIN = ("add", "sub", "mul", "div", "maximum")
_UN = ("neg", "exp", "tanh", "rsqrt")


def random_program(seed: int, mesh=(("m", 2),), max_ops=15, dims=_DIMS) -> str:
    """A random valid program over all 18 base kinds: rank
    1-3, dims drawn from `dims` (default {2,4,8}), 2-4 arguments, 4-15 ops."""
    _DIMS = dims  # noqa: N806
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
                cands = [i for i in range(r) if s[i] >= 4 and s[i] % 2 == 0]
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
