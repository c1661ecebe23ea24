"""Test-side conversion of modelgen `.pir` text into the structured arrays of
pe_graph_create_from_arrays (the binding a reference-side caller would fill
by walking partir::Program).  Regex-based: it only needs to
cover the regular text modelgen emits.  TEST INFRASTRUCTURE."""
from __future__ import annotations

import re

KINDS = ["constant", "add", "sub", "mul", "div", "neg", "exp", "tanh", "rsqrt", "maximum", "dot",
         "reduce_sum", "reduce_max", "transpose", "reshape", "broadcast_in_dim", "slice",
         "concatenate"]

_ints = lambda s: [int(x) for x in s.split(",") if x.strip()]  # noqa: E731


def to_arrays(text: str):
    mesh = re.search(r"mesh\s*\{([^}]*)\}", text)
    axes = [(n, int(v)) for n, v in re.findall(r'"([^"]+)"\s*=\s*(\d+)', mesh.group(1))] if mesh else []
    head = re.search(r"func\s+@(\S+)\s*\((.*?)\)\s*->", text, re.S)
    name = head.group(1)
    args = []
    for m in re.finditer(r'%(\S+?):\s*f32\[([^\]]*)\](?:\s*\{scope="([^"]*)"\})?', head.group(2)):
        args.append((m.group(1), _ints(m.group(2)), m.group(3) or ""))
    index = {a[0]: i for i, a in enumerate(args)}
    ops = []
    body = text[head.end():]
    stmt = re.compile(r"%(\S+)\s*=\s*(\w+)\(([^)]*)\)\s*(\{.*?\})?\s*:\s*f32\[([^\]]*)\]", re.S)
    for m in stmt.finditer(body):
        oid, kind, opnds, attrs, shape = m.groups()
        o = {"id": oid, "kind": KINDS.index(kind), "shape": _ints(shape),
             "operands": [index[x.strip()[1:]] for x in opnds.split(",") if x.strip()]}
        a = attrs or ""
        if kind == "dot":
            c = re.search(r"contract=\[\[([^\]]*)\],\s*\[([^\]]*)\]\]", a)
            b = re.search(r"batch=\[\[([^\]]*)\],\s*\[([^\]]*)\]\]", a)
            o["contract"] = (_ints(c.group(1)), _ints(c.group(2))) if c else ([], [])
            o["batch"] = (_ints(b.group(1)), _ints(b.group(2))) if b else ([], [])
        for key in ("dims", "perm", "map"):
            x = re.search(key + r"=\[([^\]]*)\]", a)
            if x:
                o["dims"] = _ints(x.group(1))
        for key in ("start", "limit"):
            x = re.search(key + r"=\[([^\]]*)\]", a)
            if x:
                o[key] = _ints(x.group(1))
        x = re.search(r"\bdim=(-?\d+)", a)
        if x:
            o["dim"] = int(x.group(1))
        x = re.search(r"value=([-+0-9.eE]+)", a)
        if x:
            o["value"] = float(x.group(1))
        index[oid] = len(args) + len(ops)
        ops.append(o)
    result = index[re.search(r"return\s+%(\S+)", body).group(1)]
    return name, axes, args, ops, result
