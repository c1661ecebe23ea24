"""Ranker: the learned node-relevance pre-filter of the worklist (SPEC ranker
module; `src/ranker.cc` is listed in the reference's CMakeLists.txt:28 but
not shipped — SURVEY.md §8(f) rank 4).

The ranker is upstream of the hot path: it narrows the static worklist to the
top-k arguments (`pe_search_config.worklist_args`, k = 25 by default,
PAPER §2.3), then search runs on the engine as usual.  It follows the SPEC
design decisions:

- `featurize`: per node (arguments, then ops), an op-kind one-hot (the 18
  base kinds, "argument", 5 hash buckets for unknown kinds = 24 slots),
  log-scaled operand-shape features padded to rank 4, the rank, and a
  partitioned-axes indicator per mesh axis.  Edges: dataflow
  (producer -> consumer) and structural (scope siblings: arguments whose
  normalised scopes match).
- `RankerModel`: 2 rounds of mean-aggregation message passing, hidden width
  32, tanh, then a per-node linear scorer; float64 numpy with hand-derived
  gradients (`loss_and_grad`).
- `train`: pairwise hinge ranking loss (a labeled argument above an unlabeled
  one by margin 1), plain gradient descent, learning rate 0.01.
- `generate_dataset`: small transformer / MLP variants (modelgen); every
  single-argument TileValue (and grouped TileValue) is evaluated
  exhaustively — on the GPU engine, the bulk evaluation it exists for — and
  the label is the set of arguments tiled by the reward-optimal plan.
- `score_and_filter`: top-k candidate arguments by score, ties by ordinal.
- Model file: versioned text header, then each parameter array in decimal.

Everything here is deterministic given seeds.
"""
from __future__ import annotations

import math
import random
import re
import zlib
from dataclasses import dataclass, field

import numpy as np

from . import capi, modelgen

KINDS = ("constant", "add", "sub", "mul", "div", "maximum", "neg", "exp", "tanh", "rsqrt",
         "dot", "reduce_sum", "reduce_max", "transpose", "reshape", "broadcast_in_dim", "slice",
         "concatenate")
KIND_SLOTS = 24                 # 18 kinds + argument + 5 hash buckets
ARG_SLOT = 18
MAX_RANK = 4
MAX_AXES = 4
N_FEATURES = KIND_SLOTS + MAX_RANK + 1 + MAX_AXES
HIDDEN = 32
ROUNDS = 2
MODEL_MAGIC = "pe-ranker 1"


def normalize_scope(scope: str) -> str:
    """SPEC scope normalisation (as pe_graph.cc normalize_scope): drop
    all-digit path segments and trailing `_<digits>` suffixes."""
    out = []
    for seg in scope.split("/"):
        if seg.isdigit():
            continue
        out.append(re.sub(r"_\d+$", "", seg))
    return "/".join(out)


@dataclass
class GraphEncoding:
    x: np.ndarray                       # [n_nodes, N_FEATURES]
    agg_to: np.ndarray                  # aggregation edges: node agg_to[e] averages
    agg_from: np.ndarray                # over its neighbours agg_from[e]
    n_args: int
    names: list = field(default_factory=list)

    @property
    def n_nodes(self) -> int:
        return self.x.shape[0]


_OP_RE = re.compile(r"^\s*%(\w+)\s*=\s*(\w+)\(([^)]*)\)", re.M)


def featurize(text: str, arg_axes=None) -> GraphEncoding:
    """SPEC featurize(p, mesh).  `arg_axes[a]` = mesh axes argument a is
    already partitioned on (the partitioned-axes indicator; default none)."""
    names, shapes = modelgen.program_values(text)
    head = re.search(r"func @\w+\((.*?)\) ->", text, re.S).group(1)
    arg_ids = re.findall(r"%(\w+)\s*:", head)
    scopes = {}
    for m in re.finditer(r"%(\w+)\s*:\s*f32\[[^\]]*\]\s*(?:\{scope=\"([^\"]*)\"\})?", head):
        scopes[m.group(1)] = m.group(2) or ""
    n_args = len(arg_ids)
    index = {n: i for i, n in enumerate(names)}
    ops = _OP_RE.findall(text)
    n = len(names)
    x = np.zeros((n, N_FEATURES))
    for i in range(n):
        if i < n_args:
            slot = ARG_SLOT
        else:
            kind = ops[i - n_args][1]
            slot = KINDS.index(kind) if kind in KINDS else \
                ARG_SLOT + 1 + zlib.crc32(kind.encode()) % (KIND_SLOTS - ARG_SLOT - 1)
        x[i, slot] = 1.0
        sh = shapes[i]
        for d, s in enumerate(sh[:MAX_RANK]):
            x[i, KIND_SLOTS + d] = math.log2(1 + s) / 16.0
        x[i, KIND_SLOTS + MAX_RANK] = len(sh) / MAX_RANK
        if arg_axes is not None and i < n_args:
            for ax in arg_axes[i]:
                x[i, KIND_SLOTS + MAX_RANK + 1 + ax] = 1.0
    to, frm = [], []
    for k, (oid, _kind, operands) in enumerate(ops):
        c = n_args + k
        for o in re.findall(r"%(\w+)", operands):
            p = index[o]
            to += [c, p]        # dataflow producer -> consumer, aggregated both ways
            frm += [p, c]
    by_scope = {}
    for a, aid in enumerate(arg_ids):
        sc = scopes.get(aid, "")
        if sc:
            by_scope.setdefault(normalize_scope(sc), []).append(a)
    for members in by_scope.values():  # structural: scope siblings
        for a in members:
            for b in members:
                if a != b:
                    to.append(a)
                    frm.append(b)
    return GraphEncoding(x, np.array(to, dtype=np.int64), np.array(frm, dtype=np.int64),
                         n_args, names)


# ---------------------------------------------------------------- model
class RankerModel:
    """2-round mean-aggregation message passing, hidden 32, tanh, then a
    per-node linear scorer (SPEC RankerModel)."""

    BLOCKS = ("W0", "b0", "W1", "b1", "W2", "b2", "wout", "bout")

    def __init__(self, seed: int = 0):
        rng = np.random.default_rng(seed)
        f, h = N_FEATURES, HIDDEN
        # std 2/sqrt(fan_in): the inputs are sparse one-hot / [0,1] features,
        # at 1/sqrt(fan_in) the tanh layers start nearly flat and plain GD at
        # lr 0.01 stalls (SPEC example: 1 example, 200 epochs -> loss < 0.1)
        self.p = {
            "W0": rng.normal(0, 2 / math.sqrt(f), (f, h)), "b0": np.zeros(h),
            "W1": rng.normal(0, 2 / math.sqrt(2 * h), (2 * h, h)), "b1": np.zeros(h),
            "W2": rng.normal(0, 2 / math.sqrt(2 * h), (2 * h, h)), "b2": np.zeros(h),
            "wout": rng.normal(0, 2 / math.sqrt(h), h), "bout": np.zeros(1),
        }
        self.final_loss = None

    def copy(self) -> "RankerModel":
        m = RankerModel.__new__(RankerModel)
        m.p = {k: v.copy() for k, v in self.p.items()}
        m.final_loss = self.final_loss
        return m

    # aggregation: m[i] = mean_{j in nbr(i)} h[j]
    @staticmethod
    def _deg(enc):
        return np.bincount(enc.agg_to, minlength=enc.n_nodes).astype(np.float64)

    @staticmethod
    def _agg(enc, h, deg):
        m = np.zeros_like(h)
        np.add.at(m, enc.agg_to, h[enc.agg_from])
        return m / np.maximum(deg, 1.0)[:, None]

    @staticmethod
    def _agg_t(enc, g, deg):
        gs = g / np.maximum(deg, 1.0)[:, None]
        out = np.zeros_like(g)
        np.add.at(out, enc.agg_from, gs[enc.agg_to])
        return out

    def forward(self, enc: GraphEncoding):
        p = self.p
        deg = self._deg(enc)
        h = np.tanh(enc.x @ p["W0"] + p["b0"])
        cache = [(None, h)]
        for r in (1, 2):
            m = self._agg(enc, h, deg)
            cat = np.concatenate([h, m], axis=1)
            h = np.tanh(cat @ p[f"W{r}"] + p[f"b{r}"])
            cache.append((cat, h))
        s = h @ p["wout"] + p["bout"][0]
        return s, (deg, cache)

    def scores(self, enc: GraphEncoding) -> np.ndarray:
        return self.forward(enc)[0]

    def backward(self, enc, ds, state):
        p = self.p
        deg, cache = state
        g = {}
        h2 = cache[2][1]
        g["wout"] = h2.T @ ds
        g["bout"] = np.array([ds.sum()])
        dh = np.outer(ds, p["wout"])
        for r in (2, 1):
            cat, h = cache[r]
            dz = dh * (1 - h * h)
            g[f"W{r}"] = cat.T @ dz
            g[f"b{r}"] = dz.sum(0)
            dcat = dz @ p[f"W{r}"].T
            dh = dcat[:, :HIDDEN] + self._agg_t(enc, dcat[:, HIDDEN:], deg)
        h0 = cache[0][1]
        dz = dh * (1 - h0 * h0)
        g["W0"] = enc.x.T @ dz
        g["b0"] = dz.sum(0)
        return g


def hinge_loss_grad(s: np.ndarray, n_args: int, labels) -> tuple:
    """Pairwise hinge (margin 1) over candidate arguments: mean over
    (labeled, unlabeled) pairs of max(0, 1 - (s_pos - s_neg))."""
    pos = sorted(set(labels))
    neg = [a for a in range(n_args) if a not in set(labels)]
    ds = np.zeros_like(s)
    if not pos or not neg:
        return 0.0, ds
    sp = s[pos][:, None]
    sn = s[neg][None, :]
    margin = 1.0 - (sp - sn)
    act = margin > 0
    npairs = len(pos) * len(neg)
    loss = float(np.where(act, margin, 0.0).sum() / npairs)
    a = act.astype(np.float64) / npairs
    np.add.at(ds, pos, -a.sum(1))
    np.add.at(ds, neg, a.sum(0))
    return loss, ds


def loss_and_grad(model: RankerModel, dataset) -> tuple:
    """Mean hinge loss over the dataset and its gradient per parameter block."""
    total = 0.0
    grads = {k: np.zeros_like(v) for k, v in model.p.items()}
    for enc, labels in dataset:
        s, st = model.forward(enc)
        loss, ds = hinge_loss_grad(s, enc.n_args, labels)
        total += loss
        if not ds.any():
            continue
        for k, v in model.backward(enc, ds, st).items():
            grads[k] += v
    n = max(1, len(dataset))
    return total / n, {k: v / n for k, v in grads.items()}


def train(dataset, epochs: int = 200, seed: int = 0, lr: float = 0.01,
          model: RankerModel | None = None) -> RankerModel:
    """SPEC train: plain gradient descent on the pairwise hinge loss."""
    m = model.copy() if model is not None else RankerModel(seed)
    loss = None
    for _ in range(epochs):
        loss, g = loss_and_grad(m, dataset)
        for k in m.p:
            m.p[k] -= lr * g[k]
    m.final_loss = loss_and_grad(m, dataset)[0] if dataset else None
    return m


def score_and_filter(enc: GraphEncoding, model: RankerModel, k: int = 25) -> list:
    """Top-k candidate arguments by score, ties by node ordinal."""
    s = model.scores(enc)[: enc.n_args]
    order = sorted(range(enc.n_args), key=lambda a: (-s[a], a))
    return sorted(order[: max(1, k)])


def filtered_config(text: str, model: RankerModel, cfg=None, k: int = 25):
    """A search config whose static worklist is the ranker's top-k."""
    cfg = cfg if cfg is not None else capi.default_search_config()
    return cfg.restrict_worklist(score_and_filter(featurize(text), model, k))


# ---------------------------------------------------------------- dataset
def single_action_candidates(text: str, group: bool):
    """Every single TileValue decision (argument x dim x axis, and the
    grouped variants), SPEC generate_dataset's exhaustive desk-scale search
    space, as (action sequence, tiled argument set)."""
    names, shapes = modelgen.program_values(text)
    head = re.search(r"func @\w+\((.*?)\) ->", text, re.S).group(1)
    n_args = len(re.findall(r"%(\w+)\s*:", head))
    mesh = re.search(r"mesh\s*\{(.*?)\}", text, re.S).group(1)
    sizes = [int(v) for v in re.findall(r"=\s*(\d+)", mesh)]
    out = []
    for a in range(n_args):
        for d, s in enumerate(shapes[a]):
            for ax, sz in enumerate(sizes):
                if s % sz == 0:
                    out.append(([(a, d, ax, capi.PE_ACT_TILE)], {a}))
    if group:
        from . import engine
        g = engine.Graph(text)
        for gi, members in enumerate(g.groups):
            if len(members) < 2:
                continue
            for d in range(MAX_RANK):
                for ax, sz in enumerate(sizes):
                    if any(d < len(shapes[m]) and shapes[m][d] % sz == 0 for m in members):
                        out.append(([(gi, d, ax, capi.PE_ACT_TILE_GROUP)], set(members)))
    return out


def sample_program(rng: random.Random) -> str:
    """A small transformer or MLP variant (desk-scale analogue of the
    paper's transformer variants)."""
    if rng.random() < 0.5:
        layers = rng.randint(1, 3)
        widths = [rng.choice((8, 16, 32)) for _ in range(layers + 1)]
        return modelgen.build_mlp(layers, tuple(widths), rng.choice((4, 8)),
                                  (("model", 2),))
    toy = dict(modelgen.TOY)
    return modelgen.build_transformer(rng.randint(1, 2), mesh=(("model", 2),), **toy)


def label_program(text: str, evaluate, budget_frac: float = 0.8, group: bool = True):
    """Labels = arguments tiled by the reward-optimal single decision under a
    memory budget of `budget_frac` x the replicated peak (the paper's regime,
    in which replication is infeasible; at 0.6 most desk-scale programs have
    no feasible single decision and the label would be empty).  `evaluate(text, seqs, cost)`
    returns pe_result objects (GPU engine or oracle)."""
    cands = single_action_candidates(text, group)
    seqs = [[]] + [c[0] for c in cands]
    cp = capi.default_cost_params()
    base = evaluate(text, [[]], cp)[0]
    cp.memory_budget_bytes = max(1, int(budget_frac * base.peak_bytes))
    res = evaluate(text, seqs, cp)
    best = max(range(len(seqs)), key=lambda i: (res[i].reward, -i))
    return set() if best == 0 else set(cands[best - 1][1])


def generate_dataset(n_programs: int, seed: int, evaluate, group: bool = True):
    """SPEC generate_dataset: [(GraphEncoding, label set)] for n sampled
    programs, reproducible for a seed."""
    rng = random.Random(seed)
    data = []
    for _ in range(n_programs):
        text = sample_program(rng)
        data.append((featurize(text), sorted(label_program(text, evaluate, group=group))))
    return data


def engine_evaluator(device: int = 0):
    """evaluate() on the GPU engine (one batched launch per program)."""
    from . import engine

    def ev(text, seqs, cp):
        eng = engine.Engine(engine.Graph(text), device=device, cost=cp)
        return eng.eval_batch(seqs)
    return ev


# ---------------------------------------------------------------- model file
def save_model(model: RankerModel, path: str) -> None:
    with open(path, "w") as f:
        f.write(f"{MODEL_MAGIC}\nfeatures {N_FEATURES} hidden {HIDDEN} rounds {ROUNDS}\n")
        for k in RankerModel.BLOCKS:
            v = model.p[k]
            f.write(f"{k} {' '.join(str(d) for d in v.shape)}\n")
            f.write(" ".join(repr(float(x)) for x in v.ravel()) + "\n")


def load_model(path: str) -> RankerModel:
    with open(path) as f:
        lines = f.read().splitlines()
    if not lines or lines[0] != MODEL_MAGIC:
        raise ValueError(f"{path}: not a {MODEL_MAGIC} model file")
    hdr = lines[1].split()
    if int(hdr[1]) != N_FEATURES or int(hdr[3]) != HIDDEN or int(hdr[5]) != ROUNDS:
        raise ValueError(f"{path}: model dimensions {hdr} do not match this build")
    m = RankerModel.__new__(RankerModel)
    m.p = {}
    m.final_loss = None
    i = 2
    for k in RankerModel.BLOCKS:
        name, *dims = lines[i].split()
        if name != k:
            raise ValueError(f"{path}: expected block {k}, found {name}")
        vals = np.array([float(t) for t in lines[i + 1].split()])
        m.p[k] = vals.reshape(tuple(int(d) for d in dims))
        i += 2
    return m
