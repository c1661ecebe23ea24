"""Differential fuzz driver shared by the CPU and GPU parity tests."""
from __future__ import annotations

from paper_2112_02958_b200 import modelgen

MESHES = ((("m", 2),), (("a", 2), ("b", 4)), (("m", 8),))
# non-power-of-two axis sizes (the device divides by them with 32-bit
# division instead of shifts), with dims drawn to be divisible by them
ODD_MESHES = ((("m", 3),), (("a", 3), ("b", 2)), (("m", 6),))
ODD_DIMS = (3, 6, 12)


def corpus(n_programs: int, seed0: int = 0, seqs_per_program: int = 4):
    """Yields (text, mesh, [action sequences])."""
    for i in range(n_programs):
        mesh = MESHES[i % len(MESHES)]
        text = modelgen.random_program(seed0 + i, mesh)
        seqs = [modelgen.random_actions((seed0 + i) * 7919 + k, text, mesh)
                for k in range(seqs_per_program)]
        yield text, mesh, seqs


def first_trace_diff(a, b):
    n = max(abs(a[0]), abs(b[0]))
    for i in range(n):
        if a[i] != b[i]:
            return i
    return -1


def legal_sequences(text, mesh, seed, n_seqs=4, max_len=6, tries=8):
    """Random action sequences whose every step is legal per the oracle
    (illegal candidates are resampled), so the fuzz reaches deep states."""
    import random

    import helpers as H
    rng = random.Random(seed)
    names, shapes = modelgen.program_values(text)
    out = []
    for _ in range(n_seqs):
        seq = []
        for _ in range(rng.randint(1, max_len)):
            cands = []
            for _ in range(tries):
                v = rng.randrange(len(names))
                if not shapes[v]:
                    continue
                ax = rng.randrange(len(mesh))
                dims = [d for d in range(len(shapes[v])) if shapes[v][d] % mesh[ax][1] == 0]
                if not dims:
                    continue
                cands.append((v, rng.choice(dims), ax, 0))
            if not cands:
                break
            res, _ = H.eval_batch("oracle", text, [seq + [c] for c in cands])
            ok = [c for c, r in zip(cands, res) if r.status != 1]
            if not ok:
                break
            seq.append(ok[0])
        out.append(seq)
    return out
