"""Throughput with candidates grouped by their first decision (predicted
from the seed: at the root every candidate has the same legal set, so the
first pick is splitmix64(seed) % (n_legal + 1)).  Results are independent of
the order; only SIMT convergence changes.  python tools/group_probe.py"""
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2112_02958_b200 import capi, engine, modelgen  # noqa: E402

M64 = (1 << 64) - 1


def splitmix(st):
    st = (st + 0x9E3779B97F4A7C15) & M64
    z = st
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


B = int(os.environ.get("B", "262144"))
text = modelgen.config_program(3)
eng = engine.Engine(engine.Graph(text), cfg=capi.default_search_config(group_scopes=1))
_, _, legal = eng.rollout_batch([[]], [0], legal=True)
nl = sum(bin(w).count("1") for w in legal[0])
print("root legal", nl)
dev = torch.device("cuda", 0)
maxd = 32
seeds_plain = list(range(10_000_000, 10_000_000 + B))
first = [splitmix(s) % (nl + 1) for s in seeds_plain]
seeds_sorted = [s for _, s in sorted(zip(first, seeds_plain))]
for name, seeds in (("plain", seeds_plain), ("grouped", seeds_sorted), ("plain", seeds_plain),
                    ("grouped", seeds_sorted)):
    sd = torch.tensor(seeds, dtype=torch.int64, device=dev)
    poff = torch.zeros(B + 1, dtype=torch.int32, device=dev)
    acts = torch.empty(B * maxd * 8, dtype=torch.uint8, device=dev)
    na = torch.empty(B, dtype=torch.int32, device=dev)
    res = torch.empty(B * 192, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream()
    sp = C.c_void_p(st.cuda_stream)

    def run():
        eng.rollout_batch_device(None, poff.data_ptr(), sd.data_ptr(), B, acts.data_ptr(),
                                 na.data_ptr(), res.data_ptr(), stream=sp)
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(3):
        run()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"{name}: {B / ms * 1e3:.0f} cand/s ({ms:.1f} ms)", flush=True)

# deeper keys: the legal set after a prefix is the same for every candidate
# that took it, so one evaluation per distinct prefix predicts the next pick
GOLD = 0x9E3779B97F4A7C15


def legal_list(prefix):
    _, _, lg = eng.rollout_batch([prefix], [0], legal=True)
    return [o for o in range(eng.n_ordinals) if (lg[0][o // 64] >> (o % 64)) & 1]


def act(o):
    a = eng.ordinal_action(o)
    return (a.value, a.dim, a.axis, a.kind)


cache = {(): legal_list([])}


def keys(seed, depth):
    prefix, key = [], []
    for step in range(depth):
        lg = cache.get(tuple(prefix))
        if lg is None:
            lg = cache[tuple(prefix)] = legal_list(prefix)
        ws = 2 if step >= 1 else 1
        if not lg:
            break
        pick = splitmix((seed + step * GOLD) & M64) % (len(lg) + ws)
        if pick >= len(lg):
            key.append(1 << 30)
            break
        key.append(lg[pick])
        prefix.append(act(lg[pick]))
    return tuple(key)


for depth in (2, 3):
    ks = [keys(s, depth) for s in seeds_plain]
    seeds_d = [s for _, s in sorted(zip(ks, seeds_plain))]
    print(f"depth {depth}: {len(cache)} prefix states probed, {len(set(ks))} keys", flush=True)
    sd = torch.tensor(seeds_d, dtype=torch.int64, device=dev)
    run()
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(3):
        run()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"grouped depth {depth}: {B / ms * 1e3:.0f} cand/s ({ms:.1f} ms)", flush=True)
