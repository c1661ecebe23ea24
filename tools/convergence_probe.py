"""Upper-bound probe: rollouts whose seeds repeat within each warp (lanes of
a warp evaluate identical candidates -> perfect SIMT convergence and
coalesced interleaved-arena accesses) vs distinct seeds."""
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2112_02958_b200 import capi, engine, modelgen  # noqa: E402

B = int(os.environ.get("B", "262144"))
text = modelgen.config_program(int(os.environ.get("CFG", "3")))
eng = engine.Engine(engine.Graph(text), cfg=capi.default_search_config(group_scopes=1))
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream()
sp = C.c_void_p(st.cuda_stream)
poff = torch.zeros(B + 1, dtype=torch.int32, device=dev)
acts = torch.empty(B * 32 * 8, dtype=torch.uint8, device=dev)
na = torch.empty(B, dtype=torch.int32, device=dev)
res = torch.empty(B * 192, dtype=torch.uint8, device=dev)
for name, seeds in (("distinct", torch.arange(B, dtype=torch.int64, device=dev)),
                    ("warp-identical", torch.arange(B, dtype=torch.int64, device=dev) // 32)):
    eng.rollout_batch_device(None, poff.data_ptr(), seeds.data_ptr(), B, acts.data_ptr(),
                             na.data_ptr(), res.data_ptr(), stream=sp)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    eng.rollout_batch_device(None, poff.data_ptr(), seeds.data_ptr(), B, acts.data_ptr(),
                             na.data_ptr(), res.data_ptr(), stream=sp)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{name}: {B / ms * 1e3:.0f} cand/s ({ms:.1f} ms)", flush=True)

# first-action grouping: the root's legal set is shared, so each rollout's
# first pick is a function of its seed alone; order seeds by first pick
M = (1 << 64) - 1


def first_pick(s, nl):
    st = (s + 0x9E3779B97F4A7C15) & M
    z = st
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    z = z ^ (z >> 31)
    return z % (nl + 1)


r, s, lg = eng.rollout_batch([[]], [0], legal=True)
nl = sum(bin(w).count("1") for w in lg[0])
base = list(range(B))
srt = sorted(base, key=lambda s: first_pick(s, nl))
seeds = torch.tensor(srt, dtype=torch.int64, device=dev)
eng.rollout_batch_device(None, poff.data_ptr(), seeds.data_ptr(), B, acts.data_ptr(),
                         na.data_ptr(), res.data_ptr(), stream=sp)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(st)
eng.rollout_batch_device(None, poff.data_ptr(), seeds.data_ptr(), B, acts.data_ptr(),
                         na.data_ptr(), res.data_ptr(), stream=sp)
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"first-action-grouped (nl={nl}): {B / ms * 1e3:.0f} cand/s ({ms:.1f} ms)", flush=True)
