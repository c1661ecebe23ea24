"""Where a rollout launch spends its time: per schedule position the start /
end %globaltimer (profiling build with -DPE_CAND_TIMES; never the product
library).  Build: tools/build_variants.sh times "-DPE_CAND_TIMES"
Run on a GPU box: B=262144 python tools/tail_profile.py variants/times.so"""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2112_02958_b200 import capi, engine, modelgen  # noqa: E402

B = int(os.environ.get("B", "262144"))
lib = capi.load(sys.argv[1])
capi._lib = lib
lib.pe_debug_cand_times.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32]
g = engine.Graph(modelgen.config_program(int(os.environ.get("CFG", "3"))))
eng = engine.Engine(g, cfg=capi.default_search_config(group_scopes=1))
dev = torch.device("cuda", 0)
maxd = 32
seeds = torch.arange(B, dtype=torch.int64, device=dev)
poff = torch.zeros(B + 1, dtype=torch.int32, device=dev)
acts = torch.empty(B * maxd * 8, dtype=torch.uint8, device=dev)
na = torch.empty(B, dtype=torch.int32, device=dev)
res = torch.empty(B * 192, dtype=torch.uint8, device=dev)
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for k in range(4):
    eng.rollout_batch_device(None, poff.data_ptr(), (seeds + (100 + k) * B).data_ptr(), B,
                             acts.data_ptr(), na.data_ptr(), res.data_ptr(), stream=sp)
torch.cuda.synchronize()
eng.rollout_batch_device(None, poff.data_ptr(), seeds.data_ptr(), B, acts.data_ptr(),
                         na.data_ptr(), res.data_ptr(), stream=sp)
torch.cuda.synchronize()
t = np.zeros(2 * B, dtype=np.uint64)
sm = np.zeros(B, dtype=np.uint32)
assert lib.pe_debug_cand_times(t.ctypes.data, sm.ctypes.data, B) == 0
t = t.reshape(B, 2).astype(np.int64)
t -= t[:, 0].min()
st, en = t[:, 0] / 1e6, t[:, 1] / 1e6  # ms, by schedule position
lat = en - st
nsteps = na.cpu().numpy()  # by candidate; schedule order unknown here, report overall
slots = eng.slots()
span = en.max()
print(f"B={B} slots={slots} span {span:.1f} ms  -> {B / span * 1e3:.0f} cand/s")
print(f"last start {st.max():.1f} ms; first-wave end min/med/max "
      f"{en[:slots].min():.1f}/{np.median(en[:slots]):.1f}/{en[:slots].max():.1f} ms")
for name, sel in (("first wave", slice(0, slots)), ("later", slice(slots, B))):
    x = lat[sel]
    if x.size:
        print(f"{name:10s} latency mean {x.mean():.1f} p50 {np.median(x):.1f} "
              f"p90 {np.percentile(x, 90):.1f} p99 {np.percentile(x, 99):.1f} max {x.max():.1f} ms")
# latency by schedule-position decile (trie order: deep nodes first)
for d in range(10):
    a, b = d * B // 10, (d + 1) * B // 10
    print(f"  positions {a:7d}-{b:7d}: start med {np.median(st[a:b]):5.1f} "
          f"latency med {np.median(lat[a:b]):5.1f} max {lat[a:b].max():5.1f} ms")
# running candidates over time
bins = np.arange(0, span + 2, 2.0)
for b0 in bins[::2]:
    run = int(((st <= b0) & (en > b0)).sum())
    print(f"  t={b0:5.1f} ms running {run:7d} ({run / slots:5.1%} of slots)")
hist = np.bincount(nsteps, minlength=33)
print("decisions histogram:", {k: int(v) for k, v in enumerate(hist) if v})
# per-SM finish time spread
smend = np.zeros(sm.max() + 1)
np.maximum.at(smend, sm, en)
print(f"per-SM last end min/med/max {smend.min():.1f}/{np.median(smend):.1f}/{smend.max():.1f} ms")
