"""Time rollout throughput of several builds of the engine library (device
timing with CUDA events).  python tools/variant_bench.py lib1.so lib2.so ..."""
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2112_02958_b200 import capi, engine, modelgen  # noqa: E402

B = int(os.environ.get("B", "65536"))
text = modelgen.config_program(int(os.environ.get("CFG", "3")))
for path in sys.argv[1:]:
    capi._lib = capi.load(path)
    capi._lib = None
    lib = capi.load(path)
    capi._lib = lib
    g = engine.Graph(text)
    eng = engine.Engine(g, cfg=capi.default_search_config(group_scopes=1))
    dev = torch.device("cuda", 0)
    maxd = 32
    seeds = torch.arange(B, dtype=torch.int64, device=dev)
    poff = torch.zeros(B + 1, dtype=torch.int32, device=dev)
    acts = torch.empty(B * maxd * 8, dtype=torch.uint8, device=dev)
    na = torch.empty(B, dtype=torch.int32, device=dev)
    res = torch.empty(B * 192, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream()
    sp = C.c_void_p(st.cuda_stream)

    def run(k):
        eng.rollout_batch_device(None, poff.data_ptr(), (seeds + k * B).data_ptr(), B,
                                 acts.data_ptr(), na.data_ptr(), res.data_ptr(), stream=sp)
    for _w in range(int(os.environ.get("WARM", "1"))):
        run(100 + _w)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for k in range(3):
        run(k)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"{os.path.basename(path)}: slots {eng.slots()} arena {eng.arena_bytes()} "
          f"{B / ms * 1e3:.0f} cand/s ({ms:.1f} ms / {B})", flush=True)
    del eng, g
