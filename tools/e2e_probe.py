"""Where the e2e time goes: host-mode pe_rollout_batch calls (pinned buffers)
with and without the per-step host seed generation, next to device mode.
python tools/e2e_probe.py"""
import ctypes as C
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2112_02958_b200 import capi, engine, modelgen  # noqa: E402

B = 262144
maxd = 32
eng = engine.Engine(engine.Graph(modelgen.config_program(3)),
                    cfg=capi.default_search_config(group_scopes=1))
lib = eng.lib
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream()
sp = C.c_void_p(st.cuda_stream)
pin_seeds = torch.empty(B, dtype=torch.int64).pin_memory()
pin_poff = torch.zeros(B + 1, dtype=torch.int32).pin_memory()
pin_acts = torch.empty(B * maxd * 8, dtype=torch.uint8).pin_memory()
pin_nacts = torch.empty(B, dtype=torch.int32).pin_memory()
pin_res = torch.empty(B * 192, dtype=torch.uint8).pin_memory()
err = capi.PeError()


def host_call(i, gen):
    if gen:
        pin_seeds.copy_(torch.arange(B, dtype=torch.int64) + 7_000_000 * (i + 1))
    rc = lib.pe_rollout_batch(eng.h, None, C.c_void_p(pin_poff.data_ptr()),
                              C.c_void_p(pin_seeds.data_ptr()), B, C.c_void_p(pin_acts.data_ptr()),
                              C.c_void_p(pin_nacts.data_ptr()), C.c_void_p(pin_res.data_ptr()),
                              None, 0, sp, C.byref(err))
    assert rc == 0


for w in range(4):
    host_call(100 + w, True)
for gen in (True, False):
    t0 = time.perf_counter()
    for i in range(5):
        host_call(i, gen)
    dt = (time.perf_counter() - t0) / 5
    print(f"host mode, seed generation {'in' if gen else 'out of'} the loop: {dt * 1e3:.1f} ms/call "
          f"= {B / dt:.0f} cand/s", flush=True)
sd = torch.arange(B, dtype=torch.int64, device=dev) + 5
poff = torch.zeros(B + 1, dtype=torch.int32, device=dev)
acts = torch.empty(B * maxd * 8, dtype=torch.uint8, device=dev)
na = torch.empty(B, dtype=torch.int32, device=dev)
res = torch.empty(B * 192, dtype=torch.uint8, device=dev)
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(5):
    eng.rollout_batch_device(None, poff.data_ptr(), (sd + i * B).data_ptr(), B, acts.data_ptr(),
                             na.data_ptr(), res.data_ptr(), stream=sp)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 5
print(f"device mode (wall): {dt * 1e3:.1f} ms/call = {B / dt:.0f} cand/s")
t = time.perf_counter()
pin_seeds.copy_(torch.arange(B, dtype=torch.int64) + 3)
print(f"host seed generation alone: {(time.perf_counter() - t) * 1e3:.2f} ms")

# bench.py's order: device steps, then host calls without a host warm-up
print("per-call host times right after device steps:")
for i in range(5):
    t = time.perf_counter()
    host_call(50 + i, True)
    print(f"  call {i}: {(time.perf_counter() - t) * 1e3:.1f} ms  (trie nodes {eng.sched_nodes()})")
