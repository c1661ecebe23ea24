"""Per-phase clock64 breakdown of the rollout kernel (profiling build with
-DPE_PHASE_TIMERS; never the product library).  Usage on a GPU box:
  python tools/phase_profile.py [batch]"""
import ctypes as C
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__ as G  # noqa: E402

PROF = os.path.join(ROOT, "paper_2112_02958_b200", "libpe_b200_prof.so")
if not os.path.exists(PROF) or os.path.getmtime(PROF) < os.path.getmtime(G.LIB):
    cmd = [G.NVCC, *[f for f in G.NVCC_FLAGS if f != "-v" and f != "-Xptxas"], "-DPE_PHASE_TIMERS",
           "-shared", "-I", os.path.join(ROOT, "include"), "-I", G.CSRC,
           *[os.path.join(G.CSRC, s) for s in G.SOURCES], "-o", PROF]
    subprocess.check_call(cmd)
from paper_2112_02958_b200 import capi, engine, modelgen  # noqa: E402

lib = capi.load(PROF)
capi._lib = lib
lib.pe_debug_phase_cycles.argtypes = [C.c_void_p, C.c_int]
names = ["init", "apply", "forward", "backward", "wrap", "legal", "analyze", "lower", "score"]
B = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
for cfgno in (3,):
    text = modelgen.config_program(cfgno)
    eng = engine.Engine(engine.Graph(text), cfg=capi.default_search_config(group_scopes=1))
    for w in range(4):  # warm the scheduling trie with full-size calls
        eng.rollout_batch([[]] * B, list(range(10_000_000 + w * B, 10_000_000 + (w + 1) * B)))
    buf = (C.c_ulonglong * 9)()
    lib.pe_debug_phase_cycles(buf, 1)
    t = time.time()
    res, seqs, _ = eng.rollout_batch([[]] * B, list(range(B)))
    dt = time.time() - t
    lib.pe_debug_phase_cycles(buf, 1)
    tot = sum(buf)
    print(f"cfg{cfgno} B={B} {B/dt:.0f} cand/s (host timed); cycles/cand {tot/B:.3g}")
    for n, v in zip(names, buf):
        print(f"  {n:9s} {100*v/tot:5.1f}%  {v/B:10.4g} cyc/cand")
