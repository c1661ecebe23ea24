import ctypes as C, os, sys, time
sys.path.insert(0, '.')
import torch
from paper_2112_02958_b200 import capi, engine, modelgen
B = 262144
text = modelgen.config_program(3)
eng = engine.Engine(engine.Graph(text), cfg=capi.default_search_config(group_scopes=int(os.environ.get("GROUP", "1"))))
dev = torch.device("cuda", 0)
maxd = 32
poff = torch.zeros(B + 1, dtype=torch.int32, device=dev)
acts = torch.empty(B * maxd * 8, dtype=torch.uint8, device=dev)
na = torch.empty(B, dtype=torch.int32, device=dev)
res = torch.empty(B * 192, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream(); sp = C.c_void_p(st.cuda_stream)
for k in range(int(os.environ.get("CALLS", "7"))):
    sd = torch.arange(B, dtype=torch.int64, device=dev) + 10_000_000 + k * B
    torch.cuda.synchronize(); t = time.time()
    eng.rollout_batch_device(None, poff.data_ptr(), sd.data_ptr(), B, acts.data_ptr(), na.data_ptr(), res.data_ptr(), stream=sp)
    torch.cuda.synchronize(); dt = time.time() - t
    print(k, "nodes", eng.sched_nodes(), f"{B/dt:.0f} cand/s ({dt*1e3:.1f} ms)", flush=True)
