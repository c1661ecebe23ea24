import sys, time, os
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import torch
from paper_2112_02958_b200 import engine, modelgen, capi
for cfgno in (2, 3):
    text = modelgen.config_program(cfgno)
    cfg = capi.default_search_config(group_scopes=1)
    t=time.time(); eng = engine.Engine(engine.Graph(text), cfg=cfg); 
    print("cfg", cfgno, "engine create %.2fs"%(time.time()-t), "arena", eng.arena_bytes(), "slots", eng.slots())
    for n in (1024, 8192, 32768):
        seeds=list(range(n))
        eng.rollout_batch([[]]*min(n,64), seeds[:min(n,64)])
        torch.cuda.synchronize()
        t=time.time(); res, seqs, _ = eng.rollout_batch([[]]*n, seeds); dt=time.time()-t
        print(f"  n={n} {n/dt:.0f} cand/s  ({dt*1e3:.1f} ms)  mean steps {sum(r.n_steps for r in res)/n:.2f} status0 {sum(r.status==0 for r in res)}")
import helpers as H
text = modelgen.config_program(3)
cfg = capi.default_search_config(group_scopes=1)
n=32
t=time.time(); H.rollout_batch("oracle", text, [[]]*n, list(range(n)), cfg, threads=os.cpu_count()); dt=time.time()-t
print(f"oracle cfg3 {os.cpu_count()} threads: {n/dt:.2f} cand/s")
text = modelgen.config_program(2)
n=512
t=time.time(); H.rollout_batch("oracle", text, [[]]*n, list(range(n)), cfg, threads=os.cpu_count()); dt=time.time()-t
print(f"oracle cfg2 {os.cpu_count()} threads: {n/dt:.2f} cand/s")
