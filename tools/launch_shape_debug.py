"""Debug: which side of a launch-shape mismatch agrees with the oracle."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import helpers as H
from paper_2112_02958_b200 import capi, engine, modelgen
from test_gpu_launch_shape import _rows_equal, _seqs, N_FULL, WAVE

cfgno = int(sys.argv[1]) if len(sys.argv) > 1 else 2
text = modelgen.config_program(cfgno)
cfg = capi.default_search_config(group_scopes=1)
eng = engine.Engine(engine.Graph(text), device=0, cfg=cfg)
seeds = np.arange(N_FULL, dtype=np.uint64) + np.uint64(1_000_003)
eng.rollout_roots_np(seeds[:N_FULL // 2] + np.uint64(9_999_999))
rf, af, nf = eng.rollout_roots_np(seeds)
parts = [eng.rollout_roots_np(seeds[i:i + WAVE]) for i in range(0, N_FULL, WAVE)]
rw = np.concatenate([p[0] for p in parts]); aw = np.concatenate([p[1] for p in parts]); nw = np.concatenate([p[2] for p in parts])
bad = _rows_equal(rf, af, nf, rw, aw, nw)
print("bad", bad.size, bad[:40])
rf2, af2, nf2 = eng.rollout_roots_np(seeds)
print("full vs full again:", _rows_equal(rf, af, nf, rf2, af2, nf2).size)
idx = bad[:24]
ref, rseqs, _ = H.rollout_batch("oracle", text, [[]] * len(idx), [int(s) for s in seeds[idx]], cfg, threads=os.cpu_count())
for j, k in enumerate(idx):
    F = capi.PeResult.from_buffer_copy(rf[k].tobytes()); W = capi.PeResult.from_buffer_copy(rw[k].tobytes())
    sf = _seqs(af[k:k+1], nf[k:k+1])[0]; sw = _seqs(aw[k:k+1], nw[k:k+1])[0]
    print(k, "full==oracle", sf == rseqs[j] and not H.compare_results(F, ref[j]),
          "wave==oracle", sw == rseqs[j] and not H.compare_results(W, ref[j]),
          "seq full", sf, "wave", sw, "oracle", rseqs[j], H.compare_results(F, W)[:4])
for k in idx[:6]:
    d = np.nonzero(rf[k] != rw[k])[0]
    print(k, "byte offsets", d, rf[k][d], rw[k][d], "fields", [n for n, _ in capi.PeResult._fields_ if any(getattr(capi.PeResult, n).offset <= x < getattr(capi.PeResult, n).offset + getattr(capi.PeResult, n).size for x in d)])
    F = capi.PeResult.from_buffer_copy(rf[k].tobytes()); W = capi.PeResult.from_buffer_copy(rw[k].tobytes())
    print(repr(F.runtime_s), repr(W.runtime_s), repr(F.reward), repr(W.reward))
