"""bench.py contract on the CPU: the reference arm runs the reference CPU
path, prints one JSON line with the contract keys, and under torchrun
(world size 2, gloo) only rank 0 prints."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(cmd, env=None):
    e = dict(os.environ)
    e.update(env or {})
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600, env=e)
    assert r.returncode == 0, r.stderr[-3000:]
    return [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]


def test_reference_arm_single(oracle_lib):
    lines = _run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                  "--warmup", "0"])
    assert len(lines) == 1
    d = lines[0]
    assert d["impl"] == "reference" and d["unit"] == "candidates/s" and d["value"] > 0
    assert d["higher_is_better"] is True and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1


def test_reference_arm_torchrun_two_ranks(oracle_lib):
    port = str(29700 + os.getpid() % 200)
    lines = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                  "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port", port,
                  "bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1",
                  "--warmup", "0"], env={"CUDA_VISIBLE_DEVICES": ""})
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2
