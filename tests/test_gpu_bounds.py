"""Device-side memory checking (compute-sanitizer is not available on this
GPU pool): the engine built with PE_BOUNDS_CHECK traps on any arena access
outside the candidate's group arena.  Every kernel runs under it
(tools/sanitize_workload.py: scheduled root rollouts including a launch
beyond the resident slots, prefix rollouts, traced evaluations, InferRest
pauses/resumes, the prefix-state cache, pe_state handles, the retry path),
and the instrumented run must still match the oracle samples it checks."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("big", ["0", "1"])
def test_every_kernel_inside_its_arena(oracle_lib, big):
    sys.path.insert(0, ROOT)
    import __graft_entry__ as ge
    lib = ge.build_debug()
    env = dict(os.environ, PE_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_workload.py"), big],
                       env=env, capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-3000:])
    assert "SANITIZE WORKLOAD DONE" in r.stdout
