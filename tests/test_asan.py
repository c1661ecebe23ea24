"""Memory-safety check of the evaluation core on the CPU (the stand-in for
compute-sanitizer, which this GPU pool does not offer): the host build of
pe_core.cuh with arena bounds checks (PE_BOUNDS_CHECK) and the oracle, both
under AddressSanitizer + UBSan, run the differential fuzz against each other.
Any out-of-bounds access, use-after-free or undefined behaviour aborts the
child run."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBS = ["/usr/lib/x86_64-linux-gnu/libasan.so.8", "/usr/lib/x86_64-linux-gnu/libubsan.so.1"]


def test_core_fuzz_under_asan_ubsan(oracle_lib):
    if not all(os.path.exists(p) for p in LIBS) or not os.path.isdir("/root/reference/proj"):
        pytest.skip("sanitizer runtimes or the reference tree not available")
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "-j8", "asan"])
    env = dict(os.environ, PE_ASAN="1", LD_PRELOAD=" ".join(LIBS),
               ASAN_OPTIONS="detect_leaks=0:abort_on_error=1",
               UBSAN_OPTIONS="halt_on_error=1:print_stacktrace=1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_core_fuzz.py"),
                        os.path.join(ROOT, "tests", "test_snapshot.py"),
                        "-k", "random_programs or illegal or resume"],
                       env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    assert "passed" in r.stdout
