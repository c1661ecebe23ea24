"""The reference-side binding of INTEGRATION.md, compiled against the
reference's own headers (partir::Program) and linked with the reference
(oracle/_ref, test infrastructure) and libpe_b200.so: a reference Program
walked into pe_graph_create_from_arrays equals the same Program printed by
the reference and read by pe_graph_create (tests/native/binding_example.cc).
Host-side only; no GPU."""
import os
import subprocess

import pytest

from paper_2112_02958_b200 import modelgen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = os.path.join(ROOT, "oracle", "_ref", "src", "include")
ORACLE = os.path.join(ROOT, "oracle", "_ref")
PKG = os.path.join(ROOT, "paper_2112_02958_b200")
EXE = os.path.join(ROOT, "tests", "native", "_build", "binding_example")


def _build():
    src = os.path.join(ROOT, "tests", "native", "binding_example.cc")
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    subprocess.check_call(["/usr/bin/g++", "-std=c++20", "-O1", "-I", REF_INC, "-I",
                           os.path.join(ROOT, "include"), src, "-L", ORACLE, "-loracle", "-L", PKG,
                           "-lpe_b200", f"-Wl,-rpath,{ORACLE}:{PKG}", "-o", EXE])


@pytest.mark.parametrize("cfgno", [1, 2, 3, 4])
def test_reference_program_through_the_array_binding(oracle_lib, tmp_path, cfgno):
    if not os.path.isdir(REF_INC):
        pytest.skip("reference headers not available")
    src = os.path.join(ROOT, "tests", "native", "binding_example.cc")
    lib = os.path.join(PKG, "libpe_b200.so")
    if not os.path.exists(EXE) or os.path.getmtime(EXE) < max(os.path.getmtime(src),
                                                               os.path.getmtime(lib)):
        _build()
    f = tmp_path / "p.pir"
    f.write_text(modelgen.config_program(cfgno))
    r = subprocess.run([EXE, str(f)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, (r.stdout, r.stderr)
    assert r.stdout.startswith("OK")


@pytest.mark.gpu
def test_drop_in_evaluation_matches_the_reference_in_process(oracle_lib, tmp_path):
    # the reference's apply_tile_action + propagate + lower_to_spmd +
    # collective_stats and pe_eval_batch, side by side in one C++ process
    if not os.path.isdir(REF_INC):
        pytest.skip("reference headers not available")
    src = os.path.join(ROOT, "tests", "native", "binding_example.cc")
    if not os.path.exists(EXE) or os.path.getmtime(EXE) < os.path.getmtime(src):
        _build()
    f = tmp_path / "p.pir"
    f.write_text(modelgen.build_transformer(2, mesh=(("batch", 2), ("model", 2)), **modelgen.TOY))
    seqs = ["l0_wq:1:model", "l0_wq:1:model,l0_w1:1:model", "x:0:batch",
            "l1_w2:0:model,l0_wk:2:model", "l0_wo:0:model,x:2:batch"]
    r = subprocess.run([EXE, str(f), "eval", *seqs], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, (r.stdout, r.stderr)
    assert "EVAL OK" in r.stdout
