"""Semantics preservation of partitioning plans (SPEC acceptance 2 and
§8(f) rank 3): the reference interpreter (REF interp.cc:640-678,
check_equivalence) runs the lowered SPMD program on a simulated device mesh
and compares it with the original program on seeded random inputs.  The
engine is bit-exact with the oracle on these programs and sequences
(test_core_fuzz / test_gpu_parity), so its plans inherit the property."""
import fuzz_util as F
import helpers as H
from paper_2112_02958_b200 import capi, engine, modelgen, search
from test_search import TWO_LAYER, evaluator, megatron, setup


def test_fuzzed_plans_preserve_semantics(oracle_lib):
    # SPEC acceptance 2: >= 200 fuzzed (program, legal action sequence) pairs
    n = 0
    for i in range(60):
        mesh = F.MESHES[i % 3]
        text = modelgen.random_program(20000 + i, mesh)
        for seq in F.legal_sequences(text, mesh, 777 + i, n_seqs=4):
            ok, diff, _ = H.oracle_check_equivalence(text, seq, trials=2, seed=i)
            assert ok, (i, seq, diff)
            n += 1
    assert n >= 200


def test_searched_plan_preserves_semantics(oracle_lib, harness_lib):
    text = modelgen.build_transformer(**TWO_LAYER)
    g, cfg, cp, ords, lw = setup(text)
    p = search.run_mcts(evaluator("harness", text, cfg, cp, lw), len(ords) - 1, ords,
                        episodes=300, seed=2, leaf_batch=32)
    assert megatron(p.result, 2)
    ok, diff, order_preserving = H.oracle_check_equivalence(text, search.plan_actions(p), trials=3)
    assert ok and not order_preserving  # Megatron has all_reduces: 1e-5 tolerance path


def test_axis_division_magic_is_exact():
    # pe_graph_view.h aquo/amod: x / d == (x * m) >> s for 0 <= x < 2^31,
    # m = ceil(2^s / d), s = 31 + ceil(log2 d) (same constants as
    # pe_graph.cc host_view)
    import random
    rng = random.Random(5)
    ds = list(range(1, 4097)) + [rng.randrange(4097, 2**31) for _ in range(2000)] + [2**31 - 1, 2**30,
                                                                                      2**30 + 1]
    for d in ds:
        lg = (d - 1).bit_length()
        s = 31 + lg
        m = -(-(1 << s) // d)
        assert m < 2**32
        xs = [0, 1, d - 1, d, d + 1, 2**31 - 1, (2**31 - 1) // d * d, (2**31 - 1) // d * d - 1]
        xs += [rng.randrange(0, 2**31) for _ in range(20)]
        for x in xs:
            if 0 <= x < 2**31:
                assert (x * m) >> s == x // d, (d, x)
