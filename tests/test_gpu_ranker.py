"""Ranker dataset generation on the GPU engine (SPEC generate_dataset's
exhaustive single-decision labels, evaluated in one batched launch per
program) and a trained model's held-out recall."""
import pytest

import helpers as H
from paper_2112_02958_b200 import modelgen, ranker

pytestmark = pytest.mark.gpu


def test_engine_labels_equal_oracle_labels(oracle_lib):
    ev_gpu = ranker.engine_evaluator(0)

    def ev_oracle(text, seqs, cp):
        return H.eval_batch("oracle", text, seqs, cp=cp)[0]

    import random
    rng = random.Random(11)
    for _ in range(6):
        text = ranker.sample_program(rng)
        assert ranker.label_program(text, ev_gpu) == ranker.label_program(text, ev_oracle)
    assert ranker.label_program(modelgen.linear(), ev_gpu) == {1}


def test_trained_ranker_recall_on_held_out_programs():
    ev = ranker.engine_evaluator(0)
    train = ranker.generate_dataset(24, seed=1, evaluate=ev)
    held = ranker.generate_dataset(12, seed=2, evaluate=ev)
    m = ranker.train(train, epochs=300, seed=0)
    assert m.final_loss < ranker.train(train, epochs=0, seed=0).final_loss

    def recall(k):
        hits = sum(1 for enc, lab in held if set(lab) <= set(ranker.score_and_filter(enc, m, k)))
        return hits / len(held)
    assert recall(25) >= 0.9  # SPEC: top-k contains all oracle-tiled args in >= 90%
    assert recall(3) >= 0.5
