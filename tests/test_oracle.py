"""Pin the CPU oracle (oracle/criterion_oracle.py) to the reference's own outputs.

The fixtures under tests/golden/ were produced by running the reference
(asrkit.criterion, /root/reference/pkg/src/asrkit/criterion.py) and its
brute-force oracles (tests/oracles.py) -- see tests/golden/make_golden.py.
No GPU needed.
"""

import math

import numpy as np
import pytest

from oracle import criterion_oracle as orc

from conftest import load_kat, load_npz


def test_ctc_known_answers():
    kat = load_kat()
    for case in kat["ctc"]:
        e = np.asarray(case["e"])
        loss, grad = orc.ctc(e, case["y"], case["blank"])
        assert abs(loss - case["loss"]) < 1e-12
        assert abs(loss - case["enum"]) < 1e-5          # test_criterion.py:83-94
        assert np.array_equal(grad, np.asarray(case["grad"], np.float32)) or \
            np.abs(grad - np.asarray(case["grad"])).max() < 1e-6


def test_asg_known_answers():
    kat = load_kat()
    for case in kat["asg"]:
        e = np.asarray(case["e"])
        a = np.asarray(case["a"], np.float32)
        loss, ge, ga = orc.asg(e, case["y"], a)
        assert abs(loss - case["loss"]) < 1e-12
        assert abs(loss - case["enum"]) < 1e-5          # test_criterion.py:97-103
        assert np.abs(ge - np.asarray(case["grad_e"])).max() < 1e-6
        assert np.abs(ga - np.asarray(case["grad_a"])).max() < 1e-6


def test_viterbi_known_answers():
    kat = load_kat()
    for case in kat["viterbi"]:
        e = np.asarray(case["e"])
        a = None if case["a"] is None else np.asarray(case["a"])
        path, score = orc.viterbi(e, a)
        assert path.tolist() == case["path"]
        assert score == case["score"]                   # bit-exact in f64
        assert abs(score - case["enum"]) < 1e-9


def test_hand_values():
    # test_criterion.py:65-78 and SPEC.md:261
    loss, grad = orc.ctc(np.full((1, 2), math.log(0.5)), [0], 1)
    assert loss == pytest.approx(math.log(2.0), abs=1e-12)
    assert grad[0].tolist() == pytest.approx([-1.0, 0.0], abs=1e-6)
    loss, _, _ = orc.asg(np.zeros((2, 2)), [0], np.zeros((2, 2), np.float32))
    assert loss == pytest.approx(math.log(4.0), abs=1e-12)
    e = np.array([[0.3, -1.2, 2.0]])
    loss, _, _ = orc.asg(e, [1], np.zeros((3, 3), np.float32))
    assert loss == pytest.approx(orc.lse(e[0]) - e[0, 1], abs=1e-12)
    path, score = orc.viterbi(np.zeros((4, 3)))
    assert path.tolist() == [0, 0, 0, 0] and score == 0.0


def test_scale_stability_matches_reference():
    kat = load_kat()
    c = kat["asg_scale"]
    loss, ge, ga = orc.asg(np.asarray(c["e"]), c["y"], np.asarray(c["a"], np.float32))
    assert loss == pytest.approx(c["loss"], rel=1e-12)
    assert np.abs(ge - np.asarray(c["grad_e"])).max() < 1e-6
    assert np.abs(ga - np.asarray(c["grad_a"])).max() < 1e-6
    c = kat["ctc_scale"]
    loss, g = orc.ctc(np.asarray(c["e"]), c["y"], c["blank"])
    assert loss == pytest.approx(c["loss"], rel=1e-12)
    assert np.abs(g - np.asarray(c["grad"])).max() < 1e-6


@pytest.mark.parametrize("name", ["asg_c1", "asg_ragged", "asg_c3_one"])
def test_asg_batches_match_reference(name):
    g = load_npz(name)
    loss, ge, ga = orc.asg_batch(g["em"], g["em_len"], g["targets"], g["tgt_len"], g["trans"])
    np.testing.assert_allclose(loss, g["loss"], rtol=1e-12, atol=1e-9)
    assert np.abs(ge - g["grad_e"]).max() < 1e-6
    want = g["grad_a_per_utt"].astype(np.float64).sum(axis=0)
    assert orc.rel_err(ga, want) < 1e-6


@pytest.mark.parametrize("name", ["ctc_c2_one", "ctc_ragged"])
def test_ctc_batches_match_reference(name):
    g = load_npz(name)
    loss, ge = orc.ctc_batch(g["em"], g["em_len"], g["targets"], g["tgt_len"], int(g["blank"]))
    np.testing.assert_allclose(loss, g["loss"], rtol=1e-12, atol=1e-9)
    assert np.abs(ge - g["grad_e"]).max() < 1e-6


def test_viterbi_c4_matches_reference_bit_exact():
    g = load_npz("viterbi_c4")
    for b in range(g["em"].shape[0]):
        p, s = orc.viterbi(g["em"][b], g["trans"])
        assert np.array_equal(p, g["paths"][b].astype(np.int64))
        assert s == g["scores"][b]
        p, s = orc.viterbi(g["em"][b], None)
        assert np.array_equal(p, g["paths_noa"][b].astype(np.int64))
        assert s == g["scores_noa"][b]


def test_validation_order():
    assert orc.asg_validate(np.zeros((2, 2)), [], np.zeros((2, 2)))[0] == "TargetError"
    assert orc.asg_validate(np.zeros((3, 3)), [1, 1], np.zeros((3, 3)))[0] == "ContractError"
    assert orc.asg_validate(np.zeros((1, 3)), [0, 1], np.zeros((3, 3)))[0] == "InfeasibleTargetError"
    assert orc.ctc_validate(np.zeros((3, 4)), [0], 3)[0] == "ContractError"
    e = orc.log_softmax_rows(np.zeros((2, 3)))
    assert orc.ctc_validate(e, [0, 0], 2)[0] == "InfeasibleTargetError"
    assert orc.ctc_validate(e, [2], 2)[0] == "TargetError"


def test_greedy_evaluation_restatement_matches_reference_goldens():
    # tests/golden/eval_golden.json: collapse_path, edit_distance and
    # split_on_silence run by the reference itself (make_eval_golden.py)
    import json
    import os
    cases = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "eval_golden.json")))
    assert len(cases) == 120
    for c in cases:
        sil = None if c["silence"] < 0 else c["silence"]
        hyp, td, wd, rw = orc.greedy_metrics(c["path"], c["ref"], c["kind"], blank_id=c["blank"],
                                             rep_id=c["rep"], silence=sil)
        assert hyp == c["hyp"]
        assert (td, wd, rw) == (c["tok_dist"], c["word_dist"], c["ref_words"])
