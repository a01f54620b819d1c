"""Generate the golden fixtures by running the REFERENCE itself.

Run in the build container, where the reference package is importable:

    python tests/golden/make_golden.py

It imports ``asrkit.criterion`` and the brute-force ``oracles`` from
/root/reference/pkg (read-only; bytecode writing disabled), draws seeded
inputs with the same generators the reference tests use
(test_criterion.py:35-60, test_acceptance.py:85-106) and the SURVEY §8(d)
synthetic generators, and stores inputs + reference outputs under
tests/golden/.  The GPU box never sees /root/reference: tests read only the
committed fixtures.
"""

from __future__ import annotations

import json
import os
import sys

sys.dont_write_bytecode = True
REF = "/root/reference/pkg"
sys.path.insert(0, os.path.join(REF, "src"))
sys.path.insert(0, os.path.join(REF, "tests"))
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402

from asrkit import criterion as ref  # noqa: E402
import oracles as ref_oracles  # noqa: E402

from oracle import criterion_oracle as port  # noqa: E402  (only for the synthetic generators)


def _norm_rows(scores):
    scores = np.asarray(scores, dtype=np.float64)
    m = scores.max(axis=1, keepdims=True)
    return scores - (np.log(np.exp(scores - m).sum(axis=1, keepdims=True)) + m)


# generators restated from test_criterion.py:35-60 (same rng call sequence)
def _ctc_instance(rng, t_max=5, n_max=4, l_max=3):
    n = int(rng.integers(2, n_max + 1))
    length = int(rng.integers(1, min(l_max, n - 1) + 1))
    target = [int(rng.integers(0, n - 1))]
    while len(target) < length:
        target.append(int(rng.integers(0, n - 1)))
    reps = sum(1 for i in range(1, len(target)) if target[i] == target[i - 1])
    if len(target) + reps > t_max:
        return None
    t = int(rng.integers(len(target) + reps, t_max + 1))
    e = _norm_rows(rng.normal(size=(t, n)) * 2.0)
    return e, target, n - 1


def _asg_instance(rng, t_max=5, n_max=4, l_max=3):
    n = int(rng.integers(2, n_max + 1))
    length = int(rng.integers(1, l_max + 1))
    target = [int(rng.integers(0, n))]
    while len(target) < length:
        nxt = int(rng.integers(0, n))
        if nxt != target[-1]:
            target.append(nxt)
    t = int(rng.integers(length, t_max + 1))
    e = rng.normal(size=(t, n)) * 2.0
    a = rng.normal(size=(n, n)).astype(np.float32)
    return e, target, a


def kat_small():
    """Enumeration-size known answers: reference loss/grads + brute force."""
    out = {"ctc": [], "asg": [], "viterbi": []}
    rng = np.random.default_rng(100)
    while len(out["ctc"]) < 50:
        inst = _ctc_instance(rng)
        if inst is None:
            continue
        e, y, blank = inst
        r = ref.ctc_loss_grad(e, np.asarray(y), blank)
        out["ctc"].append({
            "e": e.tolist(), "y": y, "blank": blank, "loss": r.loss,
            "grad": r.grad_emissions.astype(np.float64).tolist(),
            "enum": float(ref_oracles.ctc_enum_loss(e, y, blank)),
        })
    rng = np.random.default_rng(200)
    for _ in range(50):
        e, y, a = _asg_instance(rng)
        r = ref.asg_loss_grad(e, np.asarray(y), a)
        out["asg"].append({
            "e": e.tolist(), "y": y, "a": a.astype(np.float64).tolist(), "loss": r.loss,
            "grad_e": r.grad_emissions.astype(np.float64).tolist(),
            "grad_a": r.grad_transitions.astype(np.float64).tolist(),
            "enum": float(ref_oracles.asg_enum_loss(e, y, a)),
        })
    rng = np.random.default_rng(1000)
    for _ in range(20):
        t = int(rng.integers(1, 5))
        n = int(rng.integers(2, 4))
        e = rng.normal(size=(t, n))
        a = rng.normal(size=(n, n)) if rng.random() < 0.5 else None
        path, score = ref.viterbi(e, a)
        best, _ = ref_oracles.viterbi_enum(e, a)
        out["viterbi"].append({
            "e": e.tolist(), "a": None if a is None else a.tolist(),
            "path": [int(v) for v in path], "score": score, "enum": float(best),
        })
    # stability cases (test_criterion.py:179-195)
    rng = np.random.default_rng(800)
    e = rng.normal(size=(5, 3)) * 1e3
    a = (rng.normal(size=(3, 3)) * 1e3).astype(np.float32)
    r = ref.asg_loss_grad(e, np.array([0, 1]), a)
    out["asg_scale"] = {"e": e.tolist(), "y": [0, 1], "a": a.astype(np.float64).tolist(),
                        "loss": r.loss, "grad_e": r.grad_emissions.astype(np.float64).tolist(),
                        "grad_a": r.grad_transitions.astype(np.float64).tolist()}
    rng = np.random.default_rng(900)
    e = _norm_rows(rng.normal(size=(6, 4)) * 1e3)
    r = ref.ctc_loss_grad(e, np.array([0, 1]), blank_id=3)
    out["ctc_scale"] = {"e": e.tolist(), "y": [0, 1], "blank": 3, "loss": r.loss,
                        "grad": r.grad_emissions.astype(np.float64).tolist()}
    with open(os.path.join(HERE, "kat_small.json"), "w") as f:
        json.dump(out, f)


def _ref_asg_batch(em, em_len, tg, tl, a):
    loss, ge, ga = [], np.zeros(em.shape, np.float32), []
    for b in range(em.shape[0]):
        t, l = int(em_len[b]), int(tl[b])
        r = ref.asg_loss_grad(em[b, :t], tg[b, :l], a)
        loss.append(r.loss)
        ge[b, :t] = r.grad_emissions
        ga.append(r.grad_transitions)
    return np.asarray(loss), ge, np.asarray(ga)


def _ref_ctc_batch(em, em_len, tg, tl, blank):
    loss, ge = [], np.zeros(em.shape, np.float32)
    for b in range(em.shape[0]):
        t, l = int(em_len[b]), int(tl[b])
        r = ref.ctc_loss_grad(em[b, :t], tg[b, :l], blank)
        loss.append(r.loss)
        ge[b, :t] = r.grad_emissions
    return np.asarray(loss), ge


def batches():
    # C1: ASG B=4 T=100 N=30 L=20 (BASELINE.json configs[0]), seed 20260000
    em, el, tg, tl, a = port.synth_asg(20260000, 4, 100, 30, 20)
    loss, ge, ga = _ref_asg_batch(em, el, tg, tl, a)
    np.savez_compressed(os.path.join(HERE, "asg_c1.npz"), em=em, em_len=el, targets=tg,
                        tgt_len=tl, trans=a, loss=loss, grad_e=ge, grad_a_per_utt=ga)
    # ragged ASG batch
    em, el, tg, tl, a = port.synth_asg(20260010, 6, 120, 12, 30, ragged=True)
    loss, ge, ga = _ref_asg_batch(em, el, tg, tl, a)
    np.savez_compressed(os.path.join(HERE, "asg_ragged.npz"), em=em, em_len=el, targets=tg,
                        tgt_len=tl, trans=a, loss=loss, grad_e=ge, grad_a_per_utt=ga)
    # one C3-shaped ASG utterance: T=1600 N=30 L=300
    em, el, tg, tl, a = port.synth_asg(20260002, 1, 1600, 30, 300)
    loss, ge, ga = _ref_asg_batch(em, el, tg, tl, a)
    np.savez_compressed(os.path.join(HERE, "asg_c3_one.npz"), em=em, em_len=el, targets=tg,
                        tgt_len=tl, trans=a, loss=loss, grad_e=ge, grad_a_per_utt=ga)
    # CTC: one C2-shaped utterance (T=800 N=29 L=150) + a small ragged batch
    em, el, tg, tl, blank = port.synth_ctc(20260001, 1, 800, 29, 150)
    loss, ge = _ref_ctc_batch(em, el, tg, tl, blank)
    np.savez_compressed(os.path.join(HERE, "ctc_c2_one.npz"), em=em, em_len=el, targets=tg,
                        tgt_len=tl, blank=blank, loss=loss, grad_e=ge)
    em, el, tg, tl, blank = port.synth_ctc(20260011, 6, 150, 10, 40, ragged=True)
    loss, ge = _ref_ctc_batch(em, el, tg, tl, blank)
    np.savez_compressed(os.path.join(HERE, "ctc_ragged.npz"), em=em, em_len=el, targets=tg,
                        tgt_len=tl, blank=blank, loss=loss, grad_e=ge)
    # Viterbi: C4-shaped (T=1600 N=30), 4 utterances, with and without A
    em, el, _, _, a = port.synth_asg(20260003, 4, 1600, 30, 1)
    paths, scores, paths0, scores0 = [], [], [], []
    for b in range(4):
        p, s = ref.viterbi(em[b], a)
        paths.append(p)
        scores.append(s)
        p, s = ref.viterbi(em[b], None)
        paths0.append(p)
        scores0.append(s)
    np.savez_compressed(os.path.join(HERE, "viterbi_c4.npz"), em=em, trans=a,
                        paths=np.asarray(paths, np.int8), scores=np.asarray(scores),
                        paths_noa=np.asarray(paths0, np.int8), scores_noa=np.asarray(scores0))


if __name__ == "__main__":
    kat_small()
    batches()
    for name in sorted(os.listdir(HERE)):
        print(name, os.path.getsize(os.path.join(HERE, name)))
