"""batched greedy evaluation on the device against the reference's
evaluate loop (trainer.py:465-514), restated in the oracle: Viterbi paths ->
collapse_path (criterion.py:287-310) -> token and word edit distances over
silence-delimited groups (lexicon.py:182-195).  Integer results: exact."""

import numpy as np
import pytest
import torch

from oracle import criterion_oracle as orc

pytestmark = pytest.mark.gpu

C = pytest.importorskip("paper_1812_07625_b200.criterion")
from paper_1812_07625_b200.errors import ContractError  # noqa: E402


@pytest.fixture(autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _check(g, paths, plen, tg, tl, kind, blank=None, rep=None, sil=None):
    hyp, hl = g.hyp.cpu().numpy(), g.hyp_len.cpu().numpy()
    td, wd, rw = g.tok_dist.cpu().numpy(), g.word_dist.cpu().numpy(), g.ref_words.cpu().numpy()
    for b in range(paths.shape[0]):
        want_h, want_td, want_wd, want_rw = orc.greedy_metrics(
            paths[b, :plen[b]], tg[b, :tl[b]], kind, blank, rep, sil)
        assert list(hyp[b, :hl[b]]) == want_h, b
        assert (hyp[b, hl[b]:] == -1).all()
        assert (td[b], wd[b], rw[b]) == (want_td, want_wd, want_rw), b


@pytest.mark.parametrize("sil", [None, 0])
def test_ctc_viterbi_paths_vs_reference_loop(sil):
    em, el, tg, tl, blank = orc.synth_ctc(71, 16, 400, 12, 60, ragged=True)
    x = torch.from_numpy(em * 3.0).cuda()        # peakier: short non-trivial hypotheses
    paths, _ = C.viterbi_batched(x, el)
    g = C.greedy_eval_batched(paths, el, tg, tl, "ctc", blank_id=blank, silence_id=sil)
    assert (g.status.cpu().numpy() == 0).all()
    _check(g, paths.cpu().numpy(), el, tg, tl, "ctc", blank=blank, sil=sil)


@pytest.mark.parametrize("sil", [None, 3])
def test_asg_viterbi_paths_with_repetition_token(sil):
    em, el, tg, tl, a = orc.synth_asg(72, 16, 500, 10, 80, ragged=True)
    rep = 9
    x = torch.from_numpy(em).cuda()
    paths, _ = C.viterbi_batched(x, el, a)
    p = paths.cpu().numpy()
    for b in range(len(p)):   # no path may start with the repetition token
        if p[b, 0] == rep:
            p[b, 0] = 0
    g = C.greedy_eval_batched(torch.from_numpy(p).cuda(), el, tg, tl, "asg", rep_id=rep,
                              silence_id=sil)
    assert (g.status.cpu().numpy() == 0).all()
    _check(g, p, el, tg, tl, "asg", rep=rep, sil=sil)


def test_hand_made_edge_cases():
    blank = 0
    paths = np.array([
        [0, 0, 0, 0, 0, 0],          # all blank: empty hypothesis
        [1, 1, 0, 2, 2, 3],          # repeats and a blank
        [4, 4, 4, 4, 4, 4],          # one token
        [1, 0, 1, 0, 1, 5],          # the blank separates equal tokens
        [2, 3, 2, 3, 2, 3],
        [1, 2, 3, 0, 0, 0],          # path shorter than Tmax (length 4)
    ], np.int64)
    plen = np.array([6, 6, 6, 6, 6, 4], np.int32)
    tg = np.array([[1, 2, -1, -1], [1, 2, 3, -1], [4, -1, -1, -1], [1, 1, 1, 5],
                   [3, 2, 3, 2], [-1, -1, -1, -1]], np.int64)
    tl = np.array([2, 3, 1, 4, 4, 0], np.int32)   # the last reference is empty
    for sil in (None, 5, 2):
        g = C.greedy_eval_batched(paths, plen, tg, tl, "ctc", blank_id=blank, silence_id=sil)
        _check(g, paths, plen, tg, tl, "ctc", blank=blank, sil=sil)


def test_asg_repetition_token_first_is_a_contract_error():
    paths = np.array([[7, 7, 1, 2], [1, 7, 2, 2]], np.int64)   # rep_id 7
    plen = np.array([4, 4], np.int32)
    tg = np.array([[1, 1, 2], [1, 1, 2]], np.int64)
    tl = np.array([3, 3], np.int32)
    g = C.greedy_eval_batched(paths, plen, tg, tl, "asg", rep_id=7, check=False)
    st = g.status.cpu().numpy()
    assert st[0] == C.nat.ERR_CONTRACT and st[1] == 0
    assert list(g.hyp.cpu().numpy()[1, :3]) == [1, 1, 2] and g.tok_dist.cpu().numpy()[1] == 0
    with pytest.raises(ContractError):
        C.greedy_eval_batched(paths, plen, tg, tl, "asg", rep_id=7)


def test_evaluate_batch_matches_reference_loop():
    em, el, tg, tl, blank = orc.synth_ctc(73, 8, 300, 10, 40, ragged=True)
    em = orc.log_softmax_rows(3.0 * em.astype(np.float64)).astype(np.float32)   # peakier
    tl[2] = 0                                      # skipped, as the reference does
    tg[2, :] = -1
    r = C.evaluate_batch(em, el, tg, tl, "ctc", blank_id=blank, silence_id=1)
    loss_sum = tok = tok_len = word = word_len = n = 0
    for b in range(len(em)):
        if tl[b] == 0:
            continue
        path, _ = orc.viterbi(em[b, :el[b]])
        _, td, wd, rw = orc.greedy_metrics(path, tg[b, :tl[b]], "ctc", blank, None, 1)
        tok += td
        tok_len += int(tl[b])
        word += wd
        word_len += rw
        n += 1
        loss_sum += orc.ctc(em[b, :el[b]], tg[b, :tl[b]], blank)[0]
    assert r["utterances"] == n
    assert (r["tok_dist"], r["tok_len"], r["word_dist"], r["word_len"]) == (tok, tok_len, word,
                                                                            word_len)
    assert abs(r["loss_sum"] - loss_sum) <= 1e-4 * abs(loss_sum)


def test_reference_golden_cases():
    # the reference's own collapse_path / edit_distance / split_on_silence
    # outputs (tests/golden/make_eval_golden.py), batched through the kernel
    import json
    import os
    cases = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "eval_golden.json")))
    for kind in ("ctc", "asg"):
        for sil in sorted({c["silence"] for c in cases if c["kind"] == kind}):
            cs = [c for c in cases if c["kind"] == kind and c["silence"] == sil]
            t_max = max(len(c["path"]) for c in cs)
            l_max = max(1, max(len(c["ref"]) for c in cs))
            paths = np.zeros((len(cs), t_max), np.int64)
            tg = np.full((len(cs), l_max), -1, np.int64)
            for i, c in enumerate(cs):
                paths[i, :len(c["path"])] = c["path"]
                tg[i, :len(c["ref"])] = c["ref"]
            plen = np.array([len(c["path"]) for c in cs], np.int32)
            tl = np.array([len(c["ref"]) for c in cs], np.int32)
            g = C.greedy_eval_batched(paths, plen, tg, tl, kind, blank_id=cs[0]["blank"],
                                      rep_id=cs[0]["rep"], silence_id=None if sil < 0 else sil)
            hyp, hl = g.hyp.cpu().numpy(), g.hyp_len.cpu().numpy()
            for i, c in enumerate(cs):
                assert list(hyp[i, :hl[i]]) == c["hyp"]
                assert (int(g.tok_dist[i]), int(g.word_dist[i]), int(g.ref_words[i])) == \
                    (c["tok_dist"], c["word_dist"], c["ref_words"])
