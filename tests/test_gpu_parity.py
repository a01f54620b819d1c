"""GPU parity: the sm_100a kernels (through the C-ABI) against the CPU oracle
and the reference's golden fixtures.

Tolerances: per-utterance float64 API -- the reference's own test bounds
(|loss - enum| < 1e-5, FD rel 1e-3, Viterbi score abs 1e-9) and <= 1e-6
against the reference outputs; batched fp32 API -- loss and gradients within
1e-4 relative (norm-relative for gradients, oracles.rel_err), Viterbi paths
and scores bit-exact.
"""

import math

import numpy as np
import pytest
import torch

from conftest import load_kat, load_npz
from oracle import criterion_oracle as orc

pytestmark = pytest.mark.gpu

C = pytest.importorskip("paper_1812_07625_b200.criterion")
from paper_1812_07625_b200.errors import (ContractError, InfeasibleTargetError,  # noqa: E402
                                          NumericError, TargetError)
from conftest import TokenTable  # noqa: E402

REL = 1e-4


@pytest.fixture(autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _norm_rows(x):
    return orc.log_softmax_rows(x)


# ------------------------------------------- per-utterance (float64) API --

def test_hand_values():
    out = C.ctc_loss_grad(np.full((1, 2), math.log(0.5)), np.array([0]), blank_id=1)
    assert out.loss == pytest.approx(math.log(2.0), abs=1e-12)
    assert out.grad_emissions[0].tolist() == pytest.approx([-1.0, 0.0], abs=1e-6)
    out = C.asg_loss_grad(np.zeros((2, 2)), np.array([0]), np.zeros((2, 2), np.float32))
    assert out.loss == pytest.approx(math.log(4.0), abs=1e-12)
    e = np.array([[0.3, -1.2, 2.0]])
    out = C.asg_loss_grad(e, [1], np.zeros((3, 3), np.float32))
    assert out.loss == pytest.approx(orc.lse(e[0]) - e[0, 1], abs=1e-12)
    path, score = C.viterbi(np.zeros((4, 3)))
    assert path.tolist() == [0, 0, 0, 0] and score == pytest.approx(0.0)


def test_ctc_kat_and_enumeration():
    for c in load_kat()["ctc"]:
        out = C.ctc_loss_grad(np.asarray(c["e"]), np.asarray(c["y"]), c["blank"])
        assert abs(out.loss - c["enum"]) < 1e-5
        assert abs(out.loss - c["loss"]) < 1e-9
        assert np.abs(out.grad_emissions - np.asarray(c["grad"])).max() < 1e-6
        assert out.grad_emissions.dtype == np.float32 and isinstance(out.loss, float)


def test_asg_kat_and_enumeration():
    for c in load_kat()["asg"]:
        out = C.asg_loss_grad(np.asarray(c["e"]), np.asarray(c["y"]),
                              np.asarray(c["a"], np.float32))
        assert abs(out.loss - c["enum"]) < 1e-5
        assert abs(out.loss - c["loss"]) < 1e-9
        assert np.abs(out.grad_emissions - np.asarray(c["grad_e"])).max() < 1e-6
        assert np.abs(out.grad_transitions - np.asarray(c["grad_a"])).max() < 1e-6


def test_viterbi_kat_bit_exact():
    for c in load_kat()["viterbi"]:
        a = None if c["a"] is None else np.asarray(c["a"])
        path, score = C.viterbi(np.asarray(c["e"]), a)
        assert path.tolist() == c["path"]
        assert score == c["score"]
        assert abs(score - c["enum"]) < 1e-9


def test_gradients_match_finite_differences():
    # test_criterion.py:121-147 with the shim inside the finite differences
    rng = np.random.default_rng(500)
    for _ in range(6):
        n = int(rng.integers(2, 5))
        t = int(rng.integers(1, 6))
        length = int(rng.integers(1, 4))
        y = [int(rng.integers(0, n))]
        while len(y) < length:
            v = int(rng.integers(0, n))
            if v != y[-1]:
                y.append(v)
        t = max(t, len(y))
        e = rng.normal(size=(t, n)) * 2.0
        a = rng.normal(size=(n, n)).astype(np.float32)
        out = C.asg_loss_grad(e, y, a)
        fd_e = orc.finite_difference(lambda z: C.asg_loss_grad(z, y, a).loss, e, 1e-3)
        fd_a = orc.finite_difference(lambda z: C.asg_loss_grad(e, y, z.astype(np.float32)).loss,
                                     a.astype(np.float64), 1e-3)
        assert orc.rel_err(out.grad_emissions, fd_e) < 1e-3
        assert orc.rel_err(out.grad_transitions, fd_a) < 1e-3
    rng = np.random.default_rng(400)
    for _ in range(6):
        n = int(rng.integers(3, 5))
        e = _norm_rows(rng.normal(size=(5, n)) * 2.0)
        y = [int(rng.integers(0, n - 1)), int(rng.integers(0, n - 1))]
        out = C.ctc_loss_grad(e, y, n - 1)
        fd = orc.finite_difference(lambda z: C.ctc_loss_grad(z, y, n - 1).loss, e, 1e-3)
        assert orc.rel_err(out.grad_emissions, fd) < 1e-3


def test_row_sums_and_invariances():
    rng = np.random.default_rng(600)
    e = _norm_rows(rng.normal(size=(6, 4)) * 2)
    g = C.ctc_loss_grad(e, [0, 2, 1], 3).grad_emissions
    assert np.allclose(g.sum(axis=1), -1.0, atol=1e-5)
    e2 = rng.normal(size=(7, 3)) * 2
    g = C.asg_loss_grad(e2, [0, 1], rng.normal(size=(3, 3)).astype(np.float32)).grad_emissions
    assert np.allclose(g.sum(axis=1), 0.0, atol=1e-5)
    # CTC label-permutation invariance (test_criterion.py:167-176)
    e = _norm_rows(np.random.default_rng(700).normal(size=(5, 4)) * 2)
    base = C.ctc_loss_grad(e, np.array([0, 2, 1]), blank_id=3).loss
    perm = np.array([2, 0, 1, 3])
    e_p = np.empty_like(e)
    e_p[:, perm] = e
    assert C.ctc_loss_grad(e_p, perm[[0, 2, 1]], blank_id=3).loss == pytest.approx(base, abs=1e-10)


def test_scale_stability_matches_reference():
    kat = load_kat()
    c = kat["asg_scale"]
    out = C.asg_loss_grad(np.asarray(c["e"]), c["y"], np.asarray(c["a"], np.float32))
    assert out.loss == pytest.approx(c["loss"], rel=1e-12)
    assert np.abs(out.grad_emissions - np.asarray(c["grad_e"])).max() < 1e-6
    assert np.abs(out.grad_transitions - np.asarray(c["grad_a"])).max() < 1e-6
    c = kat["ctc_scale"]
    out = C.ctc_loss_grad(np.asarray(c["e"]), c["y"], c["blank"])
    assert out.loss == pytest.approx(c["loss"], rel=1e-12)
    assert np.isfinite(out.grad_emissions).all()


def test_error_contracts():
    with pytest.raises(ContractError):
        C.ctc_loss_grad(np.zeros((3, 4)), np.array([0]), blank_id=3)      # unnormalised
    e = _norm_rows(np.zeros((3, 3)))
    with pytest.raises(TargetError):
        C.ctc_loss_grad(e, np.array([2]), blank_id=2)                     # blank in target
    with pytest.raises(TargetError):
        C.ctc_loss_grad(e, np.array([7]), blank_id=2)                     # id out of range
    e = _norm_rows(np.random.default_rng(0).normal(size=(2, 3)))
    with pytest.raises(InfeasibleTargetError):
        C.ctc_loss_grad(e, np.array([0, 0]), blank_id=2)
    with pytest.raises(InfeasibleTargetError):
        C.asg_loss_grad(np.zeros((1, 3)), np.array([0, 1]), np.zeros((3, 3), np.float32))
    with pytest.raises(ContractError):
        C.asg_loss_grad(np.zeros((3, 3)), np.array([1, 1]), np.zeros((3, 3), np.float32))
    with pytest.raises(TargetError):
        C.asg_loss_grad(np.zeros((2, 2)), np.array([], dtype=np.int64), np.zeros((2, 2)))
    with pytest.raises(NumericError):
        C.asg_loss_grad(np.array([[0.0, np.nan]]), [0], np.zeros((2, 2)))
    with pytest.raises(NumericError):
        C.asg_loss_grad(np.zeros((2, 2)), [0], np.array([[0.0, np.inf], [0, 0]]))
    with pytest.raises(ContractError):
        C.asg_loss_grad(np.zeros((2, 2)), [0], np.zeros((3, 3)))
    with pytest.raises(ContractError):
        C.asg_loss_grad(np.zeros((0, 2)), [0], np.zeros((2, 2)))
    with pytest.raises(NumericError):
        C.viterbi(np.array([[np.inf, 0.0]]))


def test_criterion_adapters():
    table = TokenTable(["a", "b", "<2>"])
    crit = C.make_criterion("asg", table)
    assert crit.n_outputs == 3 and set(crit.params()) == {"criterion.transitions"}
    target = crit.prepare_target([0, 0, 1])
    assert target == [0, table.rep_id, 1]
    out = crit.loss_grad(np.random.default_rng(2).normal(size=(5, 3)), np.asarray(target))
    assert out.grad_transitions is not None and out.grad_transitions.shape == (3, 3)
    ctc = C.make_criterion("ctc", TokenTable(["a", "b", "|"]))
    assert ctc.blank_id == 3 and ctc.n_outputs == 4 and ctc.params() == {}
    e = _norm_rows(np.random.default_rng(1).normal(size=(4, 4)))
    hyp = ctc.collapse(ctc.viterbi_path(e))
    assert all(0 <= t < 3 for t in hyp)
    with pytest.raises(ContractError):
        C.make_criterion("transducer", TokenTable(["a"]))


# ------------------------------------------------- batched fp32 hot path --

def _asg_batch_check(g, rel=REL):
    em = torch.from_numpy(g["em"]).cuda()
    out = C.asg_loss_grad_batched(em, g["em_len"], g["targets"], g["tgt_len"], g["trans"],
                                  per_utterance_grad_transitions=True)
    loss = out.loss.cpu().numpy()
    np.testing.assert_allclose(loss, g["loss"], rtol=rel, atol=rel)
    ge = out.grad_emissions.cpu().numpy()
    for b in range(ge.shape[0]):
        assert orc.rel_err(ge[b], g["grad_e"][b]) < rel, b
        assert orc.rel_err(out.grad_transitions_per_utt[b].cpu().numpy(),
                           g["grad_a_per_utt"][b]) < rel, b
    want = g["grad_a_per_utt"].astype(np.float64).sum(axis=0)
    assert orc.rel_err(out.grad_transitions.cpu().numpy(), want) < rel
    # padding frames are zero
    for b in range(ge.shape[0]):
        assert not ge[b, int(g["em_len"][b]):].any()
    return out


@pytest.mark.parametrize("name", ["asg_c1", "asg_ragged", "asg_c3_one"])
def test_asg_batched_matches_reference(name):
    _asg_batch_check(load_npz(name))


@pytest.mark.parametrize("name", ["ctc_c2_one", "ctc_ragged"])
def test_ctc_batched_matches_reference(name):
    g = load_npz(name)
    out = C.ctc_loss_grad_batched(torch.from_numpy(g["em"]).cuda(), g["em_len"], g["targets"],
                                  g["tgt_len"], int(g["blank"]))
    np.testing.assert_allclose(out.loss.cpu().numpy(), g["loss"], rtol=REL, atol=REL)
    ge = out.grad_emissions.cpu().numpy()
    for b in range(ge.shape[0]):
        assert orc.rel_err(ge[b], g["grad_e"][b]) < REL, b
        assert not ge[b, int(g["em_len"][b]):].any()


def test_viterbi_batched_bit_exact():
    g = load_npz("viterbi_c4")
    em = torch.from_numpy(g["em"]).cuda()
    el = np.full(em.shape[0], em.shape[1], np.int32)
    paths, scores = C.viterbi_batched(em, el, g["trans"])
    assert np.array_equal(paths.cpu().numpy(), g["paths"].astype(np.int64))
    assert np.array_equal(scores.cpu().numpy(), g["scores"])
    paths, scores = C.viterbi_batched(em, el, None)
    assert np.array_equal(paths.cpu().numpy(), g["paths_noa"].astype(np.int64))
    assert np.array_equal(scores.cpu().numpy(), g["scores_noa"])


def test_viterbi_batched_ragged_vs_oracle():
    em, el, _, _, a = orc.synth_asg(77, 5, 300, 29, 1, ragged=True)
    paths, scores = C.viterbi_batched(torch.from_numpy(em).cuda(), el, a)
    for b in range(5):
        p, s = orc.viterbi(em[b, :el[b]], a)
        assert np.array_equal(paths[b, :el[b]].cpu().numpy(), p)
        assert not paths[b, el[b]:].any()
        assert scores[b].item() == s


def test_viterbi_batched_nonfinite_transitions_vs_oracle():
    # A is not validated by the reference's viterbi (criterion.py:270-272):
    # forbidden transitions (-inf) and a NaN entry take the NaN-aware
    # tournament (np.argmax: the first NaN is the maximum)
    rng = np.random.default_rng(83)
    B, T, N = 3, 200, 12
    em = rng.standard_normal((B, T, N)).astype(np.float32)
    el = np.array([200, 150, 37], np.int32)
    for a_mod in ("neginf", "nan"):
        a = rng.standard_normal((N, N)).astype(np.float32)
        a[rng.random((N, N)) < 0.3] = -np.inf
        a[np.arange(N), np.arange(N)] = 0.0     # keep every token reachable
        if a_mod == "nan":
            a[3, 5] = np.nan
        paths, scores = C.viterbi_batched(torch.from_numpy(em).cuda(), el, a)
        for b in range(B):
            p, sc = orc.viterbi(em[b, :el[b]], a)
            assert np.array_equal(paths[b, :el[b]].cpu().numpy(), p)
            got = scores[b].item()
            assert (np.isnan(got) and np.isnan(sc)) or got == sc


@pytest.mark.parametrize("T,N", [(1, 5), (31, 7), (32, 30), (33, 32), (65, 3),
                                 (5500, 30)])   # 5500*30 > 160 KB: backpointers in HBM
def test_viterbi_batched_chunk_edges_vs_oracle(T, N):
    # emissions are staged 32 frames at a time; lengths around the chunk size
    # and a batch whose backpointers do not fit in shared memory
    rng = np.random.default_rng(T * 100 + N)
    B = 3
    em = rng.standard_normal((B, T, N)).astype(np.float32)
    el = np.array([T, max(1, T - 1), max(1, T // 2)], np.int32)
    a = rng.standard_normal((N, N)).astype(np.float32)
    paths, scores = C.viterbi_batched(torch.from_numpy(em).cuda(), el, a)
    for b in range(B):
        p, s = orc.viterbi(em[b, :el[b]], a)
        assert np.array_equal(paths[b, :el[b]].cpu().numpy(), p)
        assert scores[b].item() == s


def test_asg_batched_c3_scale_vs_oracle():
    # C3 shape (T=1600 N=30 L=300) on a subset the oracle finishes in seconds
    em, el, tg, tl, a = orc.synth_asg(20260002, 8, 1600, 30, 300)
    out = C.asg_loss_grad_batched(torch.from_numpy(em).cuda(), el, tg, tl, a)
    loss, ge, ga = orc.asg_batch(em, el, tg, tl, a)
    np.testing.assert_allclose(out.loss.cpu().numpy(), loss, rtol=REL)
    assert orc.rel_err(out.grad_emissions.cpu().numpy(), ge) < REL
    assert orc.rel_err(out.grad_transitions.cpu().numpy(), ga) < REL


def test_ctc_batched_c5_scale_vs_oracle():
    em, el, tg, tl, blank = orc.synth_ctc(20260004, 6, 1600, 30, 300)
    out = C.ctc_loss_grad_batched(torch.from_numpy(em).cuda(), el, tg, tl, blank)
    loss, ge = orc.ctc_batch(em, el, tg, tl, blank)
    np.testing.assert_allclose(out.loss.cpu().numpy(), loss, rtol=REL)
    assert orc.rel_err(out.grad_emissions.cpu().numpy(), ge) < REL


def test_full_size_properties():
    # B=64, T=1600, N=30, L=300: size-independent invariants of the gradients
    em, el, tg, tl, a = orc.synth_asg(20260005, 64, 1600, 30, 300)
    out = C.asg_loss_grad_batched(torch.from_numpy(em).cuda(), el, tg, tl, a,
                                  per_utterance_grad_transitions=True)
    ge = out.grad_emissions.double()
    assert ge.sum(dim=2).abs().max().item() < 1e-4          # ASG rows sum to 0
    assert (out.loss >= -1e-6).all()
    # both posterior sets sum to T-1 edges -> sum of dA is 0 per utterance
    assert out.grad_transitions_per_utt.double().sum(dim=(1, 2)).abs().max().item() < 1e-2
    emc, elc, tgc, tlc, blank = orc.synth_ctc(20260006, 64, 1600, 30, 300)
    outc = C.ctc_loss_grad_batched(torch.from_numpy(emc).cuda(), elc, tgc, tlc, blank)
    assert (outc.grad_emissions.double().sum(dim=2) + 1).abs().max().item() < 1e-4


def test_batched_guard_fallback_extreme_scale():
    # +-1e3 scaled inputs break the fp32 scaled domain -> float64 recompute
    rng = np.random.default_rng(800)
    em = (rng.normal(size=(3, 5, 3)) * 1e3).astype(np.float32)
    a = (rng.normal(size=(3, 3)) * 1e3).astype(np.float32)
    tg = np.array([[0, 1], [1, 2], [2, -1]], dtype=np.int64)
    tl = np.array([2, 2, 1], dtype=np.int32)
    el = np.full(3, 5, np.int32)
    out = C.asg_loss_grad_batched(torch.from_numpy(em).cuda(), el, tg, tl, a)
    loss, ge, ga = orc.asg_batch(em, el, tg, tl, a)
    np.testing.assert_allclose(out.loss.cpu().numpy(), loss, rtol=1e-6)
    assert orc.rel_err(out.grad_emissions.cpu().numpy(), ge) < 1e-5
    assert orc.rel_err(out.grad_transitions.cpu().numpy(), ga) < 1e-5


def test_batched_errors_name_the_utterance():
    em, el, tg, tl, a = orc.synth_asg(5, 3, 20, 5, 4)
    tg[1, 1] = tg[1, 0]                       # consecutive duplicate in utterance 1
    with pytest.raises(ContractError, match="utterance 1"):
        C.asg_loss_grad_batched(torch.from_numpy(em).cuda(), el, tg, tl, a)
    em, el, tg, tl, blank = orc.synth_ctc(6, 3, 20, 5, 4)
    em[2, 3, 0] = np.nan
    with pytest.raises(NumericError, match="utterance 2"):
        C.ctc_loss_grad_batched(torch.from_numpy(em).cuda(), el, tg, tl, blank)


def test_autograd_functions():
    em, el, tg, tl, a = orc.synth_asg(9, 3, 40, 6, 8)
    x = torch.from_numpy(em).cuda().requires_grad_(True)
    A = torch.from_numpy(a).cuda().requires_grad_(True)
    w = torch.tensor([0.5, 1.0, 2.0], device="cuda")
    (C.asg_loss(x, A, el, tg, tl) * w).sum().backward()
    for b in range(3):
        _, g1, g2 = orc.asg(em[b], tg[b, :tl[b]], a)
        assert orc.rel_err(x.grad[b].cpu().numpy(), w[b].item() * g1) < REL
    want = sum(w[b].item() * orc.asg(em[b], tg[b, :tl[b]], a)[2].astype(np.float64)
               for b in range(3))
    assert orc.rel_err(A.grad.cpu().numpy(), want) < REL


def test_fast_path_holds_on_peaky_emissions():
    # log_softmax(2 N(0,1)) emissions (the bench data): the fp32 path must pass
    # its own guard (no float64 fallback) and match the oracle
    import bench
    em, el, ta, tc, tl, a, blank = bench.make_inputs(0, b=6)
    out = C.asg_loss_grad_batched(torch.from_numpy(em).cuda(), el, ta, tl, a, fallback=False)
    loss, ge, ga = orc.asg_batch(em, el, ta, tl, a)
    np.testing.assert_allclose(out.loss.cpu().numpy(), loss, rtol=REL)
    assert orc.rel_err(out.grad_emissions.cpu().numpy(), ge) < REL
    assert orc.rel_err(out.grad_transitions.cpu().numpy(), ga) < REL
    outc = C.ctc_loss_grad_batched(torch.from_numpy(em).cuda(), el, tc, tl, blank, fallback=False)
    loss, ge = orc.ctc_batch(em, el, tc, tl, blank)
    np.testing.assert_allclose(outc.loss.cpu().numpy(), loss, rtol=REL)
    assert orc.rel_err(outc.grad_emissions.cpu().numpy(), ge) < REL


def test_split_phase_calls_match_whole_calls():
    # W2L_FLAG_PHASE_CHAIN then W2L_FLAG_PHASE_GRAD == one whole call
    em, el, tg, tl, a = orc.synth_asg(31, 3, 120, 7, 12)
    ws = torch.empty(C.nat.lib().w2l_asg_workspace_bytes(3, 120, 7, 12), dtype=torch.uint8,
                     device="cuda")
    x = torch.from_numpy(em).cuda()
    whole = C.asg_loss_grad_batched(x, el, tg, tl, a)
    part = C.asg_loss_grad_batched(x, el, tg, tl, a, workspace=ws, phase="chain")
    part = C.asg_loss_grad_batched(x, el, tg, tl, a, workspace=ws, out=part, phase="grad")
    assert torch.equal(whole.loss, part.loss)
    assert torch.equal(whole.grad_emissions, part.grad_emissions)
    assert torch.equal(whole.grad_transitions, part.grad_transitions)
    emc, elc, tgc, tlc, blank = orc.synth_ctc(32, 3, 90, 6, 10)
    xc = torch.from_numpy(emc).cuda()
    wsc = torch.empty(C.nat.lib().w2l_ctc_workspace_bytes(3, 90, 6, 10), dtype=torch.uint8,
                      device="cuda")
    whole = C.ctc_loss_grad_batched(xc, elc, tgc, tlc, blank)
    part = C.ctc_loss_grad_batched(xc, elc, tgc, tlc, blank, workspace=wsc, phase="chain")
    part = C.ctc_loss_grad_batched(xc, elc, tgc, tlc, blank, workspace=wsc, out=part,
                                   phase="grad")
    assert torch.equal(whole.loss, part.loss)
    assert torch.equal(whole.grad_emissions, part.grad_emissions)
    # W2L_FLAG_PHASE_VALIDATE then W2L_FLAG_VALIDATED == one whole call, also
    # with a failing utterance (its status comes from the validation call)
    emc[1, 3, :] = 0.5   # a row that is not log-normalised: ContractError for utterance 1
    xc = torch.from_numpy(emc).cuda()
    whole = C.ctc_loss_grad_batched(xc, elc, tgc, tlc, blank, check=False)
    part = C.ctc_loss_grad_batched(xc, elc, tgc, tlc, blank, workspace=wsc, check=False,
                                   phase="validate")
    part = C.ctc_loss_grad_batched(xc, elc, tgc, tlc, blank, workspace=wsc, out=part,
                                   check=False, phase="rest")
    assert whole.status.cpu().tolist()[1] != 0
    assert torch.equal(whole.status, part.status)
    assert torch.equal(whole.loss.nan_to_num(), part.loss.nan_to_num())
    assert torch.equal(whole.grad_emissions, part.grad_emissions)
    part = C.asg_loss_grad_batched(x, el, tg, tl, a, workspace=ws, phase="validate")
    part = C.asg_loss_grad_batched(x, el, tg, tl, a, workspace=ws, out=part, phase="rest")
    whole = C.asg_loss_grad_batched(x, el, tg, tl, a)
    assert torch.equal(whole.loss, part.loss)
    assert torch.equal(whole.grad_emissions, part.grad_emissions)
    assert torch.equal(whole.grad_transitions, part.grad_transitions)


def _ctc_logits_oracle(x, el, tg, tl, blank):
    # the reference composition: log_softmax (float32 out, autodiff.py:394-411),
    # CTC on it, then the log_softmax backward g - softmax * sum(g)
    logp = orc.log_softmax_rows(x).astype(np.float32)
    loss, g = orc.ctc_batch(logp, el, tg, tl, blank)
    sm = np.exp(logp.astype(np.float64))
    gx = g - sm * g.sum(axis=-1, keepdims=True)
    for b in range(x.shape[0]):
        gx[b, el[b]:] = 0.0
    return loss, gx


def test_ctc_logits_fused_log_softmax():
    # CTC on logits with log_softmax fused in, vs the reference
    # composition; ragged batch, and the bench shape on a subset
    rng = np.random.default_rng(41)
    em, el, tg, tl, blank = orc.synth_ctc(41, 4, 160, 9, 20, ragged=True)
    x = (3.0 * rng.standard_normal(em.shape)).astype(np.float32)
    out = C.ctc_loss_grad_batched(torch.from_numpy(x).cuda(), el, tg, tl, blank, logits=True,
                                  fallback=False)
    loss, gx = _ctc_logits_oracle(x, el, tg, tl, blank)
    np.testing.assert_allclose(out.loss.cpu().numpy(), loss, rtol=REL)
    assert orc.rel_err(out.grad_emissions.cpu().numpy(), gx) < REL
    em, el, tg, tl, blank = orc.synth_ctc(42, 3, 1600, 30, 300)
    x = (2.0 * rng.standard_normal(em.shape)).astype(np.float32)
    out = C.ctc_loss_grad_batched(torch.from_numpy(x).cuda(), el, tg, tl, blank, logits=True,
                                  fallback=False)
    loss, gx = _ctc_logits_oracle(x, el, tg, tl, blank)
    np.testing.assert_allclose(out.loss.cpu().numpy(), loss, rtol=REL)
    assert orc.rel_err(out.grad_emissions.cpu().numpy(), gx) < REL


def test_ctc_logits_mixed_widths():
    # f1 on a batch mixing lattice widths (S = 2L+1 over 1..5 warps), the empty
    # target and the gradient kernel's block edges, loss-only included
    rng = np.random.default_rng(46)
    lens = [(16, 0), (128, 63), (129, 64), (256, 127), (300, 191), (520, 256)]
    b_sz, t_max, n = len(lens), 540, 29
    blank = n - 1
    x = (2.0 * rng.standard_normal((b_sz, t_max, n))).astype(np.float32)
    el = np.array([t for t, _ in lens], np.int32)
    tl = np.array([l for _, l in lens], np.int32)
    tg = np.full((b_sz, int(tl.max())), -1, np.int64)
    for b in range(b_sz):
        tg[b, :tl[b]] = rng.integers(0, n - 1, size=tl[b])
        x[b, el[b]:] = 0.0
    xd = torch.from_numpy(x).cuda()
    out = C.ctc_loss_grad_batched(xd, el, tg, tl, blank, logits=True)
    loss, gx = _ctc_logits_oracle(x, el, tg, tl, blank)
    np.testing.assert_allclose(out.loss.cpu().numpy(), loss, rtol=REL)
    assert orc.rel_err(out.grad_emissions.cpu().numpy(), gx) < REL
    lo = C.ctc_loss_grad_batched(xd, el, tg, tl, blank, logits=True, loss_only=True)
    np.testing.assert_allclose(lo.loss.cpu().numpy(), loss, rtol=REL)


def test_ctc_logits_float64_fallback():
    # extreme logits break the fp32 lattice; the float64 recompute (logits mode
    # of the exact kernel) must still match the reference composition
    rng = np.random.default_rng(43)
    em, el, tg, tl, blank = orc.synth_ctc(43, 3, 12, 5, 3)
    x = (400.0 * rng.standard_normal(em.shape)).astype(np.float32)
    out = C.ctc_loss_grad_batched(torch.from_numpy(x).cuda(), el, tg, tl, blank, logits=True,
                                  check=False)
    loss, gx = _ctc_logits_oracle(x, el, tg, tl, blank)
    ok = np.isfinite(loss)
    np.testing.assert_allclose(out.loss.cpu().numpy()[ok], loss[ok], rtol=1e-5)
    assert orc.rel_err(out.grad_emissions.cpu().numpy()[ok], gx[ok]) < 1e-5


def test_loss_only_mode_matches_full_call():
    # forward recursion + loss only (evaluation)
    em, el, tg, tl, a = orc.synth_asg(44, 5, 300, 12, 40, ragged=True)
    x = torch.from_numpy(em).cuda()
    full = C.asg_loss_grad_batched(x, el, tg, tl, a)
    lo = C.asg_loss_grad_batched(x, el, tg, tl, a, loss_only=True)
    assert torch.equal(full.loss, lo.loss)
    emc, elc, tgc, tlc, blank = orc.synth_ctc(45, 5, 300, 12, 40, ragged=True)
    xc = torch.from_numpy(emc).cuda()
    full = C.ctc_loss_grad_batched(xc, elc, tgc, tlc, blank)
    lo = C.ctc_loss_grad_batched(xc, elc, tgc, tlc, blank, loss_only=True)
    assert torch.equal(full.loss, lo.loss)
    # logits + loss only
    lo = C.ctc_loss_grad_batched(xc * 3.0, elc, tgc, tlc, blank, loss_only=True, logits=True)
    loss, _ = _ctc_logits_oracle(emc * 3.0, elc, tgc, tlc, blank)
    np.testing.assert_allclose(lo.loss.cpu().numpy(), loss, rtol=REL)


@pytest.mark.parametrize("bsz", [64, 6, 17])
def test_transitions_sgd_step_matches_reference_optimizer(bsz):
    # /B + momentum + SGD (trainer.py:442-449, autodiff.py:429-433);
    # B = 6, 17: the /B is a true division (x * (1/B) differs from x / B there)
    from paper_1812_07625_b200.distributed import sgd_step_transitions
    rng = np.random.default_rng(46)
    n, lr, mom = 30, 0.05, 0.9
    a = rng.standard_normal((n, n)).astype(np.float32)
    v = rng.standard_normal((n, n)).astype(np.float32)
    gsum = (rng.standard_normal((n, n)) * 7).astype(np.float32)
    at, vt, gt = (torch.from_numpy(x.copy()).cuda() for x in (a, v, gsum))
    for _ in range(3):
        sgd_step_transitions(at, vt, gt, bsz, lr, mom)
        g = (gsum.astype(np.float64) / bsz).astype(np.float32)
        np.multiply(v, mom, out=v)
        v += g
        a = a - lr * v
    assert np.array_equal(vt.cpu().numpy(), v)
    assert np.array_equal(at.cpu().numpy(), a)


def test_w2le_batch_feeds_the_batched_criterion(tmp_path):
    # W2LE files -> one pinned padded batch -> device -> ASG
    from paper_1812_07625_b200 import emissions_io as eio
    em, el, tg, tl, a = orc.synth_asg(47, 3, 50, 8, 9, ragged=True)
    paths = []
    for b in range(3):
        paths.append(tmp_path / f"{b}.w2le")
        eio.dump_emissions(em[b, :el[b]], paths[-1])
    x, lens = eio.load_emissions_batch(paths, device=torch.device("cuda"))
    out = C.asg_loss_grad_batched(x, lens, tg, tl, a)
    loss, ge, ga = orc.asg_batch(em, el, tg, tl, a)
    np.testing.assert_allclose(out.loss.cpu().numpy(), loss, rtol=REL)
    assert orc.rel_err(out.grad_emissions.cpu().numpy()[:, :x.shape[1]], ge[:, :x.shape[1]]) < REL


@pytest.mark.parametrize("t_max,n,l_max", [(1, 2, 1), (2, 2, 1), (5, 3, 2), (7, 4, 7), (9, 2, 5),
                                           (17, 30, 8), (130, 32, 128), (260, 32, 257)])
def test_asg_batched_edge_sizes(t_max, n, l_max):
    # fp32 fast path at the edges of its schedule: T below one 8-step block,
    # T = L (no slack), N = 2 and N = 32 (no spare fcc lane), lattices that
    # end exactly on / just past a 128-state warp boundary; ragged lengths
    em, el, tg, tl, a = orc.synth_asg(50 + t_max, 3, t_max, n, l_max, ragged=True)
    out = C.asg_loss_grad_batched(torch.from_numpy(em).cuda(), el, tg, tl, a)
    loss, ge, ga = orc.asg_batch(em, el, tg, tl, a)
    np.testing.assert_allclose(out.loss.cpu().numpy(), loss, rtol=REL, atol=1e-5)
    assert orc.rel_err(out.grad_emissions.cpu().numpy(), ge) < REL
    assert orc.rel_err(out.grad_transitions.cpu().numpy(), ga) < REL


@pytest.mark.parametrize("t_max,n,l_max", [(1, 2, 1), (3, 2, 0), (6, 3, 2), (9, 5, 4),
                                           (200, 32, 63), (300, 32, 127)])
def test_ctc_batched_edge_sizes(t_max, n, l_max):
    # including the empty target (L = 0, CTC allows it) and T = 1
    em, el, tg, tl, blank = orc.synth_ctc(60 + t_max, 3, t_max, n, max(l_max, 1), ragged=True)
    if l_max == 0:
        tg[:] = -1
        tl[:] = 0
    out = C.ctc_loss_grad_batched(torch.from_numpy(em).cuda(), el, tg, tl, blank)
    loss, ge = orc.ctc_batch(em, el, tg, tl, blank)
    np.testing.assert_allclose(out.loss.cpu().numpy(), loss, rtol=REL, atol=1e-5)
    assert orc.rel_err(out.grad_emissions.cpu().numpy(), ge) < REL


def test_asg_batched_mixed_widths_and_block_edges():
    # one batch whose utterances use 1..4 lattice warps (weff below the
    # batch's W), lengths at the 16-frame warp and 128-frame block edges of
    # the gradient kernels, and one utterance that fails validation (its rows
    # must come back zero and the others must be unaffected)
    rng = np.random.default_rng(81)
    lens = [(16, 1), (140, 127), (128, 128), (129, 129), (255, 200), (256, 256), (300, 257),
            (400, 384), (450, 385), (500, 450)]
    b_sz, t_max, n = len(lens) + 1, 520, 30
    em = rng.standard_normal((b_sz, t_max, n), dtype=np.float32)
    a = rng.standard_normal((n, n)).astype(np.float32)
    el = np.array([t for t, _ in lens] + [300], np.int32)
    tl = np.array([l for _, l in lens] + [100], np.int32)
    tg = np.full((b_sz, int(tl.max())), -1, np.int64)
    for b in range(b_sz):
        seq = [int(rng.integers(0, n))]
        while len(seq) < tl[b]:
            v = int(rng.integers(0, n))
            if v != seq[-1]:
                seq.append(v)
        tg[b, :tl[b]] = seq
        em[b, el[b]:] = 0.0
    em[-1, 5, 3] = np.nan          # the failing utterance: non-finite emission
    out = C.asg_loss_grad_batched(torch.from_numpy(em).cuda(), el, tg, tl, a, check=False,
                                  per_utterance_grad_transitions=True)
    st = out.status.cpu().numpy()
    assert st[-1] != 0 and (st[:-1] == 0).all()
    ge_gpu = out.grad_emissions.cpu().numpy()
    assert not ge_gpu[-1].any()
    good = slice(0, b_sz - 1)
    loss, ge, ga = orc.asg_batch(em[good], el[good], tg[good], tl[good], a)
    np.testing.assert_allclose(out.loss.cpu().numpy()[good], loss, rtol=REL)
    assert orc.rel_err(ge_gpu[good], ge) < REL
    assert orc.rel_err(out.grad_transitions.cpu().numpy(), ga) < REL


def test_ctc_batched_mixed_widths_and_block_edges():
    # CTC counterpart: lattices of 1..5 warps (S = 2L+1) in one batch, the
    # empty target, lengths at the gradient kernel's block edges, and one
    # utterance that fails validation (a row that is not log-normalised)
    rng = np.random.default_rng(82)
    lens = [(16, 0), (16, 3), (128, 63), (129, 64), (256, 127), (300, 128), (400, 191),
            (450, 192), (500, 255), (520, 256)]
    b_sz, t_max, n = len(lens) + 1, 600, 29
    blank = n - 1
    em = orc.log_softmax_rows(2.0 * rng.standard_normal((b_sz, t_max, n))).astype(np.float32)
    el = np.array([t for t, _ in lens] + [300], np.int32)
    tl = np.array([l for _, l in lens] + [50], np.int32)
    tg = np.full((b_sz, int(tl.max())), -1, np.int64)
    for b in range(b_sz):
        tg[b, :tl[b]] = rng.integers(0, n - 1, size=tl[b])
        em[b, el[b]:] = 0.0
    em[-1, 7, :] += 1.0            # |logsumexp| = 1 > 1e-2: ContractError
    out = C.ctc_loss_grad_batched(torch.from_numpy(em).cuda(), el, tg, tl, blank, check=False)
    st = out.status.cpu().numpy()
    assert st[-1] != 0 and (st[:-1] == 0).all()
    ge_gpu = out.grad_emissions.cpu().numpy()
    assert not ge_gpu[-1].any()
    good = slice(0, b_sz - 1)
    loss, ge = orc.ctc_batch(em[good], el[good], tg[good], tl[good], blank)
    np.testing.assert_allclose(out.loss.cpu().numpy()[good], loss, rtol=REL, atol=1e-5)
    assert orc.rel_err(ge_gpu[good], ge) < REL


def test_maximum_lattices():
    # the largest supported lattices: ASG L = 1024 (8 lattice warps) and CTC
    # L = 511 (2L+1 = 1023 states, 8 warps), N = 32
    em, el, tg, tl, a = orc.synth_asg(70, 2, 1100, 32, 1024)
    out = C.asg_loss_grad_batched(torch.from_numpy(em).cuda(), el, tg, tl, a)
    loss, ge, ga = orc.asg_batch(em, el, tg, tl, a)
    np.testing.assert_allclose(out.loss.cpu().numpy(), loss, rtol=REL)
    assert orc.rel_err(out.grad_emissions.cpu().numpy(), ge) < REL
    assert orc.rel_err(out.grad_transitions.cpu().numpy(), ga) < REL
    emc, elc, tgc, tlc, blank = orc.synth_ctc(71, 2, 1100, 32, 511)
    outc = C.ctc_loss_grad_batched(torch.from_numpy(emc).cuda(), elc, tgc, tlc, blank)
    loss, ge = orc.ctc_batch(emc, elc, tgc, tlc, blank)
    np.testing.assert_allclose(outc.loss.cpu().numpy(), loss, rtol=REL)
    assert orc.rel_err(outc.grad_emissions.cpu().numpy(), ge) < REL
