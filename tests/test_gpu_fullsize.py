"""GPU parity at the BASELINE configs' FULL sizes, the float64 path at scale,
and the fp32 path's range limits.

* C4 Viterbi B=64 T=1600 N=30: paths and scores bit-exact (criterion.py:259-284);
* C3 ASG B=64 T=1600 N=30 L=300 and C2 CTC B=32 T=800 N=29 L=150, whole
  batches: loss and per-utterance gradients within 1e-4 (norm-relative,
  oracles.rel_err), grad_A summed over the batch;
* the bench's own B=64 ASG+CTC inputs, with the float64 fallback disabled;
* the per-utterance float64 API (the reference numerics) on the T=1600 /
  T=800 golden utterances produced by the reference itself, within 1e-6;
* the float64 fallback kernel forced on 16 C3 utterances (W2L_FLAG_FORCE_EXACT);
* inputs whose fp32 weights would flush to zero identically in both
  directions (emissions ~60 sigma apart, transitions ~1e3): the fast path
  must hand them to the float64 kernel, never return a silently wrong result.

The oracle runs one utterance per process (oracle/pool.py).
"""

import numpy as np
import pytest
import torch

from conftest import load_npz
from oracle import criterion_oracle as orc
from oracle import pool

pytestmark = pytest.mark.gpu

C = pytest.importorskip("paper_1812_07625_b200.criterion")
nat = C.nat

REL = 1e-4


@pytest.fixture(autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _check_asg(out, want_loss, want_ge, want_ga_utt, el, rel=REL):
    np.testing.assert_allclose(out.loss.cpu().numpy(), want_loss, rtol=rel, atol=rel)
    ge = out.grad_emissions.cpu().numpy()
    for b in range(ge.shape[0]):
        assert orc.rel_err(ge[b], want_ge[b]) < rel, b
        assert not ge[b, int(el[b]):].any()
    want = want_ga_utt.astype(np.float64).sum(axis=0)
    assert orc.rel_err(out.grad_transitions.cpu().numpy(), want) < rel


def _check_ctc(out, want_loss, want_ge, el, rel=REL):
    np.testing.assert_allclose(out.loss.cpu().numpy(), want_loss, rtol=rel, atol=rel)
    ge = out.grad_emissions.cpu().numpy()
    for b in range(ge.shape[0]):
        assert orc.rel_err(ge[b], want_ge[b]) < rel, b
        assert not ge[b, int(el[b]):].any()


def test_viterbi_c4_full_batch_bit_exact():
    em, el, _, _, a = orc.synth_asg(20260003, 64, 1600, 30, 1)
    x = torch.from_numpy(em).cuda()
    for trans in (a, None):
        paths, scores = C.viterbi_batched(x, el, trans)
        want_p, want_s = pool.viterbi_batch(em, el, trans)
        assert np.array_equal(paths.cpu().numpy(), want_p)
        assert np.array_equal(scores.cpu().numpy(), want_s)


def test_asg_c3_full_batch():
    em, el, tg, tl, a = orc.synth_asg(20260002, 64, 1600, 30, 300)
    out = C.asg_loss_grad_batched(torch.from_numpy(em).cuda(), el, tg, tl, a)
    _check_asg(out, *pool.asg_batch(em, el, tg, tl, a), el)


def test_ctc_c2_full_batch():
    em, el, tg, tl, blank = orc.synth_ctc(20260001, 32, 800, 29, 150)
    out = C.ctc_loss_grad_batched(torch.from_numpy(em).cuda(), el, tg, tl, blank)
    _check_ctc(out, *pool.ctc_batch(em, el, tg, tl, blank), el)


def test_bench_inputs_full_batch_fast_path():
    # the exact inputs bench.py times, whole batch, float64 fallback disabled:
    # the fp32 path alone must pass its guard and match the oracle
    import bench
    em, el, ta, tc, tl, a, blank = bench.make_inputs(0)
    x = torch.from_numpy(em).cuda()
    out = C.asg_loss_grad_batched(x, el, ta, tl, a, fallback=False)
    _check_asg(out, *pool.asg_batch(em, el, ta, tl, a), el)
    outc = C.ctc_loss_grad_batched(x, el, tc, tl, blank, fallback=False)
    _check_ctc(outc, *pool.ctc_batch(em, el, tc, tl, blank), el)


def test_float64_api_on_full_length_goldens():
    # the reference-compatible per-utterance API runs the float64 kernels:
    # against the reference's own outputs at T=1600/L=300 and T=800/L=150
    g = load_npz("asg_c3_one")
    t, l = int(g["em_len"][0]), int(g["tgt_len"][0])
    out = C.asg_loss_grad(g["em"][0, :t], g["targets"][0, :l], g["trans"])
    assert out.loss == pytest.approx(float(g["loss"][0]), rel=1e-9)
    assert orc.rel_err(out.grad_emissions, g["grad_e"][0, :t]) < 1e-6
    assert orc.rel_err(out.grad_transitions, g["grad_a_per_utt"][0]) < 1e-6
    g = load_npz("ctc_c2_one")
    t, l = int(g["em_len"][0]), int(g["tgt_len"][0])
    out = C.ctc_loss_grad(g["em"][0, :t], g["targets"][0, :l], int(g["blank"]))
    assert out.loss == pytest.approx(float(g["loss"][0]), rel=1e-9)
    assert orc.rel_err(out.grad_emissions, g["grad_e"][0, :t]) < 1e-6


def test_forced_float64_fallback_at_c3():
    # the guard's fallback kernel on 16 full-length utterances at once
    em, el, tg, tl, a = orc.synth_asg(20260012, 16, 1600, 30, 300)
    out = C.asg_loss_grad_batched(torch.from_numpy(em).cuda(), el, tg, tl, a, force_exact=True)
    _check_asg(out, *pool.asg_batch(em, el, tg, tl, a), el, rel=1e-6)
    emc, elc, tgc, tlc, blank = orc.synth_ctc(20260013, 16, 1600, 30, 300)
    outc = C.ctc_loss_grad_batched(torch.from_numpy(emc).cuda(), elc, tgc, tlc, blank,
                                   force_exact=True)
    _check_ctc(outc, *pool.ctc_batch(emc, elc, tgc, tlc, blank), elc, rel=1e-6)


def test_flushed_weights_go_to_float64():
    # exp(e - max e) below ~e^-87 flushes to zero in BOTH chain
    # directions, which the fwd/bwd consistency guard cannot see.  Emissions
    # 60 sigma wide and transitions 1e3 wide must take the float64 path and
    # match the oracle; with the fallback disabled they must be reported.
    rng = np.random.default_rng(2024)
    b_sz, t, n, l = 64, 12, 4, 4
    em = (rng.standard_normal((b_sz, t, n)) * 60).astype(np.float32)
    _, el, tg, tl, a = orc.synth_asg(2025, b_sz, t, n, l)
    x = torch.from_numpy(em).cuda()
    out = C.asg_loss_grad_batched(x, el, tg, tl, a, per_utterance_grad_transitions=True)
    loss, ge, ga_utt = pool.asg_batch(em, el, tg, tl, a)
    _check_asg(out, loss, ge, ga_utt, el, rel=1e-5)
    fast = C.asg_loss_grad_batched(x, el, tg, tl, a, fallback=False, check=False)
    st = fast.status.cpu().numpy()
    ok = st == 0
    assert (~ok).any()                      # the flushed utterances were caught
    np.testing.assert_allclose(fast.loss.cpu().numpy()[ok], loss[ok], rtol=REL)
    # transitions 1e3 apart: every utterance is computed in float64
    a3 = (a * 1e3).astype(np.float32)
    emx, elx, tgx, tlx, _ = orc.synth_asg(2026, 8, 6, 3, 2)
    a3 = (rng.standard_normal((3, 3)) * 1e3).astype(np.float32)
    fast = C.asg_loss_grad_batched(torch.from_numpy(emx).cuda(), elx, tgx, tlx, a3,
                                   fallback=False, check=False)
    assert (fast.status.cpu().numpy() != 0).all()
    out = C.asg_loss_grad_batched(torch.from_numpy(emx).cuda(), elx, tgx, tlx, a3)
    loss, ge, ga = orc.asg_batch(emx, elx, tgx, tlx, a3)
    np.testing.assert_allclose(out.loss.cpu().numpy(), loss, rtol=1e-6)
    assert orc.rel_err(out.grad_emissions.cpu().numpy(), ge) < 1e-5
    # CTC: log-probabilities 60 sigma wide (lattice tokens far below the frame max)
    emc = orc.log_softmax_rows(rng.standard_normal((b_sz, t, n)) * 60).astype(np.float32)
    _, elc, tgc, tlc, blank = orc.synth_ctc(2027, b_sz, t, n, 3)
    outc = C.ctc_loss_grad_batched(torch.from_numpy(emc).cuda(), elc, tgc, tlc, blank,
                                   check=False)
    loss, ge = pool.ctc_batch(emc, elc, tgc, tlc, blank)
    fin = np.isfinite(loss)
    np.testing.assert_allclose(outc.loss.cpu().numpy()[fin], loss[fin], rtol=1e-5)
    assert orc.rel_err(outc.grad_emissions.cpu().numpy()[fin], ge[fin]) < 1e-5


def test_loss_only_is_guarded():
    # loss-only mode runs both directions and compares their totals; on inputs
    # outside the fp32 range it must fall back exactly like the full call
    rng = np.random.default_rng(77)
    em = (rng.standard_normal((16, 40, 5)) * 40).astype(np.float32)
    _, el, tg, tl, a = orc.synth_asg(78, 16, 40, 5, 10)
    x = torch.from_numpy(em).cuda()
    full = C.asg_loss_grad_batched(x, el, tg, tl, a)
    lo = C.asg_loss_grad_batched(x, el, tg, tl, a, loss_only=True)
    loss, _, _ = orc.asg_batch(em, el, tg, tl, a)
    np.testing.assert_allclose(lo.loss.cpu().numpy(), loss, rtol=1e-6)
    np.testing.assert_allclose(full.loss.cpu().numpy(), loss, rtol=1e-6)


def test_empty_batch_zero_transition_gradient():
    # an empty shard must contribute zeros to the all-reduce
    n = 7
    out = C.BatchLossOutput(loss=torch.empty(0, dtype=torch.float64, device="cuda"),
                            grad_emissions=torch.empty((0, 5, n), device="cuda"),
                            grad_transitions=torch.full((n, n), float("nan"), device="cuda"),
                            status=torch.empty(0, dtype=torch.int32, device="cuda"))
    C.asg_loss_grad_batched(torch.zeros((0, 5, n), device="cuda"), np.zeros(0, np.int32),
                            np.zeros((0, 3), np.int64), np.zeros(0, np.int32),
                            np.zeros((n, n), np.float32), out=out)
    assert torch.equal(out.grad_transitions, torch.zeros((n, n), device="cuda"))


@pytest.mark.parametrize("bsz", [6, 64, 7])
def test_transitions_sgd_step_any_batch(bsz):
    # f2 with /B by division (trainer.py:447: (total / batch.size).astype(f32))
    from paper_1812_07625_b200.distributed import sgd_step_transitions
    rng = np.random.default_rng(bsz)
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


def test_autograd_no_sync_marks_failed_utterances():
    em, el, tg, tl, a = orc.synth_asg(9, 3, 40, 6, 8)
    tg[1, 1] = tg[1, 0]                         # utterance 1 is invalid
    x = torch.from_numpy(em).cuda().requires_grad_(True)
    A = torch.from_numpy(a).cuda().requires_grad_(True)
    loss = C.asg_loss(x, A, el, tg, tl)
    assert torch.isnan(loss[1]) and torch.isfinite(loss[[0, 2]]).all()
    loss.nan_to_num().sum().backward()
    assert not x.grad[1].any()
    with pytest.raises(C.ContractError, match="utterance 1"):
        C.check_status(loss)


def test_library_nccl_allreduce_single_rank():
    # the C-ABI collective (w2l_comm_* / w2l_allreduce_grad_A) on a one-rank
    # communicator: the all-reduce of one rank is the identity, on the stream
    from paper_1812_07625_b200.distributed import NcclComm
    comm = NcclComm()
    g = torch.randn(30, 30, device="cuda")
    want = g.clone()
    comm.allreduce_grad_transitions(g)
    torch.cuda.synchronize()
    assert torch.equal(g, want)
    comm.close()
    # contract violations and a missing communicator are reported, not run
    assert nat.lib().w2l_allreduce_grad_A(g.data_ptr(), 40, None, None) == nat.ERR_CONTRACT


@pytest.mark.parametrize("scale", [10.0, 20.0])
def test_peaky_emissions_resolved_by_fp64_tier(scale):
    # trained acoustic models are peaky: log_softmax(s N(0,1)) with s = 10, 20
    # leaves the fp32 range (every utterance fails its guard or its flush
    # check) and must be resolved by the fp64 scaled-linear tier alone (the
    # log-domain kernel disabled), matching the oracle at 1e-4
    import bench
    em, el, ta, tc, tl, a, blank = bench.peaky_inputs(scale, b=12)
    x = torch.from_numpy(em).cuda()
    fast = C.asg_loss_grad_batched(x, el, ta, tl, a, fallback=False, check=False)
    assert (fast.status.cpu().numpy() != 0).any()
    out = C.asg_loss_grad_batched(x, el, ta, tl, a, fallback="f64", check=False)
    assert (out.status.cpu().numpy() == 0).all()
    _check_asg(out, *pool.asg_batch(em, el, ta, tl, a), el)
    outc = C.ctc_loss_grad_batched(x, el, tc, tl, blank, fallback="f64", check=False)
    assert (outc.status.cpu().numpy() == 0).all()
    _check_ctc(outc, *pool.ctc_batch(em, el, tc, tl, blank), el)


@pytest.mark.parametrize("scale", [2.0, 5.0, 10.0, 20.0])
def test_precision_routing_keeps_results(scale):
    # W2L_FLAG_NO_ROUTE: the routing (peaky batches straight to the fp64
    # tier) changes which tier computes, never the results: routed and
    # unrouted calls both match the oracle at 1e-4 and each other
    import bench
    em, el, ta, tc, tl, a, blank = bench.peaky_inputs(scale, b=12)
    x = torch.from_numpy(em).cuda()
    want_a = pool.asg_batch(em, el, ta, tl, a)
    want_c = pool.ctc_batch(em, el, tc, tl, blank)
    for rt in (True, False):
        out = C.asg_loss_grad_batched(x, el, ta, tl, a, route=rt, per_utterance_grad_transitions=True)
        _check_asg(out, *want_a, el)
        outc = C.ctc_loss_grad_batched(x, el, tc, tl, blank, route=rt)
        _check_ctc(outc, *want_c, el)
