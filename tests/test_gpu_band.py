"""The band-limited gradient kernels (csrc/band.cuh) against the oracle.

The gradient warps read, after their first frame, only the lattice states
within [lo_t, hi_t + step] of the previous frame's posterior band.  These
tests drive the band where it is most stressed:

* flat emissions: the widest posteriors the lattice admits (~110-160 states);
* a forced alignment (T = L + repeats): a one-path band that must move at the
  lattice's full speed, 2 states per frame (CTC) / 1 (ASG fac);
* an utterance that is blank-dominated for 60% of its frames and must then
  emit every label: the band first idles, then sweeps at full speed;
* emissions that switch between flat and peaky: the window widens and
  narrows mid-utterance;
* determinism: the token sums are fixed-point integer atomics, so repeated
  calls return bitwise identical gradients.

Tolerance: the fp32 contract of the batched path, 1e-4 (loss relative,
gradients norm-relative, oracles.rel_err).
"""

import numpy as np
import pytest
import torch

from oracle import criterion_oracle as orc
from oracle import pool

pytestmark = pytest.mark.gpu

C = pytest.importorskip("paper_1812_07625_b200.criterion")

REL = 1e-4


@pytest.fixture(autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _ctc_check(em, el, tg, tl, blank, rel=REL):
    out = C.ctc_loss_grad_batched(torch.from_numpy(em).cuda(), el, tg, tl, blank,
                                  fallback=False, check=False)
    st = out.status.cpu().numpy()
    assert (st == 0).all(), st   # the fp32 band path itself, no fallback
    loss, ge = pool.ctc_batch(em, el, tg, tl, blank)
    np.testing.assert_allclose(out.loss.cpu().numpy(), loss, rtol=rel, atol=rel)
    g = out.grad_emissions.cpu().numpy()
    for b in range(em.shape[0]):
        assert orc.rel_err(g[b], ge[b]) < rel, b


def _asg_check(em, el, tg, tl, a, rel=REL):
    out = C.asg_loss_grad_batched(torch.from_numpy(em).cuda(), el, tg, tl, a, fallback=False,
                                  check=False, per_utterance_grad_transitions=True)
    st = out.status.cpu().numpy()
    assert (st == 0).all(), st
    loss, ge, ga = pool.asg_batch(em, el, tg, tl, a)
    np.testing.assert_allclose(out.loss.cpu().numpy(), loss, rtol=rel, atol=rel)
    g = out.grad_emissions.cpu().numpy()
    for b in range(em.shape[0]):
        assert orc.rel_err(g[b], ge[b]) < rel, b
    assert orc.rel_err(out.grad_transitions.cpu().numpy(), ga.astype(np.float64).sum(0)) < rel


def test_flat_emissions_widest_band():
    rng = np.random.default_rng(7)
    b_sz, t, n, l = 3, 600, 30, 250
    em = orc.log_softmax_rows(np.zeros((b_sz, t, n))).astype(np.float32)
    _, el, tg, tl, blank = orc.synth_ctc(11, b_sz, t, n, l)
    _ctc_check(em, el, tg, tl, blank)
    ema = np.zeros((b_sz, t, n), dtype=np.float32)
    _, ela, tga, tla, a = orc.synth_asg(12, b_sz, t, n, l)
    _asg_check(ema, ela, tga, tla, (0.1 * rng.standard_normal((n, n))).astype(np.float32))


def test_forced_alignment_band_at_full_speed():
    # CTC: T = L + repeats leaves exactly one path (every label once, a blank
    # only between repeats): the band is a single state moving ~2 per frame
    n, blank = 12, 11
    rng = np.random.default_rng(3)
    y = rng.integers(0, n - 1, size=300)
    reps = int(np.sum(y[1:] == y[:-1]))
    t = 300 + reps
    em = orc.log_softmax_rows(rng.standard_normal((2, t, n))).astype(np.float32)
    tg = np.stack([y, y]).astype(np.int64)
    _ctc_check(em, np.array([t, t], np.int32), tg, np.array([300, 300], np.int32), blank)
    # ASG: T = L, one state per frame
    ya = [int(rng.integers(0, n))]
    while len(ya) < 200:
        v = int(rng.integers(0, n))
        if v != ya[-1]:
            ya.append(v)
    ema = rng.standard_normal((1, 200, n)).astype(np.float32)
    a = rng.standard_normal((n, n)).astype(np.float32)
    _asg_check(ema, np.array([200], np.int32), np.array([ya], np.int64),
               np.array([200], np.int32), a)


def test_band_idles_then_sweeps():
    # blank-dominated for the first 60% of the frames, then every label must
    # still be emitted: the band sits at the lattice start, then sweeps
    rng = np.random.default_rng(5)
    b_sz, t, n, l = 4, 400, 20, 100
    logits = rng.standard_normal((b_sz, t, n))
    logits[:, : int(0.6 * t), n - 1] += 8.0
    em = orc.log_softmax_rows(logits).astype(np.float32)
    _, el, tg, tl, blank = orc.synth_ctc(21, b_sz, t, n, l)
    _ctc_check(em, el, tg, tl, blank)


def test_window_widens_and_narrows():
    # alternating flat and peaky stretches (scale 0 / 2) over ragged lengths
    rng = np.random.default_rng(9)
    b_sz, t, n, l = 6, 900, 30, 200
    scale = np.where((np.arange(t) // 150) % 2 == 0, 0.0, 2.0)[None, :, None]
    em = orc.log_softmax_rows(scale * rng.standard_normal((b_sz, t, n))).astype(np.float32)
    _, el, tg, tl, blank = orc.synth_ctc(31, b_sz, t, n, l, ragged=True)
    for b in range(b_sz):
        em[b, el[b]:] = 0.0
    _ctc_check(em, el, tg, tl, blank)
    ema = (scale * rng.standard_normal((b_sz, t, n))).astype(np.float32)
    _, ela, tga, tla, a = orc.synth_asg(32, b_sz, t, n, l, ragged=True)
    for b in range(b_sz):
        ema[b, ela[b]:] = 0.0
    _asg_check(ema, ela, tga, tla, a)


def test_gradients_are_deterministic():
    em, el, tg, tl, a = orc.synth_asg(41, 8, 1600, 30, 300)
    x = torch.from_numpy(em).cuda()
    g1 = C.asg_loss_grad_batched(x, el, tg, tl, a, check=False)
    g2 = C.asg_loss_grad_batched(x, el, tg, tl, a, check=False)
    assert torch.equal(g1.grad_emissions, g2.grad_emissions)
    assert torch.equal(g1.grad_transitions, g2.grad_transitions)
    assert torch.equal(g1.loss, g2.loss)
    emc, elc, tgc, tlc, blank = orc.synth_ctc(42, 8, 1600, 30, 300)
    xc = torch.from_numpy(emc).cuda()
    c1 = C.ctc_loss_grad_batched(xc, elc, tgc, tlc, blank, check=False)
    c2 = C.ctc_loss_grad_batched(xc, elc, tgc, tlc, blank, check=False)
    assert torch.equal(c1.grad_emissions, c2.grad_emissions)
    assert torch.equal(c1.loss, c2.loss)


@pytest.mark.parametrize("kind", ["asg", "ctc"])
def test_streamed_gradient_matches_plain_call(kind):
    # W2L_FLAG_STREAM_GRAD: the gradient CTAs run behind the chains, gated by
    # the chains' progress words; the same kernels, so the results must be
    # bitwise identical -- ragged lengths, a failing utterance, and a batch
    # routed to the fp64 tier (peaky emissions)
    if kind == "asg":
        em, el, tg, tl, a = orc.synth_asg(56, 12, 1600, 30, 300, ragged=True)
        em[3, 7, 2] = np.nan
        x = torch.from_numpy(em).cuda()
        run = lambda x_, **kw: C.asg_loss_grad_batched(x_, el, tg, tl, a, check=False, **kw)
    else:
        em, el, tg, tl, blank = orc.synth_ctc(57, 12, 1600, 30, 300, ragged=True)
        em[3, 7, :] = 0.5
        x = torch.from_numpy(em).cuda()
        run = lambda x_, **kw: C.ctc_loss_grad_batched(x_, el, tg, tl, blank, check=False, **kw)
    peaky = x * 10.0 if kind == "asg" else torch.log_softmax(x * 10.0, dim=-1)
    if kind == "ctc":
        peaky[3, 7, :] = 0.5   # keep utterance 3 failing
    for inp in (x, peaky):
        plain = run(inp)
        streamed = run(inp, stream_grad=True)
        assert torch.equal(plain.status, streamed.status)
        assert plain.status.cpu().numpy()[3] != 0
        assert torch.equal(plain.loss.nan_to_num(), streamed.loss.nan_to_num())
        assert torch.equal(plain.grad_emissions, streamed.grad_emissions)
        if kind == "asg":
            assert torch.equal(plain.grad_transitions, streamed.grad_transitions)
