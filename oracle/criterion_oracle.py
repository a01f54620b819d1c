"""CPU oracle for the sequence-criterion hot path -- TEST INFRASTRUCTURE ONLY.

This module is a float64 numpy restatement of the reference algorithms in
``/root/reference/pkg/src/asrkit/criterion.py`` (asrkit, the wav2letter++
restatement this repo is a drop-in for) and of the brute-force oracles in
``/root/reference/pkg/tests/oracles.py``.  It exists so that

* ``tests/`` can check the CUDA path against it (parity),
* ``__graft_entry__.smoke()`` can check one small GPU invocation,
* ``bench.py`` can time it as the CPU baseline (``cpu_baseline`` /
  ``--impl reference``; kind "port").

Nothing in the product package (``paper_1812_07625_b200``) imports it; the
product path fails loudly when the CUDA library is missing.

Parity is pinned: ``tests/golden/make_golden.py`` ran the reference itself
(importable from /root/reference in the build container) and committed its
outputs as ``tests/golden/*.npz``; ``tests/test_oracle.py`` checks this file
against those fixtures (and the reference's own known-answer tests).

Conventions follow the reference exactly:
* transitions are indexed ``A[to][from]`` (criterion.py:170-171);
* losses are per-utterance sums (criterion.py:4-6);
* gradients are returned as float32, losses as Python floats, internals f64.
"""

from __future__ import annotations

import itertools
import math

import numpy as np

NEG_INF = -np.inf


# ---------------------------------------------------------------- numerics --

def lse(x, axis=None):
    """Max-shifted log-sum-exp; a non-finite max is replaced by 0 so an all
    -inf slice yields -inf rather than NaN (criterion.py:250-254)."""
    x = np.asarray(x, dtype=np.float64)
    top = np.max(x, axis=axis, keepdims=True)
    top = np.where(np.isfinite(top), top, 0.0)
    s = np.log(np.sum(np.exp(x - top), axis=axis)) + np.squeeze(top, axis=axis)
    return float(s) if axis is None else s


def rel_err(approx, exact):
    """Norm-relative error with a 1e-8 floor (tests/oracles.py:44-49)."""
    approx = np.asarray(approx, dtype=np.float64)
    exact = np.asarray(exact, dtype=np.float64)
    return float(np.linalg.norm(approx - exact) / max(np.linalg.norm(exact), 1e-8))


def finite_difference(f, x, eps=1e-3):
    """Central differences of scalar f, one probe per entry (oracles.py:27-41)."""
    x = np.array(x, dtype=np.float64, copy=True)
    out = np.zeros_like(x)
    xv, ov = x.reshape(-1), out.reshape(-1)
    for k in range(xv.size):
        keep = xv[k]
        xv[k] = keep + eps
        up = f(x)
        xv[k] = keep - eps
        dn = f(x)
        xv[k] = keep
        ov[k] = (up - dn) / (2.0 * eps)
    return out


# --------------------------------------------------------------------- CTC --

def ctc_lattice(target, blank):
    """Blank-interleaved labels and skip permissions (criterion.py:113-120)."""
    y = np.asarray(target, dtype=np.int64)
    n_states = 2 * y.size + 1
    labels = np.full(n_states, blank, dtype=np.int64)
    labels[1::2] = y
    can_skip = np.zeros(n_states, dtype=bool)
    if y.size > 1:
        can_skip[3::2] = y[1:] != y[:-1]
    return labels, can_skip


def ctc(emissions, target, blank):
    """CTC negative log marginal and d/d emissions (criterion.py:84-162).

    Returns (loss, grad float32[T,N]).  Assumes the inputs already passed the
    reference's validation (see ``ctc_validate``)."""
    e = np.asarray(emissions, dtype=np.float64)
    n_frames = e.shape[0]
    labels, can_skip = ctc_lattice(target, blank)
    n_states = labels.size
    em = e[:, labels]                                   # [T, S]

    fwd = np.full((n_frames, n_states), NEG_INF)
    fwd[0, 0] = em[0, 0]
    if n_states > 1:
        fwd[0, 1] = em[0, 1]
    for t in range(1, n_frames):
        p = fwd[t - 1]
        acc = p.copy()
        acc[1:] = np.logaddexp(acc[1:], p[:-1])          # from s-1
        if n_states > 2:                                 # from s-2 where allowed
            acc[2:] = np.where(can_skip[2:], np.logaddexp(acc[2:], p[:-2]), acc[2:])
        fwd[t] = em[t] + acc
    if n_states > 1:
        log_z = np.logaddexp(fwd[-1, -1], fwd[-1, -2])
    else:
        log_z = fwd[-1, -1]

    bwd = np.full((n_frames, n_states), NEG_INF)
    bwd[-1, -1] = em[-1, -1]
    if n_states > 1:
        bwd[-1, -2] = em[-1, -2]
    for t in range(n_frames - 2, -1, -1):
        q = bwd[t + 1]
        acc = q.copy()
        acc[:-1] = np.logaddexp(acc[:-1], q[1:])         # to s+1
        if n_states > 2:                                 # to s+2 where allowed
            acc[:-2] = np.where(can_skip[2:], np.logaddexp(acc[:-2], q[2:]), acc[:-2])
        bwd[t] = em[t] + acc

    occ = np.exp(fwd + bwd - em - log_z)                 # state posteriors
    grad = np.zeros_like(e)
    for s in range(n_states):                            # scatter by label
        grad[:, labels[s]] -= occ[:, s]
    return float(-log_z), grad.astype(np.float32)


def ctc_validate(emissions, target, blank):
    """Reference check order for ctc_loss_grad (criterion.py:92-111,140-141).
    Returns None when valid, else (exception-class-name, message)."""
    e = np.asarray(emissions, dtype=np.float64)
    if e.ndim != 2 or e.shape[0] < 1 or e.shape[1] < 1:
        return ("ContractError", f"emissions must be T-by-N with T,N >= 1, got shape {e.shape}")
    if not np.isfinite(e).all():
        return ("NumericError", "emissions contain non-finite values")
    t_frames, n = e.shape
    if not 0 <= blank < n:
        return ("ContractError", f"blank id {blank} outside [0, {n})")
    rows = lse(e, axis=1)
    if np.abs(rows).max() > 1e-2:
        return ("ContractError", "CTC emissions rows must be log-normalized")
    y = np.asarray(list(target), dtype=np.int64)
    if y.size and (y.min() < 0 or y.max() >= n):
        return ("TargetError", "target ids out of range")
    if np.any(y == blank):
        return ("TargetError", f"CTC target contains the blank id {blank}")
    reps = int(np.sum(y[1:] == y[:-1])) if y.size > 1 else 0
    if t_frames < y.size + reps:
        return ("InfeasibleTargetError", "target needs more frames")
    return None


# --------------------------------------------------------------------- ASG --

def asg(emissions, target, transitions):
    """ASG loss = full-graph score - constrained score, with gradients
    w.r.t. emissions and transitions (criterion.py:167-247).

    Naming follows wav2letter++: *fcc* is the fully connected normaliser
    (reference ``ga``/``gb``/``fal``), *fac* the force-aligned term (reference
    ``fa``/``fb``/``fcc``).  Returns (loss, grad_e f32[T,N], grad_A f32[N,N])."""
    e = np.asarray(emissions, dtype=np.float64)
    a = np.asarray(transitions, dtype=np.float64)
    y = np.asarray(list(target), dtype=np.int64)
    n_frames, n_tok = e.shape
    n_lab = y.size

    # -- fac: constrained linear graph (criterion.py:193-224)
    ey = e[:, y]                                         # [T, L]
    self_loop = a[y, y]
    advance = a[y[1:], y[:-1]] if n_lab > 1 else np.zeros(0)
    fa = np.full((n_frames, n_lab), NEG_INF)
    fa[0, 0] = ey[0, 0]
    for t in range(1, n_frames):
        p = fa[t - 1]
        acc = p + self_loop
        if n_lab > 1:
            acc[1:] = np.logaddexp(acc[1:], p[:-1] + advance)
        fa[t] = ey[t] + acc
    fac_score = fa[-1, -1]

    fb = np.full((n_frames, n_lab), NEG_INF)
    fb[-1, -1] = ey[-1, -1]
    for t in range(n_frames - 2, -1, -1):
        q = fb[t + 1]
        acc = q + self_loop
        if n_lab > 1:
            acc[:-1] = np.logaddexp(acc[:-1], q[1:] + advance)
        fb[t] = ey[t] + acc

    fac_occ = np.exp(fa + fb - ey - fac_score)           # [T, L]
    fac_ge = np.zeros((n_frames, n_tok))
    for l in range(n_lab):
        fac_ge[:, y[l]] += fac_occ[:, l]
    fac_ga = np.zeros((n_tok, n_tok))
    if n_frames > 1:
        stay_occ = np.exp(fa[:-1] + self_loop + fb[1:] - fac_score)     # [T-1, L]
        np.add.at(fac_ga, (y, y), stay_occ.sum(axis=0))
        if n_lab > 1:
            move_occ = np.exp(fa[:-1, :-1] + advance + fb[1:, 1:] - fac_score)
            np.add.at(fac_ga, (y[1:], y[:-1]), move_occ.sum(axis=0))

    # -- fcc: fully connected N x N graph (criterion.py:227-241)
    ga = np.empty((n_frames, n_tok))
    ga[0] = e[0]
    for t in range(1, n_frames):
        ga[t] = e[t] + lse(ga[t - 1][None, :] + a, axis=1)   # A[to][from]
    fcc_score = lse(ga[-1])
    gb = np.empty((n_frames, n_tok))
    gb[-1] = e[-1]
    for t in range(n_frames - 2, -1, -1):
        gb[t] = e[t] + lse(gb[t + 1][:, None] + a, axis=0)
    fcc_ge = np.exp(ga + gb - e - fcc_score)
    fcc_ga = np.zeros((n_tok, n_tok))
    for t in range(1, n_frames):
        fcc_ga += np.exp(ga[t - 1][None, :] + a + gb[t][:, None] - fcc_score)

    return (float(fcc_score - fac_score),
            (fcc_ge - fac_ge).astype(np.float32),
            (fcc_ga - fac_ga).astype(np.float32))


def asg_validate(emissions, target, transitions):
    """Reference check order for asg_loss_grad (criterion.py:174-190)."""
    e = np.asarray(emissions, dtype=np.float64)
    if e.ndim != 2 or e.shape[0] < 1 or e.shape[1] < 1:
        return ("ContractError", "bad emissions shape")
    if not np.isfinite(e).all():
        return ("NumericError", "emissions contain non-finite values")
    n = e.shape[1]
    a = np.asarray(transitions, dtype=np.float64)
    if a.shape != (n, n):
        return ("ContractError", "bad transitions shape")
    if not np.isfinite(a).all():
        return ("NumericError", "transitions contain non-finite values")
    y = np.asarray(list(target), dtype=np.int64)
    if y.size and (y.min() < 0 or y.max() >= n):
        return ("TargetError", "target ids out of range")
    if y.size == 0:
        return ("TargetError", "ASG target must be non-empty")
    if y.size > 1 and np.any(y[1:] == y[:-1]):
        return ("ContractError", "consecutive duplicates")
    if e.shape[0] < y.size:
        return ("InfeasibleTargetError", "T < L")
    return None


# ----------------------------------------------------------------- Viterbi --

def viterbi(emissions, transitions=None):
    """Best framewise path under e_t(i) + A[i][j], ties to the lowest id
    (criterion.py:259-284).  Same float64 operation order as the reference:
    cand = dp[j] + A[i][j]; first-index argmax; dp' = e[t][i] + cand."""
    e = np.asarray(emissions, dtype=np.float64)
    n_frames, n_tok = e.shape
    a = (np.zeros((n_tok, n_tok)) if transitions is None
         else np.asarray(transitions, dtype=np.float64))
    score = e[0].copy()
    back = np.zeros((n_frames, n_tok), dtype=np.int64)
    rows = np.arange(n_tok)
    for t in range(1, n_frames):
        cand = a + score[None, :]
        back[t] = np.argmax(cand, axis=1)
        score = e[t] + cand[rows, back[t]]
    last = int(np.argmax(score))
    path = np.empty(n_frames, dtype=np.int64)
    path[-1] = last
    for t in range(n_frames - 1, 0, -1):
        path[t - 1] = back[t, path[t]]
    return path, float(score[last])


# ------------------------------------------------------ host-side helpers --

def collapse(path, kind, blank_id=None, rep_id=None):
    """Framewise path -> token sequence (criterion.py:287-310)."""
    seq = [int(v) for v in path]
    uniq = [v for k, v in enumerate(seq) if k == 0 or v != seq[k - 1]]
    if kind == "ctc":
        return [v for v in uniq if v != blank_id]
    out = []
    for v in uniq:
        out.append(out[-1] if (rep_id is not None and v == rep_id) else v)
    return out


# ------------------------------------------------- greedy evaluation --
# (trainer.py:465-514, lexicon.py:182-195)

def edit_distance(ref, hyp):
    """Levenshtein distance, unit costs (trainer.py:465-476)."""
    ref, hyp = list(ref), list(hyp)
    if not ref:
        return len(hyp)
    prev = list(range(len(hyp) + 1))
    for i, r in enumerate(ref, start=1):
        cur = [i] + [0] * len(hyp)
        for j, h in enumerate(hyp, start=1):
            cur[j] = min(prev[j] + 1, cur[j - 1] + 1, prev[j - 1] + (r != h))
        prev = cur
    return prev[-1]


def split_on_silence(ids, silence):
    """Silence-free groups, empty groups dropped (lexicon.py:182-195)."""
    groups, cur = [], []
    for t in ids:
        if t == silence:
            if cur:
                groups.append(cur)
            cur = []
        else:
            cur.append(int(t))
    if cur:
        groups.append(cur)
    return groups


def greedy_metrics(path, ref, kind, blank_id=None, rep_id=None, silence=None):
    """One utterance of trainer.evaluate (trainer.py:496-510): the collapsed
    path's token edit distance, word edit distance and reference word count."""
    hyp = collapse(path, kind, blank_id, rep_id)
    ref = [int(t) for t in ref]
    if silence is not None:
        rw = [tuple(g) for g in split_on_silence(ref, silence)]
        hw = [tuple(g) for g in split_on_silence(hyp, silence)]
    else:
        rw, hw = [tuple(ref)], [tuple(hyp)]
    return hyp, edit_distance(ref, hyp), edit_distance(rw, hw), len(rw)


# ------------------------------------------------ brute-force enumeration --
# (restated from tests/oracles.py:87-144; exponential, toy sizes only)

def _collapse_ctc(path, blank):
    uniq = [k for i, k in enumerate(path) if i == 0 or k != path[i - 1]]
    return [k for k in uniq if k != blank]


def _score(e, a, path):
    s = sum(e[t][path[t]] for t in range(len(path)))
    return s + sum(a[path[t]][path[t - 1]] for t in range(1, len(path)))


def ctc_enum(emissions, target, blank):
    e = np.asarray(emissions, dtype=np.float64)
    want = list(target)
    tot = NEG_INF
    for path in itertools.product(range(e.shape[1]), repeat=e.shape[0]):
        if _collapse_ctc(path, blank) == want:
            tot = np.logaddexp(tot, sum(e[t][path[t]] for t in range(e.shape[0])))
    return float(-tot)


def asg_enum(emissions, target, transitions):
    e = np.asarray(emissions, dtype=np.float64)
    a = np.asarray(transitions, dtype=np.float64)
    n_frames, n_tok = e.shape
    y = list(target)
    full = NEG_INF
    for path in itertools.product(range(n_tok), repeat=n_frames):
        full = np.logaddexp(full, _score(e, a, path))
    con = NEG_INF
    for al in itertools.product(range(len(y)), repeat=n_frames):
        if al[0] != 0 or al[-1] != len(y) - 1:
            continue
        if any(al[t] - al[t - 1] not in (0, 1) for t in range(1, n_frames)):
            continue
        con = np.logaddexp(con, _score(e, a, [y[i] for i in al]))
    return float(full - con)


def viterbi_enum(emissions, transitions=None):
    e = np.asarray(emissions, dtype=np.float64)
    n_frames, n_tok = e.shape
    a = np.zeros((n_tok, n_tok)) if transitions is None else np.asarray(transitions, np.float64)
    best, arg = NEG_INF, []
    for path in itertools.product(range(n_tok), repeat=n_frames):
        s = _score(e, a, path)
        if s > best + 1e-12:
            best, arg = s, [list(path)]
        elif s >= best - 1e-12:
            arg.append(list(path))
    return best, arg


# --------------------------------------------------- batched convenience --

def asg_batch(em, em_len, targets, tgt_len, transitions):
    """Per-utterance oracle over the padded batch layout (data.py:91-99):
    returns loss f64[B], grad_e f32[B,Tmax,N] (zero padded), grad_A f32[N,N]
    summed over utterances (trainer.py:417-418 before the /B)."""
    b_sz, t_max, n = em.shape
    loss = np.zeros(b_sz)
    ge = np.zeros((b_sz, t_max, n), dtype=np.float32)
    ga = np.zeros((n, n), dtype=np.float64)
    for b in range(b_sz):
        t, l = int(em_len[b]), int(tgt_len[b])
        lo, g1, g2 = asg(em[b, :t], targets[b, :l], transitions)
        loss[b] = lo
        ge[b, :t] = g1
        ga += g2
    return loss, ge, ga.astype(np.float32)


def ctc_batch(em, em_len, targets, tgt_len, blank):
    b_sz, t_max, n = em.shape
    loss = np.zeros(b_sz)
    ge = np.zeros((b_sz, t_max, n), dtype=np.float32)
    for b in range(b_sz):
        t, l = int(em_len[b]), int(tgt_len[b])
        lo, g1 = ctc(em[b, :t], targets[b, :l], blank)
        loss[b] = lo
        ge[b, :t] = g1
    return loss, ge


def viterbi_batch(em, em_len, transitions=None):
    b_sz, t_max, _ = em.shape
    paths = np.zeros((b_sz, t_max), dtype=np.int64)
    scores = np.zeros(b_sz)
    for b in range(b_sz):
        t = int(em_len[b])
        p, s = viterbi(em[b, :t], transitions)
        paths[b, :t] = p
        scores[b] = s
    return paths, scores


# ------------------------------------------------------ synthetic inputs --

def log_softmax_rows(x):
    """Row log-softmax in float64 (the CTC precondition; test_criterion.py:27-32)."""
    x = np.asarray(x, dtype=np.float64)
    return x - lse(x, axis=-1)[..., None]


def synth_asg(seed, b_sz, t_max, n, l_max, ragged=False):
    """SURVEY §8(d) ASG generator: N(0,1) f32 emissions and transitions,
    targets uniform in [0,N) with consecutive duplicates resampled."""
    rng = np.random.default_rng(seed)
    em = rng.standard_normal((b_sz, t_max, n), dtype=np.float32)
    trans = rng.standard_normal((n, n)).astype(np.float32)
    em_len = np.full(b_sz, t_max, dtype=np.int32)
    tgt_len = np.full(b_sz, l_max, dtype=np.int32)
    if ragged:
        em_len = rng.integers(max(1, t_max // 2), t_max + 1, size=b_sz).astype(np.int32)
        tgt_len = rng.integers(max(1, l_max // 2), l_max + 1, size=b_sz).astype(np.int32)
        tgt_len = np.minimum(tgt_len, em_len)
    targets = np.full((b_sz, l_max), -1, dtype=np.int64)
    for b in range(b_sz):
        seq = [int(rng.integers(0, n))]
        while len(seq) < tgt_len[b]:
            v = int(rng.integers(0, n))
            if v != seq[-1]:
                seq.append(v)
        targets[b, :tgt_len[b]] = seq
        if ragged:
            em[b, em_len[b]:] = 0.0
    return em, em_len, targets, tgt_len, trans


def synth_ctc(seed, b_sz, t_max, n, l_max, ragged=False):
    """SURVEY §8(d) CTC generator: emissions = log_softmax(2 N(0,1)) computed
    in f64 then cast to f32; blank = N-1; labels uniform in [0,N-1), repeats
    allowed, feasibility T >= L + repeats enforced."""
    rng = np.random.default_rng(seed)
    em = log_softmax_rows(2.0 * rng.standard_normal((b_sz, t_max, n))).astype(np.float32)
    blank = n - 1
    em_len = np.full(b_sz, t_max, dtype=np.int32)
    if ragged:
        em_len = rng.integers(max(1, t_max // 2), t_max + 1, size=b_sz).astype(np.int32)
    targets = np.full((b_sz, l_max), -1, dtype=np.int64)
    tgt_len = np.zeros(b_sz, dtype=np.int32)
    for b in range(b_sz):
        l_b = l_max if not ragged else int(rng.integers(max(0, l_max // 2), l_max + 1))
        while True:
            seq = rng.integers(0, n - 1, size=l_b)
            reps = int(np.sum(seq[1:] == seq[:-1])) if l_b > 1 else 0
            if l_b + reps <= em_len[b]:
                break
            l_b = max(0, l_b - 1)
        targets[b, :l_b] = seq
        tgt_len[b] = l_b
        if ragged:
            em[b, em_len[b]:] = 0.0
    return em, em_len, targets, tgt_len, blank
