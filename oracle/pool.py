"""Process-pool driver for the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Full-batch parity at the BASELINE configs (B=64, T=1600) needs the float64
oracle (oracle/criterion_oracle.py) on every utterance; one utterance per
task over all host cores keeps that to seconds.  Used by tests/ (checker
only) and bench.py's CPU baseline; never by the product package.
"""

from __future__ import annotations

import concurrent.futures as cf
import multiprocessing as mp
import os

import numpy as np


def _cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def _task(args):
    from oracle import criterion_oracle as orc
    kind, payload = args
    if kind == "asg":
        e, y, a = payload
        return orc.asg(e, y, a)
    if kind == "ctc":
        e, y, blank = payload
        return orc.ctc(e, y, blank)
    if kind == "viterbi":
        e, a = payload
        return orc.viterbi(e, a)
    raise ValueError(kind)


def _run(tasks, procs):
    procs = procs or min(_cores(), len(tasks)) or 1
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ.setdefault(k, "1")
    # spawn: the parent may hold a CUDA context; the workers only run numpy
    with cf.ProcessPoolExecutor(max_workers=procs, mp_context=mp.get_context("spawn")) as ex:
        return list(ex.map(_task, tasks, chunksize=1))


def asg_batch(em, em_len, targets, tgt_len, transitions, procs=None):
    """Same contract as criterion_oracle.asg_batch, one utterance per task;
    also returns the per-utterance transition gradients."""
    b_sz, t_max, n = em.shape
    tasks = [("asg", (em[b, :int(em_len[b])], targets[b, :int(tgt_len[b])], transitions))
             for b in range(b_sz)]
    res = _run(tasks, procs)
    loss = np.array([r[0] for r in res], dtype=np.float64)
    ge = np.zeros((b_sz, t_max, n), dtype=np.float32)
    ga_utt = np.zeros((b_sz, n, n), dtype=np.float32)
    for b, r in enumerate(res):
        ge[b, :int(em_len[b])] = r[1]
        ga_utt[b] = r[2]
    return loss, ge, ga_utt


def ctc_batch(em, em_len, targets, tgt_len, blank, procs=None):
    b_sz, t_max, n = em.shape
    tasks = [("ctc", (em[b, :int(em_len[b])], targets[b, :int(tgt_len[b])], blank))
             for b in range(b_sz)]
    res = _run(tasks, procs)
    loss = np.array([r[0] for r in res], dtype=np.float64)
    ge = np.zeros((b_sz, t_max, n), dtype=np.float32)
    for b, r in enumerate(res):
        ge[b, :int(em_len[b])] = r[1]
    return loss, ge


def viterbi_batch(em, em_len, transitions=None, procs=None):
    b_sz, t_max, _ = em.shape
    res = _run([("viterbi", (em[b, :int(em_len[b])], transitions)) for b in range(b_sz)], procs)
    paths = np.zeros((b_sz, t_max), dtype=np.int64)
    scores = np.zeros(b_sz)
    for b, (p, s) in enumerate(res):
        paths[b, :int(em_len[b])] = p
        scores[b] = s
    return paths, scores
