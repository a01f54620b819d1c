"""Sequence criteria on B200: CTC, ASG with learnable transitions, Viterbi.

Drop-in for the reference criterion module (pkg/src/asrkit/criterion.py):
the same public names, signatures, return types and exception classes, with
every loss, gradient and alignment computed by the sm_100a kernels of
``libw2l_criterion.so`` (include/w2l_criterion.h).  There is no CPU
fallback: without a CUDA device or the built library every compute entry
point raises.

Two families of entry points:

* reference-compatible, per utterance (``ctc_loss_grad``, ``asg_loss_grad``,
  ``viterbi``): numpy in, numpy out, float64 internals on the GPU exactly as
  the reference specifies (criterion.py:1-7) -- the float64 log-domain
  kernels (w2l_*_f64);
* batched hot path (``asg_loss_grad_batched``, ``ctc_loss_grad_batched``,
  ``viterbi_batched``) over the padded batch layout of data.Batch
  (data.py:91-99): emissions f32 [B,T,N], int32 lengths, int64 targets padded
  with -1.  fp32 scaled-linear-domain kernels with a per-utterance guard and
  float64 recompute of any utterance that fails it.

Losses are per-utterance sums; the batch mean (and the /B of the transition
gradient) stays with the caller (criterion.py:4-6, trainer.py:442-447).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _native as nat
from .errors import (ContractError, DeviceError, InfeasibleTargetError, NumericError,
                     TargetError, raise_for_status)

# the ASG repetition token's symbol (lexicon.py:51-54); token tables are duck
# typed: the criterion path needs only len(table), table.rep_id and
# table.symbol(id), which the reference's TokenTable provides
REPETITION_SYMBOL = "<2>"

__all__ = [
    "LossOutput", "BatchLossOutput", "validate_target", "ctc_loss_grad", "asg_loss_grad",
    "viterbi", "collapse_path", "CtcCriterion", "AsgCriterion", "make_criterion",
    "asg_loss_grad_batched", "ctc_loss_grad_batched", "viterbi_batched", "asg_loss",
    "ctc_loss", "check_status", "GreedyEval", "greedy_eval_batched", "evaluate_batch",
]


@dataclass
class LossOutput:
    """criterion.py:44-48."""
    loss: float
    grad_emissions: np.ndarray
    grad_transitions: Optional[np.ndarray] = None


@dataclass
class BatchLossOutput:
    loss: torch.Tensor                       # f64 [B]
    grad_emissions: torch.Tensor             # f32 [B, Tmax, N]
    grad_transitions: Optional[torch.Tensor] = None        # f32 [N, N], sum over B
    grad_transitions_per_utt: Optional[torch.Tensor] = None  # f32 [B, N, N]
    status: Optional[torch.Tensor] = None    # int32 [B]
    stage_ms: Optional[dict] = None          # per-stage device times (trace=True)


# ------------------------------------------------------------------ plumbing --

def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise nat.NativeLibraryError(
            "no CUDA device: the criterion kernels are sm_100a-only and there is no CPU "
            "fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _stream() -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _p(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _dev_tensor(x, dtype, dev) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=dev, dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x), dtype=dtype).to(dev, non_blocking=True)


def _workspace(nbytes: int, dev, ws: Optional[torch.Tensor] = None) -> torch.Tensor:
    if ws is not None and ws.numel() >= nbytes and ws.device == dev:
        return ws
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=dev)


def _check_call(rc: int, what: str) -> None:
    if rc != nat.OK:
        detail = nat.lib().w2l_status_string(rc).decode()
        if rc == nat.ERR_CUDA:
            detail += f" ({nat.lib().w2l_last_cuda_error().decode()})"
        raise_for_status(rc, f"{what}: {detail}")


def _stage_times(kind: int, ms, n) -> dict:
    lib = nat.lib()
    return {lib.w2l_stage_name(kind, i).decode(): float(ms[i]) for i in range(n.value)}


def _first_error(status: torch.Tensor):
    bad = ctypes.c_int32(-1)
    code = nat.lib().w2l_status_first_error(_p(status), status.numel(), ctypes.byref(bad),
                                            _stream())
    return code, bad.value


# ------------------------------------------------- host-side integer prep --

def _check_emissions_shape(emissions) -> np.ndarray:
    """Shape half of _check_emissions (criterion.py:23-29); finiteness is
    checked on the device."""
    e = emissions.detach().cpu().numpy() if isinstance(emissions, torch.Tensor) else emissions
    e = np.asarray(e, dtype=np.float64)
    if e.ndim != 2 or e.shape[0] < 1 or e.shape[1] < 1:
        raise ContractError(f"emissions must be T-by-N with T,N >= 1, got shape {e.shape}")
    if e.shape[1] > nat.MAX_TOKENS:
        raise ContractError(f"at most {nat.MAX_TOKENS} output tokens are supported, got {e.shape[1]}")
    return np.ascontiguousarray(e)


def _target_ids(target) -> np.ndarray:
    """criterion.py:32-35 (the range half is checked on the device)."""
    if isinstance(target, torch.Tensor):
        target = target.detach().cpu().tolist()
    y = np.asarray(list(target), dtype=np.int64)
    if y.ndim != 1:
        raise TargetError("target must be a flat sequence of token ids")
    return y


def validate_target(tokens, criterion_kind: str, table):
    """Canonicalise a target for the criterion (criterion.py:51-79): CTC passes
    through; ASG replaces the second of each consecutive duplicate with the
    repetition token, left to right ("a a a" -> "a <2> a")."""
    ids = [int(t) for t in tokens]
    n = len(table)
    bad = [t for t in ids if not 0 <= t < n]
    if bad:
        raise TargetError(f"target id {bad[0]} outside token table of size {n}")
    if criterion_kind == "ctc":
        return ids
    if criterion_kind != "asg":
        raise ContractError(f"unknown criterion kind {criterion_kind!r}")
    out: list = []
    for t in ids:
        if not out or out[-1] != t:
            out.append(t)
            continue
        if table.rep_id is None:
            raise TargetError(f"ASG target repeats {table.symbol(t)!r} but the token table "
                              f"has no {REPETITION_SYMBOL!r} symbol")
        out.append(table.rep_id)
    return out


def collapse_path(path, criterion_kind: str, blank_id=None, rep_id=None):
    """Framewise path -> tokens (criterion.py:287-310): drop repeats; CTC then
    drops blanks, ASG expands ``<2>`` into a copy of its predecessor."""
    ids = [int(t) for t in path]
    merged = [t for k, t in enumerate(ids) if k == 0 or t != ids[k - 1]]
    if criterion_kind == "ctc":
        if blank_id is None:
            raise ContractError("CTC collapse needs blank_id")
        return [t for t in merged if t != blank_id]
    if criterion_kind != "asg":
        raise ContractError(f"unknown criterion kind {criterion_kind!r}")
    out: list = []
    for t in merged:
        if rep_id is not None and t == rep_id:
            if not out:
                raise ContractError("repetition token with no preceding token")
            out.append(out[-1])
        else:
            out.append(t)
    return out


# ------------------------------------------------ reference-compatible API --

def _asg_message(code, e, y, a):
    n = e.shape[1]
    if code == nat.ERR_NUMERIC:
        return ("emissions contain non-finite values" if not np.isfinite(e).all()
                else "transitions contain non-finite values")
    if code == nat.ERR_TARGET:
        if y.size and (y.min() < 0 or y.max() >= n):
            return f"target ids must lie in [0, {n}), got range [{y.min()}, {y.max()}]"
        return "ASG target must be non-empty"
    if code == nat.ERR_CONTRACT:
        return "ASG target has consecutive duplicates; canonicalize first"
    if code == nat.ERR_INFEASIBLE:
        return f"target of length {y.size} needs at least {y.size} frames, got {e.shape[0]}"
    return "device failure"


def asg_loss_grad(emissions, target, transitions) -> LossOutput:
    """ASG loss (full-graph score minus forced-alignment score) with gradients
    w.r.t. emissions and transitions (criterion.py:167-247).  transitions[i][j]
    scores moving from token j at t-1 to token i at t.  Float64 internals."""
    e = _check_emissions_shape(emissions)
    t_frames, n = e.shape
    a = transitions.detach().cpu().numpy() if isinstance(transitions, torch.Tensor) else transitions
    a = np.asarray(a, dtype=np.float64)
    if a.shape != (n, n):
        if not np.isfinite(e).all():          # the reference checks emissions first
            raise NumericError("emissions contain non-finite values")
        raise ContractError(f"transitions must be {n}x{n}, got {a.shape}")
    y = _target_ids(target)
    if y.size > nat.MAX_ASG_LABELS:
        raise ContractError(f"ASG targets longer than {nat.MAX_ASG_LABELS} are not supported")
    dev = _device()
    lmax = max(int(y.size), 1)
    tg = np.full((1, lmax), -1, dtype=np.int64)
    tg[0, :y.size] = y
    em_d = _dev_tensor(e[None], torch.float64, dev)
    a_d = _dev_tensor(a, torch.float64, dev)
    tg_d = _dev_tensor(tg, torch.int64, dev)
    el_d = torch.tensor([t_frames], dtype=torch.int32, device=dev)
    tl_d = torch.tensor([y.size], dtype=torch.int32, device=dev)
    loss = torch.empty(1, dtype=torch.float64, device=dev)
    ge = torch.empty((1, t_frames, n), dtype=torch.float32, device=dev)
    ga = torch.empty((n, n), dtype=torch.float32, device=dev)
    st = torch.empty(1, dtype=torch.int32, device=dev)
    lib = nat.lib()
    nbytes = lib.w2l_asg_workspace_bytes_f64(1, t_frames, n, lmax)
    ws = _workspace(nbytes, dev)
    rc = lib.w2l_asg_loss_grad_f64(_p(em_d), _p(el_d), _p(tg_d), _p(tl_d), _p(a_d), 1, t_frames,
                                   n, lmax, _p(loss), _p(ge), _p(ga), None, _p(st), _p(ws),
                                   ws.numel(), _stream())
    _check_call(rc, "w2l_asg_loss_grad_f64")
    code, _ = _first_error(st)
    if code != nat.OK:
        raise_for_status(code, _asg_message(code, e, y, a))
    return LossOutput(loss=float(loss.item()), grad_emissions=ge[0].cpu().numpy(),
                      grad_transitions=ga.cpu().numpy())


def _ctc_message(code, e, y, blank):
    n = e.shape[1]
    if code == nat.ERR_NUMERIC:
        return "emissions contain non-finite values"
    if code == nat.ERR_CONTRACT:
        if not 0 <= blank < n:
            return f"blank id {blank} outside [0, {n})"
        m = e.max(axis=1, keepdims=True)
        rows = (np.log(np.exp(e - m).sum(axis=1, keepdims=True)) + m)[:, 0]
        worst = rows[np.abs(rows).argmax()]
        return f"CTC emissions rows must be log-normalized (worst row logsumexp = {worst:.4f})"
    if code == nat.ERR_TARGET:
        if y.size and (y.min() < 0 or y.max() >= n):
            return f"target ids must lie in [0, {n}), got range [{y.min()}, {y.max()}]"
        return f"CTC target contains the blank id {blank}"
    if code == nat.ERR_INFEASIBLE:
        reps = int(np.sum(y[1:] == y[:-1])) if y.size > 1 else 0
        if e.shape[0] < y.size + reps:
            return (f"target of length {y.size} with {reps} consecutive repeats needs at least "
                    f"{y.size + reps} frames, got {e.shape[0]}")
        return "no feasible alignment (forward score is -inf)"
    return "device failure"


def ctc_loss_grad(emissions, target, blank_id: int) -> LossOutput:
    """CTC negative log marginal over blank-augmented alignments, gradient via
    forward-backward posteriors (criterion.py:84-162).  Rows must be
    log-normalised (|logsumexp| <= 1e-2).  Float64 internals."""
    e = _check_emissions_shape(emissions)
    t_frames, n = e.shape
    y = _target_ids(target)
    if y.size > nat.MAX_CTC_LABELS:
        raise ContractError(f"CTC targets longer than {nat.MAX_CTC_LABELS} are not supported")
    dev = _device()
    lmax = max(int(y.size), 1)
    tg = np.full((1, lmax), -1, dtype=np.int64)
    tg[0, :y.size] = y
    em_d = _dev_tensor(e[None], torch.float64, dev)
    tg_d = _dev_tensor(tg, torch.int64, dev)
    el_d = torch.tensor([t_frames], dtype=torch.int32, device=dev)
    tl_d = torch.tensor([y.size], dtype=torch.int32, device=dev)
    loss = torch.empty(1, dtype=torch.float64, device=dev)
    ge = torch.empty((1, t_frames, n), dtype=torch.float32, device=dev)
    st = torch.empty(1, dtype=torch.int32, device=dev)
    lib = nat.lib()
    ws = _workspace(lib.w2l_ctc_workspace_bytes_f64(1, t_frames, n, lmax), dev)
    rc = lib.w2l_ctc_loss_grad_f64(_p(em_d), _p(el_d), _p(tg_d), _p(tl_d), int(blank_id), 1,
                                   t_frames, n, lmax, _p(loss), _p(ge), _p(st), _p(ws),
                                   ws.numel(), _stream())
    _check_call(rc, "w2l_ctc_loss_grad_f64")
    code, _ = _first_error(st)
    if code != nat.OK:
        raise_for_status(code, _ctc_message(code, e, y, int(blank_id)))
    return LossOutput(loss=float(loss.item()), grad_emissions=ge[0].cpu().numpy())


def viterbi(emissions, transitions=None):
    """Highest-scoring framewise path under e_t(i) + A[i][j]; ties to the lower
    id (criterion.py:259-284).  Returns (int64 path[T], float score); paths and
    scores are bit-identical to the float64 reference."""
    e = _check_emissions_shape(emissions)
    t_frames, n = e.shape
    a = None
    if transitions is not None:
        a = transitions.detach().cpu().numpy() if isinstance(transitions, torch.Tensor) else transitions
        a = np.asarray(a, dtype=np.float64)
        if a.shape != (n, n):
            if not np.isfinite(e).all():
                raise NumericError("emissions contain non-finite values")
            raise ContractError(f"transitions must be {n}x{n}, got {a.shape}")
    dev = _device()
    em_d = _dev_tensor(e[None], torch.float64, dev)
    a_d = None if a is None else _dev_tensor(a, torch.float64, dev)
    el_d = torch.tensor([t_frames], dtype=torch.int32, device=dev)
    path = torch.empty((1, t_frames), dtype=torch.int64, device=dev)
    score = torch.empty(1, dtype=torch.float64, device=dev)
    st = torch.empty(1, dtype=torch.int32, device=dev)
    lib = nat.lib()
    ws = _workspace(lib.w2l_viterbi_workspace_bytes(1, t_frames, n), dev)
    rc = lib.w2l_viterbi_f64(_p(em_d), _p(el_d), _p(a_d), 1, t_frames, n, _p(path), _p(score),
                             _p(st), _p(ws), ws.numel(), _stream())
    _check_call(rc, "w2l_viterbi_f64")
    code, _ = _first_error(st)
    if code != nat.OK:
        raise_for_status(code, "emissions contain non-finite values")
    return path[0].cpu().numpy(), float(score.item())


# -------------------------------------------------------- batched hot path --

def _batch_inputs(emissions, em_len, targets, tgt_len, dev):
    em = _dev_tensor(emissions, torch.float32, dev)
    if em.dim() != 3:
        raise ContractError(f"batched emissions must be B x T x N, got shape {tuple(em.shape)}")
    b, t_max, n = em.shape
    if n > nat.MAX_TOKENS:
        raise ContractError(f"at most {nat.MAX_TOKENS} output tokens are supported, got {n}")
    el = _dev_tensor(em_len, torch.int32, dev).reshape(-1)
    tg = _dev_tensor(targets, torch.int64, dev)
    if tg.dim() != 2 or tg.shape[0] != b:
        raise ContractError(f"targets must be B x Lmax, got shape {tuple(tg.shape)}")
    if tg.shape[1] == 0:
        tg = torch.full((b, 1), -1, dtype=torch.int64, device=dev)
    tl = _dev_tensor(tgt_len, torch.int32, dev).reshape(-1)
    if el.numel() != b or tl.numel() != b:
        raise ContractError("em_len and tgt_len must have one entry per utterance")
    return em, el, tg, tl


def _flags(fallback, phase: str, loss_only: bool = False, logits: bool = False,
           force_exact: bool = False, route: bool = True, stream_grad: bool = False) -> int:
    # fallback: True (every precision tier), False (fp32 only) or "f64" (the
    # fp32 and fp64 scaled-linear tiers, no log-domain kernel)
    f = 0 if fallback else nat.FLAG_NO_FALLBACK
    if fallback == "f64":
        f = nat.FLAG_NO_LOG_FALLBACK
    if force_exact:
        f |= nat.FLAG_FORCE_EXACT
    if not route:
        f |= nat.FLAG_NO_ROUTE
    if loss_only:
        f |= nat.FLAG_LOSS_ONLY
    if logits:
        f |= nat.FLAG_CTC_LOGITS
    if stream_grad:
        f |= nat.FLAG_STREAM_GRAD
    if phase == "chain":
        f |= nat.FLAG_PHASE_CHAIN
    elif phase == "grad":
        f |= nat.FLAG_PHASE_GRAD
    elif phase == "validate":
        f |= nat.FLAG_PHASE_VALIDATE
    elif phase == "rest":
        f |= nat.FLAG_VALIDATED
    elif phase != "all":
        raise ContractError("phase must be 'all', 'chain', 'grad', 'validate' or 'rest', "
                            f"got {phase!r}")
    return f


def _raise_batch(status: torch.Tensor, what: str) -> None:
    code, bad = _first_error(status)
    if code != nat.OK:
        detail = nat.lib().w2l_status_string(code).decode()
        if code == nat.ERR_CUDA:
            detail += f" ({nat.lib().w2l_last_cuda_error().decode()})"
        raise_for_status(code, f"{what}: utterance {bad}: {detail}")


def asg_loss_grad_batched(emissions, em_len, targets, tgt_len, transitions, *, check=True,
                          per_utterance_grad_transitions=False, workspace=None,
                          out: Optional[BatchLossOutput] = None,
                          fallback=True, trace: bool = False,
                          phase: str = "all", loss_only: bool = False,
                          force_exact: bool = False, route: bool = True,
                          stream_grad: bool = False) -> BatchLossOutput:
    """Batched ASG loss + gradients on the device (fp32 path).

    emissions f32 [B,Tmax,N]; em_len int [B]; targets int64 [B,Lmax] padded
    with -1 (canonical: no consecutive duplicates, see validate_target);
    tgt_len int [B]; transitions f32 [N,N] (A[to][from]).  Returns loss f64 [B],
    grad_emissions f32 [B,Tmax,N], grad_transitions f32 [N,N] summed over the
    batch and (optionally) per utterance.  check=True synchronises and raises
    the reference exception for the first failing utterance.  Precision
    tiers: an utterance failing the fp32 guard is recomputed with fp64 lanes,
    one failing that guard too by the float64 log-domain kernel;
    fallback=False stops after the fp32 tier and fallback="f64" after the
    fp64 tier (the rest report W2L_ERR_PRECISION) -- diagnostics.
    phase="chain" | "grad" splits the call (W2L_FLAG_PHASE_*): "chain" runs
    the recursions into the workspace, a later "grad" call with the same
    inputs, workspace and out on the same stream order finishes it.
    phase="validate" runs only the input checks; a later phase="rest" call
    (same inputs, workspace, out) runs everything after them
    (W2L_FLAG_PHASE_VALIDATE / W2L_FLAG_VALIDATED: staggering two criteria).
    stream_grad=True (W2L_FLAG_STREAM_GRAD) starts the gradient kernels on
    the middle frames while the recursions are still running.
    loss_only=True (evaluation, W2L_FLAG_LOSS_ONLY) runs the recursions
    and the loss only: grad_emissions / grad_transitions are not computed.
    force_exact=True (W2L_FLAG_FORCE_EXACT) computes every utterance with
    the float64 log-domain kernel (the guard's fallback path).  route=False
    (W2L_FLAG_NO_ROUTE) disables the precision routing that sends a batch of
    very peaky emissions straight to the fp64 tier (the results are the same
    either way; see include/w2l_criterion.h)."""
    dev = _device()
    em, el, tg, tl = _batch_inputs(emissions, em_len, targets, tgt_len, dev)
    b, t_max, n = em.shape
    lmax = tg.shape[1]
    a = _dev_tensor(transitions, torch.float32, dev)
    if tuple(a.shape) != (n, n):
        raise ContractError(f"transitions must be {n}x{n}, got {tuple(a.shape)}")
    if lmax > nat.MAX_ASG_LABELS:
        raise ContractError(f"ASG targets longer than {nat.MAX_ASG_LABELS} are not supported")
    lib = nat.lib()
    ws = _workspace(lib.w2l_asg_workspace_bytes(b, t_max, n, lmax), dev, workspace)
    if out is None:
        out = BatchLossOutput(
            loss=torch.empty(b, dtype=torch.float64, device=dev),
            grad_emissions=torch.empty((b, t_max, n), dtype=torch.float32, device=dev),
            grad_transitions=torch.empty((n, n), dtype=torch.float32, device=dev),
            grad_transitions_per_utt=(torch.empty((b, n, n), dtype=torch.float32, device=dev)
                                      if per_utterance_grad_transitions else None),
            status=torch.empty(b, dtype=torch.int32, device=dev))
    args = (_p(em), _p(el), _p(tg), _p(tl), _p(a), b, t_max, n, lmax, _p(out.loss),
            _p(out.grad_emissions), _p(out.grad_transitions), _p(out.grad_transitions_per_utt),
            _p(out.status), _p(ws), ws.numel(), _flags(fallback, phase, loss_only,
                                                       force_exact=force_exact, route=route,
                                                       stream_grad=stream_grad),
            _stream())
    if trace:
        ms, cnt = (ctypes.c_float * 16)(), ctypes.c_int(0)
        rc = lib.w2l_asg_loss_grad_traced(*args, ms, ctypes.byref(cnt))
        out.stage_ms = _stage_times(0, ms, cnt)
    else:
        rc = lib.w2l_asg_loss_grad(*args)
    _check_call(rc, "w2l_asg_loss_grad")
    if check:
        _raise_batch(out.status, "asg_loss_grad_batched")
    return out


def ctc_loss_grad_batched(emissions, em_len, targets, tgt_len, blank_id: int, *, check=True,
                          workspace=None, out: Optional[BatchLossOutput] = None,
                          fallback=True, trace: bool = False,
                          phase: str = "all", loss_only: bool = False,
                          logits: bool = False, force_exact: bool = False,
                          route: bool = True, stream_grad: bool = False) -> BatchLossOutput:
    """Batched CTC loss + gradient on the device (fp32 path); emissions are
    log-probabilities f32 [B,Tmax,N] with |row logsumexp| <= 1e-2.  phase and
    loss_only: as for asg_loss_grad_batched.  logits=True
    (W2L_FLAG_CTC_LOGITS): emissions are unnormalised logits with
    log_softmax fused in (autodiff.py:394-411); the loss is that of
    log_softmax(emissions) and grad_emissions is the gradient with respect to
    the logits (softmax - posterior)."""
    dev = _device()
    em, el, tg, tl = _batch_inputs(emissions, em_len, targets, tgt_len, dev)
    b, t_max, n = em.shape
    lmax = tg.shape[1]
    if lmax > nat.MAX_CTC_LABELS:
        raise ContractError(f"CTC targets longer than {nat.MAX_CTC_LABELS} are not supported")
    lib = nat.lib()
    ws = _workspace(lib.w2l_ctc_workspace_bytes(b, t_max, n, lmax), dev, workspace)
    if out is None:
        out = BatchLossOutput(
            loss=torch.empty(b, dtype=torch.float64, device=dev),
            grad_emissions=torch.empty((b, t_max, n), dtype=torch.float32, device=dev),
            status=torch.empty(b, dtype=torch.int32, device=dev))
    args = (_p(em), _p(el), _p(tg), _p(tl), int(blank_id), b, t_max, n, lmax, _p(out.loss),
            _p(out.grad_emissions), _p(out.status), _p(ws), ws.numel(),
            _flags(fallback, phase, loss_only, logits, force_exact, route, stream_grad), _stream())
    if trace:
        ms, cnt = (ctypes.c_float * 16)(), ctypes.c_int(0)
        rc = lib.w2l_ctc_loss_grad_traced(*args, ms, ctypes.byref(cnt))
        out.stage_ms = _stage_times(1, ms, cnt)
    else:
        rc = lib.w2l_ctc_loss_grad(*args)
    _check_call(rc, "w2l_ctc_loss_grad")
    if check:
        _raise_batch(out.status, "ctc_loss_grad_batched")
    return out


def viterbi_batched(emissions, em_len, transitions=None, *, check=True, workspace=None):
    """Batched best paths: (int64 paths [B,Tmax] zero padded, f64 scores [B]).
    float64 max-plus on the device, bit-exact with the reference."""
    dev = _device()
    em = _dev_tensor(emissions, torch.float32, dev)
    if em.dim() != 3:
        raise ContractError(f"batched emissions must be B x T x N, got {tuple(em.shape)}")
    b, t_max, n = em.shape
    el = _dev_tensor(em_len, torch.int32, dev).reshape(-1)
    a = None if transitions is None else _dev_tensor(transitions, torch.float32, dev)
    if a is not None and tuple(a.shape) != (n, n):
        raise ContractError(f"transitions must be {n}x{n}, got {tuple(a.shape)}")
    lib = nat.lib()
    ws = _workspace(lib.w2l_viterbi_workspace_bytes(b, t_max, n), dev, workspace)
    path = torch.empty((b, t_max), dtype=torch.int64, device=dev)
    score = torch.empty(b, dtype=torch.float64, device=dev)
    st = torch.empty(b, dtype=torch.int32, device=dev)
    rc = lib.w2l_viterbi(_p(em), _p(el), _p(a), b, t_max, n, _p(path), _p(score), _p(st),
                         _p(ws), ws.numel(), _stream())
    _check_call(rc, "w2l_viterbi")
    if check:
        _raise_batch(st, "viterbi_batched")
    return path, score


# ---------------------------------------------------- greedy evaluation --

@dataclass
class GreedyEval:
    """Per-utterance greedy metrics of a batch (trainer.py:465-514):
    the collapsed hypotheses (-1 padded), their lengths, the token and word
    edit distances to the references and the references' word counts."""
    hyp: torch.Tensor
    hyp_len: torch.Tensor
    tok_dist: torch.Tensor
    word_dist: torch.Tensor
    ref_words: torch.Tensor
    status: torch.Tensor


def greedy_eval_batched(paths, path_len, targets, tgt_len, kind: str, *, blank_id=None,
                        rep_id=None, silence_id=None, check=True) -> GreedyEval:
    """Collapse a batch of framewise paths (collapse_path, criterion.py:287-310)
    and score them against the targets (edit_distance and split_on_silence,
    trainer.py:465-510) on the device.  kind "ctc" needs blank_id; "asg"
    takes the repetition token rep_id (or None)."""
    dev = _device()
    pa = _dev_tensor(paths, torch.int64, dev)
    if pa.dim() != 2:
        raise ContractError(f"paths must be B x Tmax, got {tuple(pa.shape)}")
    b, t_max = pa.shape
    pl = _dev_tensor(path_len, torch.int32, dev).reshape(-1)
    tg = _dev_tensor(targets, torch.int64, dev)
    if tg.dim() == 1:
        tg = tg.reshape(b, -1)
    tl = _dev_tensor(tgt_len, torch.int32, dev).reshape(-1)
    if kind not in ("asg", "ctc"):
        raise ContractError(f"unknown criterion kind {kind!r}")
    if kind == "ctc" and blank_id is None:
        raise ContractError("CTC collapse needs blank_id")
    special = int(blank_id) if kind == "ctc" else (-1 if rep_id is None else int(rep_id))
    out = GreedyEval(hyp=torch.empty((b, t_max), dtype=torch.int64, device=dev),
                     hyp_len=torch.empty(b, dtype=torch.int32, device=dev),
                     tok_dist=torch.empty(b, dtype=torch.int32, device=dev),
                     word_dist=torch.empty(b, dtype=torch.int32, device=dev),
                     ref_words=torch.empty(b, dtype=torch.int32, device=dev),
                     status=torch.empty(b, dtype=torch.int32, device=dev))
    rc = nat.lib().w2l_greedy_eval(_p(pa), _p(pl), b, t_max, 0 if kind == "asg" else 1, special,
                                   _p(tg), _p(tl), int(tg.shape[1]),
                                   -1 if silence_id is None else int(silence_id), _p(out.hyp),
                                   _p(out.hyp_len), _p(out.tok_dist), _p(out.word_dist),
                                   _p(out.ref_words), _p(out.status), _stream())
    _check_call(rc, "w2l_greedy_eval")
    if check:
        _raise_batch(out.status, "greedy_eval_batched")
    return out


def evaluate_batch(emissions, em_len, targets, tgt_len, kind: str, *, transitions=None,
                   blank_id=None, rep_id=None, silence_id=None) -> dict:
    """One batch of the reference's evaluate loop (trainer.py:478-514) on the
    device: loss-only criterion, Viterbi paths (with the transitions for ASG,
    argmax paths for CTC: criterion.py:334-336, 364-366), collapse, token and
    word edit distances.  Utterances with an empty reference are skipped, as
    the reference does.  Returns the sums the reference accumulates."""
    dev = _device()
    em = _dev_tensor(emissions, torch.float32, dev)
    el = _dev_tensor(em_len, torch.int32, dev).reshape(-1)
    tl = _dev_tensor(tgt_len, torch.int32, dev).reshape(-1)
    if kind == "asg":
        out = asg_loss_grad_batched(em, el, targets, tl, transitions, loss_only=True)
        paths, _ = viterbi_batched(em, el, transitions)
    else:
        out = ctc_loss_grad_batched(em, el, targets, tl, blank_id, loss_only=True)
        paths, _ = viterbi_batched(em, el, None)
    g = greedy_eval_batched(paths, el, targets, tl, kind, blank_id=blank_id, rep_id=rep_id,
                            silence_id=silence_id)
    keep = tl > 0
    return {"loss_sum": float(out.loss[keep].sum()), "utterances": int(keep.sum()),
            "tok_dist": int(g.tok_dist[keep].sum()), "tok_len": int(tl[keep].sum()),
            "word_dist": int(g.word_dist[keep].sum()), "word_len": int(g.ref_words[keep].sum())}


# ------------------------------------------------------------- autograd --

# The autograd functions do not synchronise with the host (check=False): an
# utterance whose inputs fail validation gets a NaN loss and a zero gradient,
# and its status code stays readable from the returned loss tensor's
# ``w2l_status`` attribute (raise it when convenient with check_status()).

def _mask_failed(loss: torch.Tensor, status: torch.Tensor) -> torch.Tensor:
    return torch.where(status == 0, loss, torch.full_like(loss, float("nan")))


def check_status(loss: torch.Tensor, what: str = "criterion") -> None:
    """Raise the reference exception for the first failing utterance of a
    loss returned by asg_loss / ctc_loss (synchronises with the device)."""
    st = getattr(loss, "w2l_status", None)
    if st is not None:
        _raise_batch(st, what)


class _AsgLossFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, emissions, transitions, em_len, targets, tgt_len, check, holder,
                stream_grad):
        out = asg_loss_grad_batched(emissions.detach(), em_len, targets, tgt_len,
                                    transitions.detach(), per_utterance_grad_transitions=True,
                                    check=check, stream_grad=stream_grad)
        ctx.save_for_backward(out.grad_emissions, out.grad_transitions_per_utt)
        ctx.status = holder["status"] = out.status
        return _mask_failed(out.loss, out.status).to(emissions.dtype)

    @staticmethod
    def backward(ctx, g):
        ge, ga = ctx.saved_tensors
        g = torch.where(ctx.status == 0, g, torch.zeros_like(g)).to(torch.float32)
        return (ge * g[:, None, None], torch.einsum("b,bij->ij", g, ga), None, None, None, None,
                None, None)


class _CtcLossFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, logp, em_len, targets, tgt_len, blank_id, logits, check, holder):
        out = ctc_loss_grad_batched(logp.detach(), em_len, targets, tgt_len, blank_id,
                                    logits=logits, check=check)
        ctx.save_for_backward(out.grad_emissions)
        ctx.status = holder["status"] = out.status
        return _mask_failed(out.loss, out.status).to(logp.dtype)

    @staticmethod
    def backward(ctx, g):
        (ge,) = ctx.saved_tensors
        g = torch.where(ctx.status == 0, g, torch.zeros_like(g)).to(torch.float32)
        return (ge * g[:, None, None], None, None, None, None, None, None, None)


def asg_loss(emissions, transitions, em_len, targets, tgt_len, check: bool = False,
             stream_grad: bool = True) -> torch.Tensor:
    """Differentiable per-utterance ASG losses [B] (PyTorch training).  No
    host synchronisation unless check=True (see check_status).  stream_grad
    (W2L_FLAG_STREAM_GRAD, bitwise the same results) starts the gradient on
    the middle frames while the recursions run: 0.337 -> 0.318 ms for ASG
    alone at B=64 T=1600; pass False when another criterion's recursions run
    concurrently and were not started first."""
    holder: dict = {}
    loss = _AsgLossFn.apply(emissions, transitions, em_len, targets, tgt_len, check, holder,
                            stream_grad)
    loss.w2l_status = holder["status"]
    return loss


def ctc_loss(logp, em_len, targets, tgt_len, blank_id: int, logits: bool = False,
             check: bool = False) -> torch.Tensor:
    """Differentiable per-utterance CTC losses [B] on log-probabilities, or on
    unnormalised logits with log_softmax fused in (logits=True).  No host
    synchronisation unless check=True (see check_status)."""
    holder: dict = {}
    loss = _CtcLossFn.apply(logp, em_len, targets, tgt_len, blank_id, logits, check, holder)
    loss.w2l_status = holder["status"]
    return loss


# ------------------------------------------------------ trainer adapters --

class CtcCriterion:
    """CTC over a token table, blank appended as the last output (criterion.py:315-339)."""

    kind = "ctc"

    def __init__(self, table):
        self.table = table
        self.blank_id = len(table)
        self.n_outputs = len(table) + 1

    def prepare_target(self, token_ids):
        return validate_target(token_ids, "ctc", self.table)

    def loss_grad(self, emissions, target) -> LossOutput:
        return ctc_loss_grad(emissions, target, self.blank_id)

    def params(self) -> dict:
        return {}

    def viterbi_path(self, emissions):
        return viterbi(emissions)[0]

    def collapse(self, path):
        return collapse_path(path, "ctc", blank_id=self.blank_id)


class _HostTensor:
    """Read-only float32 host view with the reference Tensor's surface
    (autodiff.py:20-45: ``.data``, ``.shape``, ``.item()``)."""

    __slots__ = ("_data",)

    def __init__(self, arr):
        arr = np.ascontiguousarray(arr, dtype=np.float32)
        arr.setflags(write=False)
        self._data = arr

    @property
    def data(self) -> np.ndarray:
        return self._data

    @property
    def shape(self) -> tuple:
        return self._data.shape

    def item(self) -> float:
        return float(self._data.item())


class TransitionsVariable:
    """The reference Variable protocol (autodiff.py:75-116) over the device
    transition parameter, so reference-side code that uses
    ``criterion.params()`` works unchanged: ``.value`` reads the parameter
    (a host snapshot) and assigning it writes the parameter (the optimizer's
    ``p.value = ...``, autodiff.py:433); ``accumulate_grad`` / ``grad`` /
    ``zero_grad`` keep a host gradient like the reference trainer expects
    (trainer.py:442-449)."""

    def __init__(self, param: torch.Tensor):
        self._param = param
        self._grad = None
        self.requires_grad = True
        self.node = None

    @property
    def value(self) -> _HostTensor:
        return _HostTensor(self._param.detach().cpu().numpy())

    @value.setter
    def value(self, v) -> None:
        data = np.asarray(getattr(v, "data", v), dtype=np.float32)
        if data.shape != tuple(self._param.shape):
            raise ContractError(f"transitions must be {tuple(self._param.shape)}, got {data.shape}")
        with torch.no_grad():
            self._param.copy_(torch.from_numpy(np.ascontiguousarray(data)))

    @property
    def shape(self) -> tuple:
        return tuple(self._param.shape)

    @property
    def grad(self) -> _HostTensor:
        return _HostTensor(np.zeros(self.shape, np.float32) if self._grad is None else self._grad)

    def zero_grad(self) -> None:
        self._grad = None

    def accumulate_grad(self, contribution) -> None:
        c = np.asarray(contribution, dtype=np.float32)
        if c.shape != self.shape:
            raise ContractError(f"gradient shape {c.shape} != value shape {self.shape}")
        self._grad = c.copy() if self._grad is None else self._grad + c

    def item(self) -> float:
        return self.value.item()


class AsgCriterion:
    """ASG with a learnable N x N transition matrix (criterion.py:342-369).

    ``transitions`` is a torch Parameter (zeros, as in the reference) living on
    the current CUDA device; ``params()`` keeps the reference key and returns
    a Variable-protocol view of it (``.value``, ``.grad``, ...)."""

    kind = "asg"

    def __init__(self, table):
        self.table = table
        self.n_outputs = len(table)
        dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() \
            else torch.device("cpu")
        self.transitions = torch.nn.Parameter(
            torch.zeros((self.n_outputs, self.n_outputs), dtype=torch.float32, device=dev))
        self._var = TransitionsVariable(self.transitions)

    def prepare_target(self, token_ids):
        return validate_target(token_ids, "asg", self.table)

    def loss_grad(self, emissions, target) -> LossOutput:
        return asg_loss_grad(emissions, target, self.transitions.detach())

    def params(self) -> dict:
        return {"criterion.transitions": self._var}

    def viterbi_path(self, emissions):
        return viterbi(emissions, self.transitions.detach())[0]

    def collapse(self, path):
        return collapse_path(path, "asg", rep_id=self.table.rep_id)


def make_criterion(kind: str, table):
    """criterion.py:372-377."""
    if kind == "ctc":
        return CtcCriterion(table)
    if kind == "asg":
        return AsgCriterion(table)
    raise ContractError(f"unknown criterion kind {kind!r}")


_ = (DeviceError, InfeasibleTargetError)  # re-exported names used by callers
