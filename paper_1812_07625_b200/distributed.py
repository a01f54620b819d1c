"""Data-parallel plumbing for the criterion path (one process per GPU).

The reference trains data-parallel in one process: the batch is split into
K contiguous shards (``np.array_split(np.arange(B), K)``, trainer.py:433),
every shard's transition gradient is summed per utterance
(trainer.py:417-418), the shard sums are added and divided by the batch size
(trainer.py:442-447).  Here each rank owns one contiguous shard on its own
GPU; utterances are independent, so the only exchange is ONE all-reduce
(sum) of the N x N transition gradient (3.6 KB at N = 30) over
NCCL/NVLink, enqueued on the compute stream right after the ASG kernels.
CTC has no parameters and needs no exchange.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.distributed as dist


def shard_bounds(batch_size: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of rank's contiguous shard, identical to
    np.array_split(np.arange(batch_size), world)[rank] (trainer.py:433)."""
    base, extra = divmod(batch_size, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


class NcclComm:
    """The library's own NCCL communicator (C-ABI w2l_comm_*,
    include/w2l_criterion.h): the transition-gradient all-reduce is enqueued
    by ``w2l_allreduce_grad_A`` on the compute stream, the same entry a
    non-Python host uses.  The 128-byte unique id travels over the default
    torch.distributed group (any channel would do)."""

    def __init__(self, group=None):
        from . import _native as nat
        self._nat = nat
        lib = nat.lib()
        if not lib.w2l_comm_available():
            raise nat.NativeLibraryError("libnccl.so.2 could not be loaded")
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        uid = ctypes.create_string_buffer(128)
        if rank == 0:
            self._check(lib.w2l_comm_unique_id(uid), "w2l_comm_unique_id")
        if world > 1:
            box = [bytes(uid.raw)]
            dist.broadcast_object_list(box, src=0, group=group)
            uid = ctypes.create_string_buffer(box[0], 128)
        self._comm = ctypes.c_void_p()
        self._check(lib.w2l_comm_init(uid, world, rank, ctypes.byref(self._comm)), "w2l_comm_init")
        self.world, self.rank = world, rank

    def _check(self, rc, what):
        if rc != self._nat.OK:
            from .errors import raise_for_status
            raise_for_status(rc, f"{what} failed ({self._nat.lib().w2l_status_string(rc).decode()})")

    def allreduce_grad_transitions(self, grad: torch.Tensor) -> torch.Tensor:
        if not (grad.is_cuda and grad.dtype == torch.float32 and grad.is_contiguous()):
            raise ValueError("grad_transitions must be a contiguous CUDA f32 tensor")
        stream = ctypes.c_void_p(torch.cuda.current_stream(grad.device).cuda_stream)
        self._check(self._nat.lib().w2l_allreduce_grad_A(grad.data_ptr(), grad.shape[0],
                                                         self._comm, stream),
                    "w2l_allreduce_grad_A")
        return grad

    def close(self):
        if self._comm:
            self._nat.lib().w2l_comm_destroy(self._comm)
            self._comm = ctypes.c_void_p()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def allreduce_grad_transitions(grad: torch.Tensor, group=None) -> torch.Tensor:
    """In-place sum of the per-rank transition-gradient sums (the exchange
    trainer.py:442-446 performs across shards).  The caller divides by the
    global batch size (trainer.py:447)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=group)
    return grad


def sgd_step_transitions(transitions: torch.Tensor, velocity: torch.Tensor,
                         grad_sum: torch.Tensor, batch_size: int, lr: float,
                         momentum: float) -> None:
    """The step after the all-reduce (trainer.py:442-449 with the
    optimizer of autodiff.py:429-433): g = grad_sum / B, v = momentum v + g,
    A -= lr v, in one device kernel with the reference's float32 rounding.
    transitions and velocity are updated in place."""
    from . import _native as nat
    from .criterion import _check_call, _stream
    for t in (transitions, velocity, grad_sum):
        if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
            raise ValueError("transitions, velocity and grad_sum must be contiguous CUDA f32")
    n = transitions.shape[0]
    rc = nat.lib().w2l_transitions_sgd_step(transitions.data_ptr(), velocity.data_ptr(),
                                            grad_sum.data_ptr(), n, int(batch_size),
                                            float(lr), float(momentum), _stream())
    _check_call(rc, "w2l_transitions_sgd_step")


def allreduce_loss_sum(loss: torch.Tensor, group=None) -> torch.Tensor:
    """Sum of per-utterance losses over all ranks (trainer.py:452 loss_sum)."""
    total = loss.sum().to(torch.float64).reshape(1)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(total, op=dist.ReduceOp.SUM, group=group)
    return total


def sharded_asg_step(emissions, em_len, targets, tgt_len, transitions, loss_grad_fn, *,
                     world: int, rank: int, group=None):
    """One data-parallel ASG step on this rank's shard of a global batch.

    ``loss_grad_fn(em, em_len, targets, tgt_len, transitions)`` computes the
    shard's per-utterance losses and the transition gradient summed over the
    shard (on the GPU: ``criterion.asg_loss_grad_batched``).  Returns
    (shard losses, global grad_A / B_global, global loss sum), matching the
    reference's single-process union-batch result."""
    b_global = len(em_len)
    lo, hi = shard_bounds(b_global, world, rank)
    loss, grad_a = loss_grad_fn(emissions[lo:hi], em_len[lo:hi], targets[lo:hi],
                                tgt_len[lo:hi], transitions)
    grad_a = allreduce_grad_transitions(grad_a, group)
    total = allreduce_loss_sum(loss, group)
    return loss, grad_a / b_global, total


def as_numpy(x):
    return x.detach().cpu().numpy() if isinstance(x, torch.Tensor) else np.asarray(x)
