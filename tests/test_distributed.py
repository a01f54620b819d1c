"""Data-parallel semantics of the transition-gradient exchange on CPU (gloo,
world size 2), shaped after the reference's worker-equivalence tests
(test_trainer.py:224-242, test_acceptance.py:411-421): sharded gradients
must reproduce the union-batch gradient.  The per-shard math comes from the
CPU oracle here (test infrastructure); on the GPU the same helper runs the
CUDA kernels (tests/test_gpu_parity.py, bench.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import criterion_oracle as orc
from paper_1812_07625_b200.distributed import sharded_asg_step, shard_bounds


def test_shard_bounds_match_array_split():
    for b in (1, 5, 6, 8, 64, 513):
        for w in (1, 2, 3, 4, 8):
            want = np.array_split(np.arange(b), w)
            for r in range(w):
                lo, hi = shard_bounds(b, w, r)
                assert list(range(lo, hi)) == want[r].tolist()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_shard(em, el, tg, tl, a):
    loss, _, ga = orc.asg_batch(em, el, tg, tl, a)
    return torch.from_numpy(loss), torch.from_numpy(ga.astype(np.float32))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        em, el, tg, tl, a = orc.synth_asg(11, 6, 9, 4, 3)
        loss, ga, total = sharded_asg_step(em, el, tg, tl, a, _oracle_shard,
                                           world=world, rank=rank)
        q.put((rank, ga.numpy(), float(total.item()), loss.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_grad_matches_union_batch(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    em, el, tg, tl, a = orc.synth_asg(11, 6, 9, 4, 3)
    loss, _, ga = orc.asg_batch(em, el, tg, tl, a)
    want = ga.astype(np.float64) / len(el)
    for rank, got, total, shard_loss in out:
        assert orc.rel_err(got, want) < 1e-5            # WORKER_REL (test_acceptance.py:54)
        assert total == pytest.approx(loss.sum(), rel=1e-6)
        lo, hi = shard_bounds(len(el), world, rank)
        np.testing.assert_allclose(shard_loss, loss[lo:hi], rtol=1e-12)


# ------------------------------------------------ the CUDA path, sharded --

def _gpu_shard(em, el, tg, tl, a):
    from paper_1812_07625_b200 import criterion as C
    out = C.asg_loss_grad_batched(torch.from_numpy(np.ascontiguousarray(em)).cuda(), el, tg, tl,
                                  a)
    return out.loss, out.grad_transitions


def _gpu_worker(rank, world, port, q, b_sz):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)      # both ranks share the one GPU; gloo carries CUDA tensors
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        em, el, tg, tl, a = orc.synth_asg(12, b_sz, 300, 30, 60, ragged=True)
        loss, ga, total = sharded_asg_step(em, el, tg, tl, a, _gpu_shard, world=world,
                                           rank=rank)
        q.put((rank, ga.cpu().numpy(), float(total.item()), loss.cpu().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("b_sz", [6, 1])      # b_sz=1: rank 1's shard is empty
def test_cuda_sharded_grad_matches_union_batch(b_sz):
    # test_trainer.py:224-242 on the CUDA criterion: 2 ranks (gloo, CUDA
    # tensors) each run asg_loss_grad_batched on a contiguous shard; the
    # all-reduced grad_A / B must equal the union batch's within WORKER_REL
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, q, b_sz))
             for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    em, el, tg, tl, a = orc.synth_asg(12, b_sz, 300, 30, 60, ragged=True)
    loss, _, ga = orc.asg_batch(em, el, tg, tl, a)
    union = _gpu_shard(em, el, tg, tl, a)
    want = ga.astype(np.float64) / b_sz
    for rank, got, total, shard_loss in out:
        assert orc.rel_err(got, want) < 1e-4                      # vs the oracle (fp32 path)
        assert orc.rel_err(got, union[1].cpu().numpy() / b_sz) < 1e-5   # WORKER_REL
        assert total == pytest.approx(loss.sum(), rel=1e-6)
        lo, hi = shard_bounds(b_sz, world, rank)
        np.testing.assert_allclose(shard_loss, loss[lo:hi], rtol=1e-4)
