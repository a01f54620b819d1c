"""Where the e2e step time goes: bench.py's e2e loop with parts removed.
Modes: copies only, compute only (device-resident inputs, same stream
structure), full, and full with the input copies issued on a high-priority
stream."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1812_07625_b200 import _native, criterion as C  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    em, em_len, asg_t, ctc_t, tgt_len, trans, blank = bench.make_inputs(0)
    B, T, N = em.shape
    lib = _native.lib()
    A_d = torch.from_numpy(trans).to(dev)
    ws_a = torch.empty(lib.w2l_asg_workspace_bytes(B, T, N, bench.L_LAB), dtype=torch.uint8,
                       device=dev)
    ws_c = torch.empty(lib.w2l_ctc_workspace_bytes(B, T, N, bench.L_LAB), dtype=torch.uint8,
                       device=dev)
    host = dict(em=torch.from_numpy(em).pin_memory(), ta=torch.from_numpy(asg_t).pin_memory(),
                tc=torch.from_numpy(ctc_t).pin_memory(), el=torch.from_numpy(em_len).pin_memory(),
                tl=torch.from_numpy(tgt_len).pin_memory())
    NB = 3
    bufs = [{k: v.to(dev) for k, v in host.items()} for _ in range(NB)]
    spare = {k: v.to(dev) for k, v in host.items()}
    main_s = torch.cuda.current_stream(dev)
    side = torch.cuda.Stream(device=dev)
    loss_h = torch.empty(B, dtype=torch.float64).pin_memory()
    outs = [(C.asg_loss_grad_batched(b["em"], b["el"], b["ta"], b["tl"], A_d, check=False,
                                     workspace=ws_a),
             C.ctc_loss_grad_batched(b["em"], b["el"], b["tc"], b["tl"], blank, check=False,
                                     workspace=ws_c)) for b in bufs[:2]]

    def both(bi, o):
        side.wait_stream(main_s)
        with torch.cuda.stream(side):
            C.ctc_loss_grad_batched(bi["em"], bi["el"], bi["tc"], bi["tl"], blank, check=False,
                                    workspace=ws_c, out=o[1])
        C.asg_loss_grad_batched(bi["em"], bi["el"], bi["ta"], bi["tl"], A_d, check=False,
                                workspace=ws_a, out=o[0])
        main_s.wait_stream(side)

    def run(mode, steps=30, prio=0):
        copy_s = torch.cuda.Stream(device=dev, priority=prio)
        copied = [torch.cuda.Event() for _ in range(NB)]
        consumed = [torch.cuda.Event() for _ in range(NB)]
        nb = 3 if mode == "triple" else 2

        def issue_copy(i):
            bi = bufs[i % nb]
            with torch.cuda.stream(copy_s):
                if i >= nb:
                    copy_s.wait_event(consumed[i % nb])
                for k in host:
                    bi[k].copy_(host[k], non_blocking=True)
                copied[i % nb].record(copy_s)

        def step(i):
            bi = bufs[i & 1]
            if mode in ("triple", "ahead"):
                # the copy for step i was issued earlier (before step i-1's
                # compute for "ahead": prefetch distance 1, issue order swapped)
                bi = bufs[i % nb]
                if i == 0:
                    issue_copy(0)
                main_s.wait_event(copied[i % nb])
                both(bi, outs[i & 1])
                consumed[i % nb].record(main_s)
                loss_h.copy_(outs[i & 1][0].loss, non_blocking=True)
                issue_copy(i + 1)
                return
            if mode == "nodeps":
                # physical overlap only: copies into a third buffer, no events
                with torch.cuda.stream(copy_s):
                    for k in host:
                        spare[k].copy_(host[k], non_blocking=True)
                both(bi, outs[i & 1])
                return
            if mode in ("copies", "full"):
                with torch.cuda.stream(copy_s):
                    if i >= 2:
                        copy_s.wait_event(consumed[i & 1])
                    for k in host:
                        bi[k].copy_(host[k], non_blocking=True)
                    copied[i & 1].record(copy_s)
                main_s.wait_event(copied[i & 1])
            if mode in ("compute", "full"):
                both(bi, outs[i & 1])
            consumed[i & 1].record(main_s)
            if mode in ("compute", "full"):
                loss_h.copy_(outs[i & 1][0].loss, non_blocking=True)

        for i in range(5):
            step(i)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main_s)
        copy_s.wait_stream(main_s)
        for i in range(steps):
            step(i)
        e1.record(main_s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps

    lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") \
        else (0, -1)
    for mode, prio in (("compute", 0), ("full", 0), ("ahead", 0), ("triple", 0),
                       ("full", 0), ("ahead", 0), ("triple", 0)):
        print(f"{mode:8s} prio={prio:3d}: {run(mode, prio=prio):.4f} ms/step")


if __name__ == "__main__":
    main()
