"""Two-stream timeline of one bench step (ASG on the main stream, CTC on a
side stream), split into the chain and gradient phases with events between
them.  Prints each phase's start/end relative to the step start (ms), the
median over several steps.  Usage: python tools/timeline.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1812_07625_b200 import _native, criterion as C  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    em, em_len, asg_t, ctc_t, tgt_len, trans, blank = bench.make_inputs(0)
    B, T, N = em.shape
    em_d = torch.from_numpy(em).to(dev)
    el_d = torch.from_numpy(em_len).to(dev)
    ta_d = torch.from_numpy(asg_t).to(dev)
    tc_d = torch.from_numpy(ctc_t).to(dev)
    tl_d = torch.from_numpy(tgt_len).to(dev)
    A_d = torch.from_numpy(trans).to(dev)
    lib = _native.lib()
    ws_a = torch.empty(lib.w2l_asg_workspace_bytes(B, T, N, bench.L_LAB), dtype=torch.uint8,
                       device=dev)
    ws_c = torch.empty(lib.w2l_ctc_workspace_bytes(B, T, N, bench.L_LAB), dtype=torch.uint8,
                       device=dev)
    oa = C.asg_loss_grad_batched(em_d, el_d, ta_d, tl_d, A_d, check=True, workspace=ws_a)
    oc = C.ctc_loss_grad_batched(em_d, el_d, tc_d, tl_d, blank, check=True, workspace=ws_c)
    side = torch.cuda.Stream(device=dev)
    main_s = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def step(split, rec):
        t0 = ev()
        t0.record(main_s)
        side.wait_stream(main_s)
        marks = {}
        with torch.cuda.stream(side):
            if split:
                C.ctc_loss_grad_batched(em_d, el_d, tc_d, tl_d, blank, check=False,
                                        workspace=ws_c, out=oc, phase="chain")
                marks["ctc_chain"] = ev()
                marks["ctc_chain"].record(side)
                C.ctc_loss_grad_batched(em_d, el_d, tc_d, tl_d, blank, check=False,
                                        workspace=ws_c, out=oc, phase="grad")
            else:
                C.ctc_loss_grad_batched(em_d, el_d, tc_d, tl_d, blank, check=False,
                                        workspace=ws_c, out=oc)
            marks["ctc_end"] = ev()
            marks["ctc_end"].record(side)
        if split:
            C.asg_loss_grad_batched(em_d, el_d, ta_d, tl_d, A_d, check=False, workspace=ws_a,
                                    out=oa, phase="chain")
            marks["asg_chain"] = ev()
            marks["asg_chain"].record(main_s)
            C.asg_loss_grad_batched(em_d, el_d, ta_d, tl_d, A_d, check=False, workspace=ws_a,
                                    out=oa, phase="grad")
        else:
            C.asg_loss_grad_batched(em_d, el_d, ta_d, tl_d, A_d, check=False, workspace=ws_a,
                                    out=oa)
        marks["asg_end"] = ev()
        marks["asg_end"].record(main_s)
        main_s.wait_stream(side)
        t1 = ev()
        t1.record(main_s)
        rec.append((t0, marks, t1))

    def stagger(rec):
        # ASG chain first; the CTC chain then overlaps the ASG gradient phase
        t0 = ev()
        t0.record(main_s)
        marks = {}
        C.asg_loss_grad_batched(em_d, el_d, ta_d, tl_d, A_d, check=False, workspace=ws_a,
                                out=oa, phase="chain")
        marks["asg_chain"] = ev()
        marks["asg_chain"].record(main_s)
        side.wait_stream(main_s)
        with torch.cuda.stream(side):
            C.ctc_loss_grad_batched(em_d, el_d, tc_d, tl_d, blank, check=False,
                                    workspace=ws_c, out=oc, phase="chain")
            marks["ctc_chain"] = ev()
            marks["ctc_chain"].record(side)
            C.ctc_loss_grad_batched(em_d, el_d, tc_d, tl_d, blank, check=False,
                                    workspace=ws_c, out=oc, phase="grad")
            marks["ctc_end"] = ev()
            marks["ctc_end"].record(side)
        C.asg_loss_grad_batched(em_d, el_d, ta_d, tl_d, A_d, check=False, workspace=ws_a,
                                out=oa, phase="grad")
        marks["asg_end"] = ev()
        marks["asg_end"].record(main_s)
        main_s.wait_stream(side)
        t1 = ev()
        t1.record(main_s)
        rec.append((t0, marks, t1))

    hi_s = torch.cuda.Stream(device=dev, priority=-5)   # clamped to the device's range

    def prio(rec, asg_hi=True):
        # ASG (the tail of the step) on a high-priority stream, CTC on a
        # normal one (asg_hi=False: the other way round)
        t0 = ev()
        t0.record(main_s)
        a_s, c_s = (hi_s, side) if asg_hi else (side, hi_s)
        a_s.wait_stream(main_s)
        c_s.wait_stream(main_s)
        marks = {}
        with torch.cuda.stream(c_s):
            C.ctc_loss_grad_batched(em_d, el_d, tc_d, tl_d, blank, check=False,
                                    workspace=ws_c, out=oc)
            marks["ctc_end"] = ev()
            marks["ctc_end"].record(c_s)
        with torch.cuda.stream(a_s):
            C.asg_loss_grad_batched(em_d, el_d, ta_d, tl_d, A_d, check=False, workspace=ws_a,
                                    out=oa)
            marks["asg_end"] = ev()
            marks["asg_end"].record(a_s)
        main_s.wait_stream(a_s)
        main_s.wait_stream(c_s)
        t1 = ev()
        t1.record(main_s)
        rec.append((t0, marks, t1))

    for split in (False, True, "stagger", "asg_hi", "ctc_hi", False):
        recs = []
        for i in range(25):
            flush.zero_()
            if split == "stagger":
                stagger(recs if i >= 5 else [])
            elif split in ("asg_hi", "ctc_hi"):
                prio(recs if i >= 5 else [], split == "asg_hi")
            else:
                step(split, recs if i >= 5 else [])
        torch.cuda.synchronize()
        rows = {}
        for t0, marks, t1 in recs:
            for k, e in marks.items():
                rows.setdefault(k, []).append(t0.elapsed_time(e))
            rows.setdefault("step", []).append(t0.elapsed_time(t1))
        print({False: "whole", True: "split", "stagger": "stagger", "asg_hi": "asg_hi",
               "ctc_hi": "ctc_hi"}[split], {k: round(float(np.median(v)), 4)
                                             for k, v in rows.items()})
    # each criterion alone
    for name, fn in (("asg_alone", lambda: C.asg_loss_grad_batched(
            em_d, el_d, ta_d, tl_d, A_d, check=False, workspace=ws_a, out=oa)),
                     ("ctc_alone", lambda: C.ctc_loss_grad_batched(
            em_d, el_d, tc_d, tl_d, blank, check=False, workspace=ws_c, out=oc))):
        ts = []
        for i in range(25):
            flush.zero_()
            a, b = ev(), ev()
            a.record()
            fn()
            b.record()
            if i >= 5:
                ts.append((a, b))
        torch.cuda.synchronize()
        print(name, round(float(np.median([a.elapsed_time(b) for a, b in ts])), 4))


if __name__ == "__main__":
    main()
