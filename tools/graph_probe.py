"""Two-stream bench step (ASG + CTC) launched eagerly vs replayed from a CUDA
graph captured once (the same kernels; the graph removes launch gaps)."""
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
    ref_loss = (oa.loss.clone(), oc.loss.clone(), oa.grad_emissions.clone())
    side = torch.cuda.Stream(device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    def both():
        cur = torch.cuda.current_stream(dev)
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            C.ctc_loss_grad_batched(em_d, el_d, tc_d, tl_d, blank, check=False, workspace=ws_c,
                                    out=oc)
        C.asg_loss_grad_batched(em_d, el_d, ta_d, tl_d, A_d, check=False, workspace=ws_a,
                                out=oa)
        cur.wait_stream(side)

    cap = torch.cuda.Stream(device=dev)
    cap.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(cap):
        for _ in range(3):
            both()
    torch.cuda.current_stream(dev).wait_stream(cap)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        both()
    torch.cuda.synchronize()

    def timed(fn, n=30):
        ts = []
        for i in range(n + 5):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            if i >= 5:
                ts.append((a, b))
        torch.cuda.synchronize()
        return float(np.median([a.elapsed_time(b) for a, b in ts]))

    for _ in range(2):
        print(f"eager {timed(both):.4f} ms/step   graph {timed(g.replay):.4f} ms/step")
    same = (torch.equal(oa.loss, ref_loss[0]) and torch.equal(oc.loss, ref_loss[1])
            and torch.equal(oa.grad_emissions, ref_loss[2]))
    print("graph outputs identical to the eager call:", same)


if __name__ == "__main__":
    main()
