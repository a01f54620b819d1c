"""Per-step times inside bench.py's e2e loop (pinned H2D copies on a copy
stream, the two-criteria step, loss read-back), stagger on or off:
    python tools/e2e_steps.py [stagger 0|1] [steps]"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1812_07625_b200 import criterion as C  # noqa: E402

stagger = (sys.argv[1] != "0") if len(sys.argv) > 1 else True
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
em, el, ta, tc, tl, A, blank = bench.make_inputs(0)
dev = torch.device("cuda")
main = torch.cuda.current_stream()
side, copy_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
host = {k: torch.from_numpy(v).pin_memory() for k, v in dict(em=em, ta=ta, tc=tc, el=el, tl=tl).items()}
bufs = [{k: torch.empty_like(v, device=dev) for k, v in host.items()} for _ in range(2)]
A_d = torch.from_numpy(A).to(dev)
x0 = bufs[0]
for k in host:
    x0[k].copy_(host[k])
outs = [(C.asg_loss_grad_batched(x0["em"], x0["el"], x0["ta"], x0["tl"], A_d, check=False),
         C.ctc_loss_grad_batched(x0["em"], x0["el"], x0["tc"], x0["tl"], blank, check=False))
        for _ in range(2)]
loss_h = torch.empty(len(em), dtype=torch.float64).pin_memory()
copied = [torch.cuda.Event() for _ in range(2)]
consumed = [torch.cuda.Event() for _ in range(2)]
read_back = [torch.cuda.Event() for _ in range(2)]
validated = torch.cuda.Event()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]


def step(i, rec):
    bi = bufs[i & 1]
    oa_, oc_ = outs[i & 1]
    with torch.cuda.stream(copy_s):
        if i >= 2:
            copy_s.wait_event(consumed[i & 1])
        for k in host:
            bi[k].copy_(host[k], non_blocking=True)
        copied[i & 1].record(copy_s)
    main.wait_event(copied[i & 1])
    if i >= 2:
        main.wait_event(read_back[i & 1])
    if rec:
        ev[i][0].record(main)
    side.wait_stream(main)
    with torch.cuda.stream(side):
        if stagger:
            C.ctc_loss_grad_batched(bi["em"], bi["el"], bi["tc"], bi["tl"], blank, check=False,
                                    out=oc_, phase="validate")
            validated.record(side)
            C.ctc_loss_grad_batched(bi["em"], bi["el"], bi["tc"], bi["tl"], blank, check=False,
                                    out=oc_, phase="rest")
        else:
            C.ctc_loss_grad_batched(bi["em"], bi["el"], bi["tc"], bi["tl"], blank, check=False,
                                    out=oc_)
    if stagger:
        main.wait_event(validated)
    C.asg_loss_grad_batched(bi["em"], bi["el"], bi["ta"], bi["tl"], A_d, check=False, out=oa_)
    main.wait_stream(side)
    if rec:
        ev[i][1].record(main)
    consumed[i & 1].record(main)
    with torch.cuda.stream(d2h_s):
        d2h_s.wait_event(consumed[i & 1])
        loss_h.copy_(oa_.loss, non_blocking=True)
        read_back[i & 1].record(d2h_s)


for i in range(5):
    step(i, False)
torch.cuda.synchronize()
t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0.record()
for i in range(steps):
    step(i, True)
main.wait_stream(d2h_s)
t1.record()
torch.cuda.synchronize()
t = np.array([a.elapsed_time(b) for a, b in ev])
gaps = np.array([ev[i - 1][1].elapsed_time(ev[i][0]) for i in range(1, steps)])
print(f"stagger {int(stagger)}: total {t0.elapsed_time(t1) / steps:.4f} ms/step; step mean {t.mean():.4f}"
      f" median {np.median(t):.4f}; gap between steps mean {gaps.mean():.4f}; sorted steps: "
      + " ".join(f"{x:.3f}" for x in np.sort(t)))
