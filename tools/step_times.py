"""Per-step device times of bench.py's two-stream step (same inputs, flush and
stream setup), to see whether a mean hides a bimodal distribution.
usage: python tools/step_times.py [asg_delay_cycles] [steps]"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1812_07625_b200 import criterion as C  # noqa: E402

delay = int(sys.argv[1]) if len(sys.argv) > 1 else 0
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
em, el, ta, tc, tl, A, blank = bench.make_inputs(0)
d = torch.from_numpy(em).cuda()
el_d, ta_d, tc_d, tl_d, A_d = (torch.from_numpy(x).cuda() for x in (el, ta, tc, tl, A))
main = torch.cuda.current_stream()
side = torch.cuda.Stream()
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
oa = C.asg_loss_grad_batched(d, el_d, ta_d, tl_d, A_d, check=False)
oc = C.ctc_loss_grad_batched(d, el_d, tc_d, tl_d, blank, check=False)


def step():
    side.wait_stream(main)
    with torch.cuda.stream(side):
        C.ctc_loss_grad_batched(d, el_d, tc_d, tl_d, blank, check=False, out=oc)
    if delay:
        torch.cuda._sleep(delay)
    C.asg_loss_grad_batched(d, el_d, ta_d, tl_d, A_d, check=False, out=oa)
    main.wait_stream(side)


for _ in range(5):
    step()
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
for s, e in ev:
    flush.zero_()
    s.record()
    step()
    e.record()
torch.cuda.synchronize()
t = np.array([s.elapsed_time(e) for s, e in ev])
print(f"delay {delay}: mean {t.mean():.4f} median {np.median(t):.4f} min {t.min():.4f} max {t.max():.4f} ms;"
      f" sorted: " + " ".join(f"{x:.3f}" for x in np.sort(t)))
