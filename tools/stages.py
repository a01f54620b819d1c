"""Per-stage device times (traced calls) of one ASG and one CTC batched call at the bench shape."""
import sys, torch
sys.path.insert(0, ".")
import bench
from paper_1812_07625_b200 import criterion as C
em, el, ta, tc, tl, A, blank = bench.make_inputs(0)
d = torch.from_numpy(em).cuda()
for _ in range(3):
    oc = C.ctc_loss_grad_batched(d, el, tc, tl, blank, check=False, trace=True)
    oa = C.asg_loss_grad_batched(d, el, ta, tl, A, check=False, trace=True)
print("CTC", {k: round(v*1000) for k, v in oc.stage_ms.items()}, "fallbacks", (oc.status!=0).sum().item())
print("ASG", {k: round(v*1000) for k, v in oa.stage_ms.items()}, "fallbacks", (oa.status!=0).sum().item())
