"""One ASG and one CTC batched call at the bench shape (for ncu captures)."""
import sys, torch
sys.path.insert(0, ".")
import bench
from paper_1812_07625_b200 import criterion as C
em, el, ta, tc, tl, A, blank = bench.make_inputs(0)
d = torch.from_numpy(em).cuda()
which = sys.argv[1] if len(sys.argv) > 1 else "all"
for _ in range(2):
    if which in ("all", "ctc"):
        C.ctc_loss_grad_batched(d, el, tc, tl, blank, check=False)
    if which in ("all", "asg"):
        C.asg_loss_grad_batched(d, el, ta, tl, A, check=False)
torch.cuda.synchronize()
