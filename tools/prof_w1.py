"""CTC chain with a single lattice warp (L=20) for ncu source-level analysis."""
import sys, torch
sys.path.insert(0, ".")
from oracle import criterion_oracle as orc
from paper_1812_07625_b200 import criterion as C
em, el, tg, tl, blank = orc.synth_ctc(20260004, 64, 1600, 30, 20)
d = torch.from_numpy(em).cuda()
for _ in range(2):
    C.ctc_loss_grad_batched(d, el, tg, tl, blank, check=False)
torch.cuda.synchronize()
