"""One batched Viterbi call at C4 shape (B=64 T=1600 N=30) for ncu."""
import sys, torch
sys.path.insert(0, ".")
from oracle import criterion_oracle as orc
from paper_1812_07625_b200 import criterion as C
em, el, _, _, a = orc.synth_asg(20260003, 64, 1600, 30, 1)
d = torch.from_numpy(em).cuda()
for _ in range(2):
    C.viterbi_batched(d, el, a, check=False)
torch.cuda.synchronize()
