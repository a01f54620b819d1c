"""One batched Viterbi call at C4 shape (B=64 T=1600 N=30) for ncu."""
import sys, torch
sys.path.insert(0, ".")
import bench
from paper_1812_07625_b200 import criterion as C
em, el, _, _, _, a, _ = bench.make_inputs(0)
d = torch.from_numpy(em).cuda()
for _ in range(2):
    C.viterbi_batched(d, el, a, check=False)
torch.cuda.synchronize()
