"""Batched Viterbi time at the C4 shape (B=64, T=1600, N=30), CUDA events."""
import sys, torch
sys.path.insert(0, ".")
import bench
from paper_1812_07625_b200 import criterion as C
em, el, ta, tc, tl, A, blank = bench.make_inputs(0)
d = torch.from_numpy(em).cuda(); eld = torch.from_numpy(el).cuda(); Ad = torch.from_numpy(A).cuda()
for _ in range(5):
    C.viterbi_batched(d, eld, Ad, check=False)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20):
    C.viterbi_batched(d, eld, Ad, check=False)
e.record(); e.synchronize()
print("viterbi ms", s.elapsed_time(e) / 20)
