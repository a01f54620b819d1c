"""Chain-stage time vs lattice width (lattice warps W = ceil((2L+1)/128)) at B=64 T=1600."""
import sys, torch
sys.path.insert(0, ".")
import bench
from paper_1812_07625_b200 import criterion as C
for L in (20, 60, 120, 180, 240, 300):
    em, el, _, tg, tl, _, blank = bench.make_inputs(0, l=L)
    d = torch.from_numpy(em).cuda()
    best = 1e9
    for _ in range(4):
        o = C.ctc_loss_grad_batched(d, el, tg, tl, blank, check=False, trace=True)
        best = min(best, o.stage_ms["chain"])
    print(f"CTC L={L:4d} S={2*L+1:4d} W={(2*L+1+127)//128}: chain {best*1e3:7.1f} us  ({best*1e6/1600*1.965:6.0f} cyc/step)  fallbacks {(o.status != 0).sum().item()}")
