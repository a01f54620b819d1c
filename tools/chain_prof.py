"""Steady-state per-warp cycle profile of the chain kernels (library built with
-DW2L_PROF): consumers blocks 40..159 (120 blocks of 8 steps), producer chunks
10..39 (30 chunks of 32 frames)."""
import ctypes, sys
import numpy as np, torch
sys.path.insert(0, ".")
import bench
from paper_1812_07625_b200 import criterion as C, _native
lib = _native.lib()
buf = np.zeros(64 * 2 * 16 * 8, np.uint64)
em, el, ta, tc, tl, A, blank = bench.make_inputs(0)
d = torch.from_numpy(em).cuda()
for which in ("ctc", "asg"):
    for _ in range(2):
        if which == "ctc":
            C.ctc_loss_grad_batched(d, el, tc, tl, blank, check=False)
        else:
            C.asg_loss_grad_batched(d, el, ta, tl, A, check=False)
        torch.cuda.synchronize()
        getattr(lib, "w2l_debug_prof_" + which)(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), 1)
    p = buf.reshape(64, 2, 16, 8).view(np.int64).astype(np.float64)
    print(which, "steady state, cycles per 8 steps: span(block40->159)/120, waits prod/up/dn/wait3, compute; producer: cons-wait/cpasync/convert per 8 frames")
    for dr in range(2):
        t0 = p[:, dr, 0, 4]
        print("  dir", dr, "clock at block 100 (frames 800..807) minus producer publish of chunk 25 (frames 800..831):", [round((p[:, dr, w, 4] - t0).mean()) for w in range(1, 8) if p[:, dr, w, 0].mean() > 0])
        for w in range(8):
            if p[:, dr, w, 0].mean() == 0: continue
            if w == 0:
                print(f"  dir{dr} producer: cons-wait {p[:,dr,w,1].mean()/120:7.1f} cp.async {p[:,dr,w,2].mean()/120:7.1f} convert(+wait) {p[:,dr,w,3].mean()/120:7.1f}")
                continue
            span = -p[:, dr, w, 5].mean() / 119
            print(f"  dir{dr} warp{w}: span {span:7.1f}  prod {p[:,dr,w,1].mean()/120:6.1f}  up {p[:,dr,w,2].mean()/120:6.1f}  dn {p[:,dr,w,3].mean()/120:6.1f}  wait3 {p[:,dr,w,6].mean()/120:6.1f}  compute {p[:,dr,w,7].mean()/120:6.1f}")
