"""One criterion alone (the usual training call): plain vs streamed gradient
(W2L_FLAG_STREAM_GRAD), device time per call at the bench shape."""
import sys, torch
sys.path.insert(0, ".")
import bench
from paper_1812_07625_b200 import criterion as C
em, el, ta, tc, tl, A, blank = bench.make_inputs(0)
d = torch.from_numpy(em).cuda()
el_d, ta_d, tc_d, tl_d, A_d = (torch.from_numpy(x).cuda() for x in (el, ta, tc, tl, A))
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
oa = C.asg_loss_grad_batched(d, el_d, ta_d, tl_d, A_d, check=False)
oc = C.ctc_loss_grad_batched(d, el_d, tc_d, tl_d, blank, check=False)
calls = {
    "asg": lambda sg: C.asg_loss_grad_batched(d, el_d, ta_d, tl_d, A_d, check=False, out=oa, stream_grad=sg),
    "ctc": lambda sg: C.ctc_loss_grad_batched(d, el_d, tc_d, tl_d, blank, check=False, out=oc, stream_grad=sg),
}
for name, fn in calls.items():
    for sg in (False, True, False, True):
        for _ in range(5):
            fn(sg)
        ts = []
        for _ in range(20):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); fn(sg); e.record(); ts.append((s, e))
        torch.cuda.synchronize()
        print(f"{name} stream_grad={int(sg)}: {sum(a.elapsed_time(b) for a, b in ts) / 20:.4f} ms")
