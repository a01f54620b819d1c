"""Host-side cost of one batched API call (enqueue only) vs its device time."""
import sys, time, torch
sys.path.insert(0, ".")
import bench
from paper_1812_07625_b200 import criterion as C, _native
em, el, ta, tc, tl, A, blank = bench.make_inputs(0)
dev = torch.device("cuda")
em_d, el_d = torch.from_numpy(em).to(dev), torch.from_numpy(el).to(dev)
ta_d, tc_d, tl_d = torch.from_numpy(ta).to(dev), torch.from_numpy(tc).to(dev), torch.from_numpy(tl).to(dev)
A_d = torch.from_numpy(A).to(dev)
lib = _native.lib()
B, T, N = em.shape
ws_a = torch.empty(lib.w2l_asg_workspace_bytes(B, T, N, 300), dtype=torch.uint8, device=dev)
ws_c = torch.empty(lib.w2l_ctc_workspace_bytes(B, T, N, 300), dtype=torch.uint8, device=dev)
oa = C.asg_loss_grad_batched(em_d, el_d, ta_d, tl_d, A_d, check=False, workspace=ws_a)
oc = C.ctc_loss_grad_batched(em_d, el_d, tc_d, tl_d, blank, check=False, workspace=ws_c)
torch.cuda.synchronize()
for name, fn in [("asg all", lambda: C.asg_loss_grad_batched(em_d, el_d, ta_d, tl_d, A_d, check=False, workspace=ws_a, out=oa)),
                 ("asg chain", lambda: C.asg_loss_grad_batched(em_d, el_d, ta_d, tl_d, A_d, check=False, workspace=ws_a, out=oa, phase="chain")),
                 ("ctc all", lambda: C.ctc_loss_grad_batched(em_d, el_d, tc_d, tl_d, blank, check=False, workspace=ws_c, out=oc))]:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name:10s} host enqueue {1e6*(t1-t0)/20:8.1f} us/call   wall incl. device {1e6*(t2-t0)/20:8.1f} us/call")

side = torch.cuda.Stream()
main_s = torch.cuda.current_stream()
def old():
    side.wait_stream(main_s)
    with torch.cuda.stream(side):
        C.ctc_loss_grad_batched(em_d, el_d, tc_d, tl_d, blank, check=False, workspace=ws_c, out=oc)
    C.asg_loss_grad_batched(em_d, el_d, ta_d, tl_d, A_d, check=False, workspace=ws_a, out=oa)
    main_s.wait_stream(side)
def split():
    side.wait_stream(main_s)
    with torch.cuda.stream(side):
        C.ctc_loss_grad_batched(em_d, el_d, tc_d, tl_d, blank, check=False, workspace=ws_c, out=oc, phase="chain")
    C.asg_loss_grad_batched(em_d, el_d, ta_d, tl_d, A_d, check=False, workspace=ws_a, out=oa, phase="chain")
    side.wait_stream(main_s)
    main_s.wait_stream(side)
    with torch.cuda.stream(side):
        C.ctc_loss_grad_batched(em_d, el_d, tc_d, tl_d, blank, check=False, workspace=ws_c, out=oc, phase="grad")
    C.asg_loss_grad_batched(em_d, el_d, ta_d, tl_d, A_d, check=False, workspace=ws_a, out=oa, phase="grad")
    main_s.wait_stream(side)
def seq():
    C.ctc_loss_grad_batched(em_d, el_d, tc_d, tl_d, blank, check=False, workspace=ws_c, out=oc)
    C.asg_loss_grad_batched(em_d, el_d, ta_d, tl_d, A_d, check=False, workspace=ws_a, out=oa)
def chains_only():
    side.wait_stream(main_s)
    with torch.cuda.stream(side):
        C.ctc_loss_grad_batched(em_d, el_d, tc_d, tl_d, blank, check=False, workspace=ws_c, out=oc, phase="chain")
    C.asg_loss_grad_batched(em_d, el_d, ta_d, tl_d, A_d, check=False, workspace=ws_a, out=oa, phase="chain")
    main_s.wait_stream(side)
for name, fn in [("old", old), ("split", split), ("seq", seq), ("chains", chains_only), ("old", old), ("split", split)]:
    for _ in range(3): fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(20): fn()
    e.record(); torch.cuda.synchronize()
    print(f"{name:8s} {s.elapsed_time(e)/20*1e3:8.1f} us/step")
