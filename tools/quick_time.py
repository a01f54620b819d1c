import time, torch, numpy as np, sys
sys.path.insert(0, '.')
from oracle import criterion_oracle as orc
from paper_1812_07625_b200 import criterion as C
em, el, tg, tl, a = orc.synth_asg(20260002, 64, 1600, 30, 300)
emd = torch.from_numpy(em).cuda()
def run():
    return C.asg_loss_grad_batched(emd, el, tg, tl, a, check=False)
out = run(); torch.cuda.synchronize()
print("status", out.status.cpu().numpy()[:8], "needs_exact?")
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
for _ in range(3): run()
s.record()
for _ in range(10): run()
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e)/10
print(f"ASG C3 B=64: {ms:.3f} ms/step, {64*1600/ms*1e3:.3e} frames/s")
emc, elc, tgc, tlc, blank = orc.synth_ctc(20260004, 64, 1600, 30, 300)
emcd = torch.from_numpy(emc).cuda()
def runc(): return C.ctc_loss_grad_batched(emcd, elc, tgc, tlc, blank, check=False)
runc(); torch.cuda.synchronize()
s.record()
for _ in range(10): runc()
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e)/10
print(f"CTC B=64 T=1600 L=300: {ms:.3f} ms/step, {64*1600/ms*1e3:.3e} frames/s")
def runv(): return C.viterbi_batched(emd, el, a, check=False)
runv(); torch.cuda.synchronize()
s.record()
for _ in range(10): runv()
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e)/10
print(f"Viterbi B=64 T=1600: {ms:.3f} ms/step, {64*1600/ms*1e3:.3e} frames/s")
from paper_1812_07625_b200 import _native
print(_native.probe_peaks())
