import sys, torch
sys.path.insert(0, '.')
from oracle import criterion_oracle as orc
from paper_1812_07625_b200 import criterion as C
which = sys.argv[1] if len(sys.argv) > 1 else "all"
em, el, tg, tl, a = orc.synth_asg(20260002, 64, 1600, 30, 300)
emd = torch.from_numpy(em).cuda()
emc, elc, tgc, tlc, blank = orc.synth_ctc(20260004, 64, 1600, 30, 300)
emcd = torch.from_numpy(emc).cuda()
for _ in range(2):
    if which in ("all", "asg"): C.asg_loss_grad_batched(emd, el, tg, tl, a, check=False)
    if which in ("all", "ctc"): C.ctc_loss_grad_batched(emcd, elc, tgc, tlc, blank, check=False)
    if which in ("all", "vit"): C.viterbi_batched(emd, el, a, check=False)
torch.cuda.synchronize()
