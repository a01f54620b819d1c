import sys, torch, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
from conftest import load_npz
from paper_1812_07625_b200 import criterion as C
from oracle import criterion_oracle as orc
for name in ["ctc_c2_one", "ctc_ragged"]:
    g = load_npz(name)
    out = C.ctc_loss_grad_batched(torch.from_numpy(g["em"]).cuda(), g["em_len"], g["targets"], g["tgt_len"], int(g["blank"]), check=False, fallback=False)
    torch.cuda.synchronize()
    print(name, "status", out.status.cpu().numpy(), "loss", out.loss.cpu().numpy()[:4], "ref", g["loss"][:4])
    print("  grad rel", [round(orc.rel_err(out.grad_emissions[b].cpu().numpy(), g["grad_e"][b]), 8) for b in range(len(g["loss"]))])
