import sys, torch, numpy as np
sys.path.insert(0,'.')
from conftest import load_npz
from paper_1812_07625_b200 import criterion as C
from oracle import criterion_oracle as orc
for name in ["asg_c1", "asg_c3_one", "asg_ragged"]:
    g = load_npz(name)
    try:
        out = C.asg_loss_grad_batched(torch.from_numpy(g["em"]).cuda(), g["em_len"], g["targets"], g["tgt_len"], g["trans"], check=False, fallback=False)
        torch.cuda.synchronize()
        print(name, out.status.cpu().numpy(), out.loss.cpu().numpy()[:4], g["loss"][:4])
        print("  grad rel", [orc.rel_err(out.grad_emissions[b].cpu().numpy(), g["grad_e"][b]) for b in range(len(g["loss"]))])
    except Exception as ex:
        print(name, "ERR", ex)
for name in ["ctc_c2_one", "ctc_ragged"]:
    g = load_npz(name)
    try:
        out = C.ctc_loss_grad_batched(torch.from_numpy(g["em"]).cuda(), g["em_len"], g["targets"], g["tgt_len"], int(g["blank"]), check=False, fallback=False)
        torch.cuda.synchronize()
        print(name, out.status.cpu().numpy(), out.loss.cpu().numpy()[:4], g["loss"][:4])
        print("  grad rel", [orc.rel_err(out.grad_emissions[b].cpu().numpy(), g["grad_e"][b]) for b in range(len(g["loss"]))])
    except Exception as ex:
        print(name, "ERR", ex)
