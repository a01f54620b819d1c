import sys, torch, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
from conftest import load_npz
from paper_1812_07625_b200 import criterion as C, _native as nat
from oracle import criterion_oracle as orc
def al(x): return (x + 255)//256*256
g = load_npz("asg_c1")
B, T, N = g["em"].shape; L = g["targets"].shape[1]
spl = 2 if 64 >= L else 4; lpad = spl*32; nblk = (T+63)//64; BT = B*T
ws = torch.zeros(nat.lib().w2l_asg_workspace_bytes(B, T, N, L), dtype=torch.uint8, device="cuda")
out = C.asg_loss_grad_batched(torch.from_numpy(g["em"]).cuda(), g["em_len"], g["targets"], g["tgt_len"], g["trans"], check=False, fallback=False, workspace=ws)
torch.cuda.synchronize()
print("status", out.status.cpu().numpy(), "loss", out.loss.cpu().numpy(), "ref", g["loss"])
off = 0; offs = {}
for name, nb in [("fcc_a", BT*32*4), ("fcc_b", BT*32*4), ("fcc_ka", BT*4), ("fcc_kb", BT*4), ("fac_a", BT*lpad*4), ("fac_b", BT*lpad*4), ("fac_ea", BT*32*4), ("fac_eb", BT*32*4), ("scal", B*4*8), ("pA", B*nblk*1024*4), ("pE", B*nblk*2*lpad*4), ("pG", B*nblk*4*4)]:
    offs[name] = (off, nb); off = al(off + nb)
def get(name, dt):
    o, nb = offs[name]; return ws[o:o+nb].view(dt).cpu().numpy()
scal = get("scal", torch.float64).reshape(B, 4); print("scal", scal)
pg = get("pG", torch.float32).reshape(B, nblk, 4); print("guard", pg[0])
fa = get("fcc_a", torch.float32).reshape(B, T, 32); ka = get("fcc_ka", torch.int32).reshape(B, T)
print("fcc_a row0..2", fa[0, :3, :6], ka[0, :5])
fb = get("fcc_b", torch.float32).reshape(B, T, 32); kb = get("fcc_kb", torch.int32).reshape(B, T)
print("fcc_b rows", fb[0, -3:, :6], kb[0, -5:])
for b in range(B):
    print(b, "grad rel", orc.rel_err(out.grad_emissions[b].cpu().numpy(), g["grad_e"][b]), "gA", orc.rel_err(out.grad_transitions.cpu().numpy(), g["grad_a_per_utt"].sum(0)))
