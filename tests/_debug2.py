import sys, torch, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
from conftest import load_npz
from paper_1812_07625_b200 import criterion as C, _native as nat
from oracle import criterion_oracle as orc
def al(x): return (x + 255)//256*256
name = sys.argv[1] if len(sys.argv) > 1 else "asg_c1"; g = load_npz(name)
B, T, N = g["em"].shape; L = g["targets"].shape[1]
spl = next(o for o in [2,4,8,10,12,16,20,24,32] if 32*o >= L); lpad = spl*32; nblk = (T+63)//64; BT = B*T
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
import math
print("fcc_a nan rows", np.where(~np.isfinite(fa[0]).all(axis=1))[0][:10], "ka range", ka[0].min(), ka[0].max())
print("fcc_b nan rows", np.where(~np.isfinite(fb[0]).all(axis=1))[0][:10], "kb range", kb[0].min(), kb[0].max())
print("fcc_a row sums log2 (first 12)", np.log2(fa[0,:12].sum(1)))
print("fcc_b row sums log2 (last 12)", np.log2(fb[0,-12:].sum(1)))
fac = get("fac_a", torch.float32).reshape(B, T, lpad); ea = get("fac_ea", torch.int32).reshape(B, T, 32)
print("fac_a nan rows", np.where(~np.isfinite(fac[0]).all(axis=1))[0][:10])
ge = out.grad_emissions[0].cpu().numpy(); print("grad nan rows", np.where(~np.isfinite(ge).all(axis=1))[0][:10])
pA = get("pA", torch.float32).reshape(B, nblk, 32, 32); pE = get("pE", torch.float32).reshape(B, nblk, 2, lpad)
print("pA nonfinite blocks", np.where(~np.isfinite(pA[0]).all(axis=(1,2)))[0])
print("pE nonfinite blocks", np.where(~np.isfinite(pE[0]).all(axis=(1,2)))[0])
bad = np.where(~np.isfinite(pE[0]))
print("pE bad idx", list(zip(*[x[:10] for x in bad])))
ebv = get("fac_eb", torch.int32).reshape(B, T, 32)
print("ea/eb rows 60..66 lanes 0..12:\n", ea[0, 60:67, :12], "\n", ebv[0, 60:67, :12])
