import sys, torch, numpy as np
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import bench
from paper_1812_07625_b200 import criterion as C, _native as nat
def al(x): return (x + 255)//256*256
em, el, ta, tc, tl, A, blank = bench.make_inputs(0)
B, T, N = em.shape; L = ta.shape[1]
spl = next(o for o in [2,4,8,10,12,16,20,24,32] if 32*o >= L); lpad = spl*32; nblk = (T+63)//64; BT = B*T
tpad = (T + 1 + 7)//8*8
ws = torch.zeros(nat.lib().w2l_asg_workspace_bytes(B, T, N, L), dtype=torch.uint8, device="cuda")
out = C.asg_loss_grad_batched(torch.from_numpy(em).cuda(), el, ta, tl, A, check=False, fallback=False, workspace=ws)
torch.cuda.synchronize()
st = out.status.cpu().numpy(); bad = np.where(st != 0)[0]; print("bad utts", bad, st[bad])
off = 0; offs = {}
for name, nb in [("fcc_a", BT*32*4), ("fcc_b", BT*32*4), ("fcc_ka", B*tpad*4), ("fcc_kb", B*tpad*4), ("fac_a", BT*lpad*4), ("fac_b", BT*lpad*4), ("fac_ea", BT*32*4), ("fac_eb", BT*32*4), ("scal", B*4*8), ("pA", B*nblk*1024*4), ("pE", B*nblk*2*lpad*4), ("pG", B*nblk*4*4)]:
    offs[name] = (off, nb); off = al(off + nb)
def get(name, dt):
    o, nb = offs[name]; return ws[o:o+nb].view(dt).cpu().numpy()
scal = get("scal", torch.float64).reshape(B, 4)
pg = get("pG", torch.float32).reshape(B, nblk, 4)
for b in bad[:3]:
    print("utt", b, "scal", scal[b], "fwd-bwd", scal[b,0]-scal[b,1], scal[b,2]-scal[b,3])
    print(" guard min/max per block (log2): fcc", pg[b,:,0].min(), pg[b,:,1].max(), " fac", pg[b,:,2].min(), pg[b,:,3].max())
    print(" worst fac blocks", np.argsort(-np.abs(pg[b,:,2:]).max(1))[:5], np.abs(pg[b,:,2:]).max(1).max())
good = [b for b in range(B) if st[b]==0][:3]
for b in good:
    print("good", b, "fcc dev", np.abs(pg[b,:,:2]).max(), "fac dev", np.abs(pg[b,:,2:]).max(), scal[b,0]-scal[b,1], scal[b,2]-scal[b,3])
allg = np.abs(pg[:, :, :]).max(axis=(1,))
print("per-utt max |dev| fcc", np.round(np.abs(pg[:,:,:2]).max(axis=(1,2)),6)[:20])
print("per-utt max |dev| fac", np.round(np.abs(pg[:,:,2:]).max(axis=(1,2)),6)[:20])
