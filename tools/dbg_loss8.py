import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_1812_07625_b200 import criterion as C
rng = np.random.default_rng(81)
lens = [(16, 1), (140, 127), (128, 128), (129, 129), (255, 200), (256, 256), (300, 257), (400, 384), (450, 385), (500, 450)]
b_sz, t_max, n = len(lens) + 1, 520, 30
em = rng.standard_normal((b_sz, t_max, n), dtype=np.float32)
a = rng.standard_normal((n, n)).astype(np.float32)
el = np.array([t for t, _ in lens] + [300], np.int32)
tl = np.array([l for _, l in lens] + [100], np.int32)
tg = np.full((b_sz, int(tl.max())), -1, np.int64)
for b in range(b_sz):
    seq = [int(rng.integers(0, n))]
    while len(seq) < tl[b]:
        v = int(rng.integers(0, n))
        if v != seq[-1]: seq.append(v)
    tg[b, :tl[b]] = seq
    em[b, el[b]:] = 0.0
em[-1, 5, 3] = np.nan
x = torch.from_numpy(em).cuda()
for fb in [False, "f64", True]:
    out = C.asg_loss_grad_batched(x, el, tg, tl, a, check=False, fallback=fb)
    print(fb, out.status.cpu().numpy(), out.loss.cpu().numpy()[7:10])
