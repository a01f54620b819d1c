import numpy as np, sys
sys.path.insert(0, '.')
import bench
from scipy.special import logsumexp
em, el, ta, tc, tl, A, blank = bench.make_inputs(0, b=4)
def ctc_ab(e, y, blank):
    T = e.shape[0]; L = len(y); S = 2*L+1
    lab = np.full(S, blank); lab[1::2] = y
    skip = np.zeros(S, bool); 
    for s in range(3, S, 2): skip[s] = y[s//2] != y[s//2-1]
    la = np.full((T,S), -np.inf); lb = np.full((T,S), -np.inf)
    la[0,0] = e[0,lab[0]]; la[0,1] = e[0,lab[1]]
    for t in range(1,T):
        p = la[t-1]
        x = np.logaddexp(p, np.concatenate([[-np.inf], p[:-1]]))
        x2 = np.where(skip, np.concatenate([[-np.inf,-np.inf], p[:-2]]), -np.inf)
        la[t] = e[t, lab] + np.logaddexp(x, x2)
    lb[T-1, S-1] = 0; lb[T-1, S-2] = 0
    for t in range(T-2, -1, -1):
        w = lb[t+1] + e[t+1, lab]
        x = np.logaddexp(w, np.concatenate([w[1:], [-np.inf]]))
        sk2 = np.concatenate([skip[2:], [False, False]])
        x2 = np.where(sk2, np.concatenate([w[2:], [-np.inf,-np.inf]]), -np.inf)
        lb[t] = np.logaddexp(x, x2)
    return la, lb
for spl in (2, 4, 8):
  worst = 0; worstpost = 0
  for b in range(2):
    e = em[b].astype(np.float64); y = tc[b, :tl[b]]
    la, lb = ctc_ab(e, y, blank)
    lz = logsumexp(la[-1, -2:])
    post = la + lb - lz
    S = la.shape[1]; Sp = (S + spl - 1)//spl*spl
    for arr in (la, lb):
        a = np.full((arr.shape[0], Sp), -np.inf); a[:, :S] = arr
        blk = a.reshape(arr.shape[0], -1, spl)
        mx = blk.max(axis=2, keepdims=True)
        span = (mx - blk) / np.log(2)   # log2 below lane max
        p = np.full((arr.shape[0], Sp), -np.inf); p[:, :S] = post
        p = p.reshape(blk.shape)
        rel = np.isfinite(p) & (p > np.log(1e-9))
        if rel.any():
            worst = max(worst, span[rel].max())
  print("spl", spl, "max log2 span below lane max among states with posterior>1e-9:", worst)
