"""CTA timeline of one streamed (PDL) call: when the chain CTAs run and when
the gradient CTAs are dispatched, released by the chains' progress words and
finish.  Needs a -DW2L_TIMELINE build:
    bash tools/ab_flags.sh tl -DW2L_TIMELINE
    W2L_LIB=abl/tl.so python tools/timeline_pdl.py [ctc|asg|both]
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1812_07625_b200 import _native, criterion as C  # noqa: E402

lib = _native.lib()
fn = lib.w2l_timeline_read if hasattr(lib, "w2l_timeline_read") else None
if fn is None:
    fn = ctypes.CDLL(_native.LIB).w2l_timeline_read
fn.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
fn.restype = ctypes.c_int
buf = np.zeros((1 << 16, 4), dtype=np.uint64)


def read(kind):
    n = fn(kind, buf.ctypes.data, 1 << 16)
    return buf[:n].copy()


em, el, ta, tc, tl, A, blank = bench.make_inputs(0)
d = torch.from_numpy(em).cuda()
el_d, ta_d, tc_d, tl_d, A_d = (torch.from_numpy(x).cuda() for x in (el, ta, tc, tl, A))
side = torch.cuda.Stream()
main = torch.cuda.current_stream()
which = sys.argv[1] if len(sys.argv) > 1 else "both"
FB = os.environ.get("TL_NOFB") != "1"   # TL_NOFB=1: no fallback tiers (timing-only builds)


ASG_DELAY = int(os.environ.get("TL_ASG_DELAY", "0"))   # cycles the second stream is held back


SCHED = os.environ.get("TL_SCHED", "bench")   # "bench": bench.py's schedule; "plain"
validated = torch.cuda.Event()


def call():
    bench_sched = SCHED == "bench" and which == "both"
    asg = lambda **kw: C.asg_loss_grad_batched(d, el_d, ta_d, tl_d, A_d, check=False, fallback=FB,
                                               stream_grad=bench_sched and bench.STREAM_ASG, **kw)
    ctc = lambda **kw: C.ctc_loss_grad_batched(d, el_d, tc_d, tl_d, blank, check=False,
                                               fallback=FB,
                                               stream_grad=bench_sched and bench.STREAM_CTC, **kw)
    if which != "both":
        (asg if which == "asg" else ctc)()
        return
    # bench.py's schedule (first criterion, stagger) or both started together
    first, second = (asg, ctc) if bench.FIRST == "asg" else (ctc, asg)
    side.wait_stream(main)
    if bench_sched and bench.STAGGER:
        first(phase="validate")
        validated.record(main)
        first(phase="rest")
        side.wait_event(validated)
    else:
        first()
    with torch.cuda.stream(side):
        if ASG_DELAY:
            torch.cuda._sleep(ASG_DELAY)
        second()
    main.wait_stream(side)


for _ in range(5):
    call()
torch.cuda.synchronize()
read(0), read(1)
# LOOP=n: n bench-like steps back to back (L2 flush + call), the last one
# analysed; otherwise one call behind a ~1 ms sleep, so every launch is
# queued before the GPU reaches it (the host's enqueue latency would show up
# as gaps)
loops = int(os.environ.get("LOOP", "0"))
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda") if loops else None
torch.cuda._sleep(2_000_000)
g0 = torch.cuda.Event(enable_timing=True)
g1 = torch.cuda.Event(enable_timing=True)
if loops:
    for i in range(loops):
        flush.zero_()
        if i == loops - 1:
            g0.record()
        call()
else:
    g0.record()
    call()
g1.record()
torch.cuda.synchronize()
print(f"call (events, after the sleep): {g0.elapsed_time(g1)*1e3:.1f} us")
recs = np.concatenate([read(0), read(1)])
if loops:   # keep the last step: records after its first chain start
    kk = recs[:, 0].astype(np.int64) // 1000000
    cs = np.sort(recs[(kk == 1) | (kk == 3), 1].astype(np.int64))
    gaps = np.nonzero(np.diff(cs) > 150000)[0]   # steps are > 150 us apart
    t_last = cs[gaps[-1] + 1] if len(gaps) else cs[0]
    recs = recs[recs[:, 1].astype(np.int64) >= t_last - 20000]
if os.environ.get("TL_DUMP"):   # raw records for offline analysis
    np.save(os.environ["TL_DUMP"], recs)
tag = recs[:, 0].astype(np.int64)
kind = tag // 1000000
t = recs[:, 1:].astype(np.int64)
t0 = t[kind % 2 == 1, 0].min()   # first chain CTA start
us = lambda x: (x - t0) / 1e3
for k, name in [(1, "ctc_chain"), (3, "asg_chain")]:
    m = kind == k
    if m.any():
        print(f"{name:10s} n={m.sum():4d} start {us(t[m,0].min()):7.1f}..{us(t[m,0].max()):7.1f}"
              f"  end {us(t[m,1].min()):7.1f}..{us(t[m,1].max()):7.1f} us")
# chain CTAs per SM (t2 of a chain record is its SM id) vs their end times
ch = (kind == 1) | (kind == 3)
if ch.any():
    slot0 = t[ch, 2] >> 16        # hardware warp slot of the CTA's warp 0
    t[ch, 2] &= 0xffff
    sm = t[ch, 2]
    # ASG CTAs sharing an SM with a CTC CTA: who took the lower warp slots
    kinds_ = kind[ch]
    first, second = [], []
    for smv in np.unique(sm):
        idx = np.nonzero(sm == smv)[0]
        if len(idx) == 2 and set(kinds_[idx]) == {1, 3}:
            ia = idx[kinds_[idx] == 3][0]
            ic = idx[kinds_[idx] == 1][0]
            (first if slot0[ia] < slot0[ic] else second).append(ia)
    for nm, lst in [("ASG below CTC (ASG slots first)", first), ("ASG above CTC", second)]:
        if lst:
            e = us(t[ch, 1][np.array(lst)])
            sl = slot0[np.array(lst)]
            print(f"  {nm}: n={len(lst)} end {e.min():7.1f}/{np.median(e):7.1f}/{e.max():7.1f} us;"
                  f" ASG warp-0 slot mod 4: {np.bincount(sl % 4, minlength=4).tolist()}")
    cnt = {s: int((sm == s).sum()) for s in np.unique(sm)}
    for c in sorted(set(cnt.values())):
        m = np.array([cnt[s] == c for s in sm])
        e = us(t[ch, 1][m])
        print(f"chains on SMs hosting {c}: n={m.sum():4d} end {e.min():7.1f}/{np.median(e):7.1f}/{e.max():7.1f} us")
    # SMs hosting two chain CTAs: which kinds share them
    kinds = kind[ch]
    pair = {}
    for smv in np.unique(sm):
        idx = np.nonzero(sm == smv)[0]
        if len(idx) == 2:
            pair[smv] = "+".join(sorted("asg" if kinds[i] == 3 else "ctc" for i in idx))
    for pt in sorted(set(pair.values())):
        m = np.array([pair.get(s_) == pt for s_ in sm])
        e = us(t[ch, 1][m])
        print(f"  pair {pt}: {m.sum() // 2:3d} SMs, chain end {e.min():7.1f}/{np.median(e):7.1f}/{e.max():7.1f} us;"
              f" chain start spread {us(t[ch, 0][m]).min():.1f}..{us(t[ch, 0][m]).max():.1f}")
    k2 = kind[ch]
    for kk, nm in [(1, "ctc"), (3, "asg")]:
        mm = k2 == kk
        if mm.any():
            e = us(t[ch, 1][mm]); d = (tag[ch][mm] % 10)
            print(f"  {nm}: fwd end med {np.median(e[d == 0]):7.1f} bwd end med {np.median(e[d == 1]):7.1f};"
                  f" slowest 5 (b,dir,sm,end): " + ", ".join(
                      f"({int(tag[ch][mm][i] % 1000000 // 10)},{int(d[i])},{int(sm[mm][i])},{e[i]:.0f})"
                      for i in np.argsort(-e)[:5]))
for k, name in [(2, "ctc_grad"), (4, "asg_grad")]:
    m = kind == k
    if not m.any():
        continue
    cend = us(t[kind == k - 1, 1].max())
    s, w, e = us(t[m, 0]), us(t[m, 1]), us(t[m, 2])
    busy = e - w
    print(f"{name:10s} n={m.sum():4d} dispatch {s.min():7.1f}/{np.median(s):7.1f}/{s.max():7.1f}"
          f"  released {w.min():7.1f}/{np.median(w):7.1f}/{w.max():7.1f}"
          f"  end {e.min():7.1f}/{np.median(e):7.1f}/{e.max():7.1f} us (min/med/max)")
    before = np.clip(np.minimum(e, cend) - w, 0, None).sum() / busy.sum()
    print(f"{'':10s} CTA busy {busy.mean():6.1f} us mean; {before*100:4.1f}% of gradient CTA time"
          f" before its chain ended ({cend:.1f} us); waited {np.mean(w - s):6.1f} us mean")
    if k == 4:   # fac (x even) vs fcc (x odd) CTA bodies
        body = (tag[m] % 1000000) // 500000
        for bb, nm in [(0, "fac"), (1, "fcc")]:
            mm = body == bb
            print(f"{'':10s} {nm}: n={mm.sum()} busy {busy[mm].mean():6.1f} us mean, dispatch med "
                  f"{np.median(s[mm]):7.1f}, end med {np.median(e[mm]):7.1f} max {e[mm].max():7.1f}")
    # CTAs of this launch running at once (sampled every 2 us)
    grid_t = np.arange(w.min(), e.max(), 2.0)
    conc = [int(((w <= x) & (e > x)).sum()) for x in grid_t]
    print(f"{'':10s} concurrent CTAs: max {max(conc)}, median {int(np.median(conc))}")
    hist = np.histogram(e, bins=12)
    print(f"{'':10s} end histogram: " + " ".join(f"{int(c)}@{b:.0f}" for c, b in zip(hist[0], hist[1])))
