"""Stall-reason breakdown from `ncu -i X --page source --csv --print-source sass`
for one kernel: totals per reason and the hottest SASS lines.
usage: python tools/stalls.py src.csv <kernel-substring> [top]"""
import csv, sys, collections
path, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
rows = list(csv.reader(open(path)))
cur = None; hdr = None; out = []
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = r[1]; hdr = None; continue
    if r and r[0] == "Address":
        hdr = r; continue
    if hdr and cur and pat in cur and len(r) == len(hdr):
        out.append(dict(zip(hdr, r)))
def f(x):
    try: return float(x)
    except: return 0.0
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
for d in out:
    for h in reasons: tot[h] += f(d[h])
S = sum(f(d["Warp Stall Sampling (All Samples)"]) for d in out)
print(f"{pat}: {len(out)} SASS lines, {S:.0f} samples")
for h, v in tot.most_common(): 
    if v: print(f"  {h:28s} {v/S*100:5.1f}%")
print("hottest lines (samples, top reasons):")
hot = sorted(range(len(out)), key=lambda i: -f(out[i]["Warp Stall Sampling (All Samples)"]))[:top]
for i in sorted(hot):
    d = out[i]
    rs = sorted(((f(d[h]), h[6:]) for h in reasons), reverse=True)[:3]
    print(f"  {d['Address']:>6s} {f(d['Warp Stall Sampling (All Samples)']):7.0f} {f(d['Instructions Executed']):9.0f}  {d['Source'][:60]:60s} " + " ".join(f"{h}:{v:.0f}" for v, h in rs if v))
