"""Histogram of executed SASS instructions (ncu --page source --csv of a
report) per opcode, and the hottest instruction windows, for one kernel."""
import collections
import csv
import sys

path, pat = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(path)))
out, cur, hdr = [], None, None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = r[1]
        hdr = None
        continue
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and cur and pat in cur and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        out.append(d)
key = "Instructions Executed"
tot = sum(float(d[key] or 0) for d in out)
ops = collections.Counter()
for d in out:
    op = d["Source"].split()[0] if d["Source"] else "?"
    if op.startswith("@"):
        op = d["Source"].split()[1]
    ops[op.split(".")[0]] += float(d[key] or 0)
print(f"{pat}: {tot:.4g} warp instructions, {len(out)} SASS lines")
for op, v in ops.most_common(30):
    print(f"  {op:12s} {v/tot*100:5.1f}%")
if len(sys.argv) > 3:
    win = int(sys.argv[3])
    vals = [float(d[key] or 0) for d in out]
    best = sorted(range(0, len(out), win), key=lambda i: -sum(vals[i:i + win]))[:6]
    for i in sorted(best):
        print(f"--- window {i}: {sum(vals[i:i+win])/tot*100:.1f}%")
        for d in out[i:i + win]:
            print(f"  {d['Address']} {float(d[key] or 0):10.0f} {d['Source'][:80]}")
