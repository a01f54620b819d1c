"""Per-CUDA-source-line instruction counts and stall samples from
`ncu -i X --page source --csv --print-source cuda,sass -k <kernel>`:
usage: python tools/src_lines.py mix.csv [frames] [top]"""
import csv, sys, collections
path = sys.argv[1]
frames = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
rows = list(csv.reader(open(path)))
hdr = None; cur_file = None; cur_line = None; cur_src = ""
inst = collections.Counter(); smp = collections.Counter(); src = {}
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur_file = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) != len(hdr): continue
    if r[0]:
        cur_line = (cur_file, int(r[0])); src[cur_line] = r[1]
    if cur_line is None: continue
    if r[2]:
        try:
            inst[cur_line] += float(r[7]); smp[cur_line] += float(r[4])
        except ValueError:
            pass
T = sum(inst.values()); S = sum(smp.values())
print(f"total {T:.0f} inst ({T/frames:.1f}/frame), {S:.0f} samples")
for k, v in sorted(inst.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{str(k[0]):>14s}:{(k[1] if k[1] is not None else -1):<5d} {v/frames:7.1f}/fr {smp[k]/S*100:5.1f}%smp  {src.get(k,'').strip()[:70]}")
