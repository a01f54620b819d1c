"""Turn the gpurun_out/ artefacts of tools/profile_round.sh into the committed
summaries under profiles/<round>/ (bench lines, launch list, ncu full summary)
and profiles/traffic.json (ncu DRAM bytes per launch, read by bench.py)."""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
rnd = sys.argv[1] if len(sys.argv) > 1 else "r1"
dst = os.path.join(ROOT, "profiles", rnd)
os.makedirs(dst, exist_ok=True)
shutil.copy(os.path.join(OUT, "bench.json"), os.path.join(dst, "bench.json"))
shutil.copy(os.path.join(OUT, "ref.json"), os.path.join(dst, "bench_reference.json"))
shutil.copy(os.path.join(OUT, "launches.csv"), os.path.join(dst, "launches_bench.csv"))


def short(name):
    n = name.replace("(int)", "")   # demangled template arguments (ncu --kernel-name-base demangled)
    n = n.split("(")[0].replace("void ", "").replace("w2l::", "")
    return n.replace("(anonymous namespace)::", "").replace("<unnamed>::", "").split("::")[-1]


# launch list of the bench
lines = open(os.path.join(OUT, "launches.csv")).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
agg = collections.defaultdict(list)
for r in csv.DictReader(lines[start:]):
    if r["Metric Name"] == "gpu__time_duration.sum":
        agg[short(r["Kernel Name"])[-48:]].append(float(r["Metric Value"]) / 1000)
tot = sum(sum(v) for v in agg.values())
out = ["# ncu --metrics gpu__time_duration.sum --clock-control none, "
       "`python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sub`",
       "# (cold-cache, serialised launches: compare SHARES, not absolutes; includes warmup, "
       "setup and the peak-probe launches)",
       f"{'kernel':50s}{'launches':>9s}{'mean_us':>10s}{'share':>8s}"]
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    out.append(f"{k:50s}{len(v):9d}{sum(v)/len(v):10.1f}{sum(v)/tot*100:7.1f}%")
open(os.path.join(dst, "launches_summary.txt"), "w").write("\n".join(out) + "\n")

# ncu --set full capture
metrics = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
           "sm__inst_executed.avg.per_cycle_active", "launch__registers_per_thread"]
raw = subprocess.run(["ncu", "-i", os.path.join(OUT, "full.ncu-rep"), "--page", "raw", "--csv",
                      "--metrics", ",".join(metrics)], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, units, data = rows[0], rows[1], rows[2:]
ix = {m: h.index(m) for m in metrics}
ik = h.index("Kernel Name")


def to_mb(v, u):
    v = float(v.replace(",", ""))
    return {"byte": v / 1e6, "Kbyte": v / 1e3, "Mbyte": v, "Gbyte": v * 1e3}.get(u, v)


keymap = {"asg_chain_kernel": "asg_chain", "ctc_chain_kernel": "ctc_chain",
          "asg_fcc_grad_kernel": "asg_grad_fcc"}
traffic = {}
out = ["# ncu --set full --clock-control none --import-source on --kernel-name-base demangled "
       "-k regex:'(chain_kernel<float|grad_kernel<[^>]*, float)' -s 4 -c 4 "
       "(tools/prof_chain.py all; bench shape B=64 T=1600 N=30 L=300; the fp32 tier)",
       f"{'kernel':30s}{'dur_us':>9s}{'dram_rd_MB':>11s}{'dram_wr_MB':>11s}{'occ%':>7s}"
       f"{'inst/frame':>11s}{'IPC':>6s}{'regs':>6s}"]
for r in data:
    name = short(r[ik])
    dur = float(r[ix["gpu__time_duration.sum"]].replace(",", ""))
    if units[ix["gpu__time_duration.sum"]] == "nsecond":
        dur /= 1e3
    rd = to_mb(r[ix["dram__bytes_read.sum"]], units[ix["dram__bytes_read.sum"]])
    wr = to_mb(r[ix["dram__bytes_write.sum"]], units[ix["dram__bytes_write.sum"]])
    key = next((v for k, v in keymap.items() if name.startswith(k)),
               "asg_grad" if name.startswith("asg_grad") else
               ("asg_grad_fac" if name.startswith("asg_fac_grad") else
                ("ctc_grad" if name.startswith("ctc_grad") else name)))
    traffic[key] = int((rd + wr) * 1e6)
    inst = float(r[ix["smsp__inst_executed.sum"]].replace(",", "")) / 102400
    out.append(f"{name:30s}{dur:9.1f}{rd:11.1f}{wr:11.1f}"
               f"{float(r[ix['sm__warps_active.avg.pct_of_peak_sustained_active']]):7.1f}"
               f"{inst:11.1f}{float(r[ix['sm__inst_executed.avg.per_cycle_active']]):6.2f}"
               f"{r[ix['launch__registers_per_thread']]:>6s}")
open(os.path.join(dst, "ncu_full_summary.txt"), "w").write("\n".join(out) + "\n")
if "asg_grad_fcc" in traffic and "asg_grad_fac" in traffic:   # the bench's "asg_grad" stage
    traffic["asg_grad"] = traffic["asg_grad_fcc"] + traffic["asg_grad_fac"]
json.dump(traffic, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)
print("\n".join(out))
