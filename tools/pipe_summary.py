"""Per-kernel pipe utilisation from an ncu --set full report (profiles/<round>/ncu_pipes.txt):
% of peak sustained issue per pipe (FMA, ALU, XU = MUFU/SFU, LSU, FP64, tensor, TMA, TMEM),
the issue-slot busy %, DRAM throughput % -- the evidence for 'no GEMM-shaped work'.
usage: python tools/pipe_summary.py gpurun_out/full.ncu-rep profiles/r2/ncu_pipes.txt"""
import csv, subprocess, sys
rep, out = sys.argv[1], sys.argv[2]
pipes = ["fma", "alu", "xu", "lsu", "fp64", "tc", "tma", "tmem", "uniform"]
mets = [f"sm__inst_executed_pipe_{p}.avg.pct_of_peak_sustained_active" for p in pipes]
mets += ["sm__inst_issued.avg.pct_of_peak_sustained_active",
         "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
         "gpu__time_duration.sum"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(mets)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
lines = ["# ncu --set full (" + rep.split("/")[-1] + "): % of peak sustained per pipe, issue-active %, "
         "DRAM throughput %",
         f"{'kernel':30s}" + "".join(f"{p:>8s}" for p in pipes) + f"{'issue%':>8s}{'dram%':>7s}{'us':>8s}"]
for r in rows[2:]:
    name = r[h.index("Kernel Name")].replace("(int)", "").split("(")[0].split("::")[-1][:29]
    vals = [float(r[h.index(m)].replace(",", "") or 0) for m in mets]
    unit = rows[1][h.index("gpu__time_duration.sum")]
    us = vals[-1] / 1000 if unit == "nsecond" else (vals[-1] * 1000 if unit == "msecond" else vals[-1])
    lines.append(f"{name:30s}" + "".join(f"{v:8.1f}" for v in vals[:len(pipes)]) +
                 f"{vals[-3]:8.1f}{vals[-2]:7.1f}{us:8.1f}")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
