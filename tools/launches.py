"""Summarise an ncu --metrics gpu__time_duration.sum CSV (second half of the launches)."""
import csv, sys
lines = open(sys.argv[1]).read().splitlines()
start = [i for i,l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.DictReader(lines[start:]))
rows = [r for r in rows if r.get("Metric Name") == "gpu__time_duration.sum"]
for r in rows[len(rows)//2:]:
    n = r["Kernel Name"].split("(")[0][-50:]
    print(f'{n:50s} {r["Metric Value"]:>12} {r["Metric Unit"]}')
