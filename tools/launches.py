"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv): per-kernel time of the last step."""
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10][1:]
eng = [i for i, r in enumerate(rows) if "engine_kernel" in r[4]]
start = eng[-2] + 1 if len(eng) >= 2 else 0
tot = collections.OrderedDict()
for r in rows[start:eng[-1] + 1]:
    name = r[4].split("(")[0].replace("void ", "")[:60]
    tot[name] = tot.get(name, 0) + float(r[-1]) / 1e6
for k, v in tot.items():
    print(f"{v:9.3f} ms  {k}")
print(f"{sum(tot.values()):9.3f} ms  total (one step)")
