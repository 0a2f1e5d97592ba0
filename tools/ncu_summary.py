"""Summarise one `ncu --set full` capture of the engine kernel into
profiles/<tag>_engine_ncu.json (read back by bench.py for roofline.traffic).

    python tools/ncu_summary.py <report.ncu-rep> <out.json> <workload text> <command text> [iters.json]

iters.json (tools/profile_engine.py) adds the profiled launch's engine-iterations.
"""
import csv
import io
import json
import subprocess
import sys

rep, outp, workload, command = sys.argv[1:5]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]


def g(n):
    return float(v[h.index(n)])


keys = ["gpu__time_duration.sum", "dram__bytes.sum.per_second", "sm__inst_issued.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__average_warp_latency_per_inst_issued.ratio",
        "smsp__inst_executed.sum", "launch__grid_size", "launch__registers_per_thread",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct"]
stall = [n for n in h if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")]
rd = g("dram__bytes_read.sum") * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u[h.index("dram__bytes_read.sum")]]
wr = g("dram__bytes_write.sum") * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u[h.index("dram__bytes_write.sum")]]
d = {"kernel": "engine_kernel", "command": command, "workload": workload,
     "dram_bytes_per_launch": rd + wr, "dram_bytes_read": rd, "dram_bytes_write": wr,
     "metrics": {k: (g(k), u[h.index(k)]) for k in keys if k in h},
     "stalls_per_issue": {n[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]: g(n)
                          for n in stall if g(n) > 0.001}}
if len(sys.argv) > 5:
    it = json.load(open(sys.argv[5]))
    d["engine_iterations"] = it["engine_iterations"]
    d["plan"] = it["plan"]
json.dump(d, open(outp, "w"), indent=1)
print(json.dumps(d, indent=1))
