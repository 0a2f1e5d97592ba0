#!/usr/bin/env bash
# One GPU-box pass for a change: the -m gpu suite, smoke, the C2 bench line,
# and (with "san") the compute-sanitizer runs.
#   gpurun --timeout 2400 -- bash tools/gpu_pass.sh TAG [san]
set -u
OUT=gpurun_out/${1:-pass}
mkdir -p "$OUT"
timeout 1200 python -m pytest tests -m gpu -q > "$OUT/pytest_gpu.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "rc=$?" >> "$OUT/smoke.log"
timeout 900 python bench.py --no-sweeps > "$OUT/bench_c2.json" 2> "$OUT/bench_c2.err"; echo "rc=$?" >> "$OUT/bench_c2.err"
if [ "${2:-}" = "san" ]; then bash tools/gpu_sanitize.sh "$(basename "$OUT")/san"; fi
echo done > "$OUT/DONE"
