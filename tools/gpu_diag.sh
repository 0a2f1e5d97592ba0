#!/usr/bin/env bash
# Parity + per-scenario diagnostics on the GPU box (no profiler).
#   gpurun --timeout 1200 -- bash tools/gpu_diag.sh [tag]
set -u
TAG=${1:-diag}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 900 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python tools/c2_full_parity.py > "$OUT/c2_parity.log" 2>&1; echo "rc=$?" >> "$OUT/c2_parity.log"
timeout 300 python tools/diag_slow.py > "$OUT/diag_slow.log" 2>&1
[ -f paper_2508_08343_b200/lib/libloratwin_gpu_prof.so ] && timeout 300 python tools/diag_phase.py > "$OUT/diag_phase.log" 2>&1
timeout 300 python tools/heavy_batch.py 3 > "$OUT/heavy.log" 2>&1
timeout 600 python bench.py --no-cpu-baseline > "$OUT/bench.json" 2> "$OUT/bench.err"
echo done > "$OUT/DONE"
