#!/usr/bin/env bash
# Parity + e2e host timing breakdown.
set -u
TAG=${1:-e2e}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 900 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python tools/c2_full_parity.py > "$OUT/c2_parity.log" 2>&1; echo "rc=$?" >> "$OUT/c2_parity.log"
LT_HOST_TIMING=1 timeout 600 python bench.py --no-cpu-baseline --steps 3 --warmup 3 > "$OUT/bench.json" 2> "$OUT/bench.err"
echo done > "$OUT/DONE"
