#!/usr/bin/env bash
# Parity + launch list + bench (no cpu baseline) on the GPU box.
set -u
TAG=${1:-perf}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 900 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python tools/c2_full_parity.py > "$OUT/c2_parity.log" 2>&1; echo "rc=$?" >> "$OUT/c2_parity.log"
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-sweeps \
  > "$OUT/ncu_launch.log" 2>&1
timeout 600 python bench.py --no-cpu-baseline > "$OUT/bench.json" 2> "$OUT/bench.err"
echo done > "$OUT/DONE"
