#!/usr/bin/env bash
# Engine change check: GPU parity, full C2 parity, critical-path engines,
# C2 bench (no CPU leg) and the C3/C4/C5 configs (no CPU samples).
#   gpurun --timeout 1800 -- bash tools/gpu_check.sh TAG
set -u
OUT=gpurun_out/${1:-check}
mkdir -p "$OUT"
timeout 900 python -m pytest tests -m gpu -x -q > "$OUT/pytest.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest.log"
timeout 300 python tools/c2_full_parity.py > "$OUT/c2_parity.log" 2>&1
timeout 300 python tools/heavy_batch.py 2 > "$OUT/heavy.log" 2>&1
timeout 600 python bench.py --no-cpu-baseline > "$OUT/bench.json" 2> "$OUT/bench.err"
timeout 600 python tools/bench_configs.py c3 c4 c5 --no-ref > "$OUT/cfg.jsonl" 2> "$OUT/cfg.err"
echo done > "$OUT/DONE"
