#!/usr/bin/env bash
# compute-sanitizer over tools/sanitize_batch.py (memcheck, racecheck, synccheck).
#   gpurun --timeout 2400 -- bash tools/gpu_sanitize.sh TAG
set -u
OUT=gpurun_out/${1:-san}
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
for T in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $T --target-processes all --print-limit 20 python tools/sanitize_batch.py \
    > "$OUT/$T.log" 2>&1
  echo "rc=$?" >> "$OUT/$T.log"
done
echo done > "$OUT/DONE"
