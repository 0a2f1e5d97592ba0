#!/usr/bin/env bash
# Focused ncu capture of the engine on the critical-path C2 engines.
set -u
TAG=${1:-heavy}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 300 python tools/heavy_batch.py 3 > "$OUT/heavy.log" 2>&1
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:engine_kernel -s 1 -c 1 \
  -o "$OUT/heavy_full" -f python tools/heavy_batch.py 2 > "$OUT/ncu.log" 2>&1
echo done > "$OUT/DONE"
