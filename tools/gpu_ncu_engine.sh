#!/usr/bin/env bash
# ncu --set full capture of one engine launch per workload (first bench plan),
# with its iteration count, summarised into gpurun_out/TAG/engine_ncu_W.json.
#   gpurun -- bash tools/gpu_ncu_engine.sh TAG c2 c5 ...
set -u
TAG=$1; shift
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
NCU=/usr/local/cuda/bin/ncu
for W in "$@"; do
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:engine_kernel -s 1 -c 1 \
    -o "$OUT/engine_$W" -f python tools/profile_engine.py $W "$OUT/iters_$W.json" > "$OUT/ncu_full_$W.log" 2>&1
  python tools/ncu_summary.py "$OUT/engine_$W.ncu-rep" "$OUT/engine_ncu_$W.json" "$W first bench plan" \
    "ncu --set full --clock-control none --import-source on -k regex:engine_kernel -s 1 -c 1 python tools/profile_engine.py $W" \
    "$OUT/iters_$W.json" > /dev/null 2>&1
done
echo done > "$OUT/DONE"
