#!/usr/bin/env bash
# Same-box A/B of library variants on the full C4 placement search:
#   gpurun -- bash tools/gpu_ab_c4.sh TAG NAME...   (lib/ab/libloratwin_gpu_NAME.so; "head" = the in-tree build)
set -u
OUT=gpurun_out/$1; shift
mkdir -p "$OUT"
for r in 1 2; do
  for n in "$@"; do
    if [ "$n" = head ]; then unset LT_GPU_LIB; else export LT_GPU_LIB=paper_2508_08343_b200/lib/ab/libloratwin_gpu_$n.so; fi
    timeout 300 python bench.py --workload c4 --steps 1 --warmup 0 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$n', d['value'], d['ms_per_step'])" >> "$OUT/ab.log"
  done
done
echo done > "$OUT/DONE"
