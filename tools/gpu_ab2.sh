#!/usr/bin/env bash
# Same-box A/B of engine library variants by engine time of the first bench
# plan of C2 / C3 (heaviest plan) / C5 (tools/engine_times.py), 3 interleaved rounds:
#   gpurun -- bash tools/gpu_ab2.sh TAG NAME[@VARIANT]...
set -u
OUT=gpurun_out/$1; shift
mkdir -p "$OUT"
for r in 1 2 3; do
  for nv in "$@"; do
    n=${nv%@*}; v=; [ "$nv" != "$n" ] && v=${nv#*@}
    export LT_GPU_LIB=paper_2508_08343_b200/lib/ab/libloratwin_gpu_$n.so
    if [ -n "$v" ]; then export LT_ENGINE_VARIANT=$v; else unset LT_ENGINE_VARIANT; fi
    timeout 300 python tools/engine_times.py c2 c3 c5 2>/dev/null | sed "s/^/$nv /" >> "$OUT/ab.log"
  done
done
echo done > "$OUT/DONE"
