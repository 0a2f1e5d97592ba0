#!/usr/bin/env bash
# Same-box A/B of engine library variants (tools/build_variant.sh):
#   gpurun -- bash tools/gpu_ab.sh TAG NAME[@VARIANT]... [-- c3]
# NAME@V runs library NAME with LT_ENGINE_VARIANT=V.
set -u
OUT=gpurun_out/$1; shift
C3=0
ARGS=()
for a in "$@"; do [ "$a" = "c3" ] && C3=1 || ARGS+=("$a"); done
mkdir -p "$OUT"
for r in 1 2 3; do
  for nv in "${ARGS[@]}"; do
    n=${nv%@*}; v=1; [ "$nv" != "$n" ] && v=${nv#*@}
    L=paper_2508_08343_b200/lib/ab/libloratwin_gpu_$n.so
    echo "== $nv round $r" >> "$OUT/ab.log"
    export LT_GPU_LIB=$L LT_ENGINE_VARIANT=$v
    timeout 300 python tools/heavy_batch.py 2 >> "$OUT/ab.log" 2>&1
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-sweeps 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2 ms_per_step', round(d['ms_per_step'],3))" >> "$OUT/ab.log" 2>&1
    timeout 300 python tools/bench_configs.py c5 --c5-count 8192 --no-ref 2>/dev/null \
      | python -c "import json,sys; [print('C5', round(json.loads(l)['device_ms'],2)) for l in sys.stdin]" >> "$OUT/ab.log" 2>&1
    if [ $C3 = 1 ]; then
      timeout 300 python tools/bench_configs.py c3 --no-ref 2>/dev/null \
        | python -c "import json,sys; [print('C3', round(json.loads(l)['device_ms'],1)) for l in sys.stdin]" >> "$OUT/ab.log" 2>&1
    fi
  done
done
unset LT_GPU_LIB LT_ENGINE_VARIANT
echo done > "$OUT/DONE"
