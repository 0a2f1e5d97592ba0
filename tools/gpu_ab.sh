#!/usr/bin/env bash
# Same-box A/B of engine library variants (tools/build_variant.sh):
#   gpurun -- bash tools/gpu_ab.sh TAG NAME...
set -u
OUT=gpurun_out/$1; shift
mkdir -p "$OUT"
for r in 1 2 3; do
  for n in "$@"; do
    L=paper_2508_08343_b200/lib/ab/libloratwin_gpu_$n.so
    echo "== $n round $r" >> "$OUT/ab.log"
    LT_GPU_LIB=$L timeout 300 python tools/heavy_batch.py 2 >> "$OUT/ab.log" 2>&1
    LT_GPU_LIB=$L timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-sweeps 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2 ms_per_step', round(d['ms_per_step'],3))" >> "$OUT/ab.log" 2>&1
    LT_GPU_LIB=$L timeout 300 python tools/bench_configs.py c5 --c5-count 8192 --no-ref 2>/dev/null \
      | python -c "import json,sys; [print('C5', round(json.loads(l)['device_ms'],2)) for l in sys.stdin]" >> "$OUT/ab.log" 2>&1
  done
done
echo done > "$OUT/DONE"
