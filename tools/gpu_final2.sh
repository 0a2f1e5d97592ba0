#!/usr/bin/env bash
# Final evidence without the sanitizers (closed on this pool): the -m gpu
# suite and smoke, engine ncu captures (C2, C5) copied into profiles/ before
# the bench lines that cite them, bench lines of every workload + the
# reference arm + the predictor comparison, the C2 launch list.
#   gpurun --timeout 5400 -- bash tools/gpu_final2.sh TAG
set -u
TAG=${1:-final}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
timeout 1200 python -m pytest tests -m gpu -q > "$OUT/pytest_gpu.log" 2>&1; echo "rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "rc=$?" >> "$OUT/smoke.log"
bash tools/gpu_ncu_engine.sh "$TAG/ncu" c2 c5
cp "$OUT/ncu/engine_ncu_c2.json" profiles/r2_engine_ncu_c2.json
cp "$OUT/ncu/engine_ncu_c5.json" profiles/r2_engine_ncu_c5.json
bash tools/gpu_bench_all.sh "$TAG/bench"
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file "$OUT/launches_c2.csv" python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-sweeps \
  > "$OUT/ncu_launch.log" 2>&1
echo done > "$OUT/DONE"
