#!/usr/bin/env bash
# One GPU-box pass: parity tests, smoke, bench, ncu launch list + one full
# capture of the engine kernel. Everything lands in gpurun_out/.
#   gpurun --timeout 2400 -- bash tools/gpu_round.sh [tag]
set -u
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi > "$OUT/nvidia-smi.txt" 2>&1
nproc > "$OUT/nproc.txt"
timeout 1200 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/smoke.log"
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?" >> "$OUT/bench.err"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file "$OUT/launches.csv" python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-sweeps \
  > "$OUT/ncu_launch_bench.log" 2>&1
timeout 1500 $NCU --set full --clock-control none --import-source on -k regex:engine_kernel -s 1 -c 1 \
  -o "$OUT/engine_full" -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-sweeps \
  > "$OUT/ncu_full.log" 2>&1
timeout 1200 python tools/bench_configs.py > "$OUT/configs.jsonl" 2> "$OUT/configs.err"
echo done > "$OUT/DONE"
