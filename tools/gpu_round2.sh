#!/usr/bin/env bash
# One GPU-box pass: all GPU tests, smoke, the C2 bench line (+ reference arm),
# the C5 full sweep line, ncu launch list of C2, engine ncu captures of C2 and
# C5 (first bench plan) with their iteration counts, and the C4 full search.
#   gpurun --timeout 3600 -- bash tools/gpu_round2.sh TAG [skip-c4]
set -u
TAG=${1:-r2}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
NCU=/usr/local/cuda/bin/ncu
nproc > "$OUT/nproc.txt"
timeout 1200 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.log"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/smoke.log"
timeout 900 python bench.py > "$OUT/bench_c2.json" 2> "$OUT/bench_c2.err"; echo "rc=$?" >> "$OUT/bench_c2.err"
timeout 900 python bench.py --workload c5 --steps 2 --warmup 1 > "$OUT/bench_c5.json" 2> "$OUT/bench_c5.err"; echo "rc=$?" >> "$OUT/bench_c5.err"
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file "$OUT/launches_c2.csv" python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-sweeps \
  > "$OUT/ncu_launch.log" 2>&1
for W in c2 c5; do
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:engine_kernel -s 1 -c 1 \
    -o "$OUT/engine_$W" -f python tools/profile_engine.py $W "$OUT/iters_$W.json" > "$OUT/ncu_full_$W.log" 2>&1
  python tools/ncu_summary.py "$OUT/engine_$W.ncu-rep" "$OUT/engine_ncu_$W.json" "$W first bench plan" \
    "ncu --set full --clock-control none --import-source on -k regex:engine_kernel -s 1 -c 1 python tools/profile_engine.py $W" \
    "$OUT/iters_$W.json" > /dev/null 2>&1
done
if [ "${2:-}" != "skip-c4" ]; then
  timeout 1500 python bench.py --workload c4 --steps 1 --warmup 0 > "$OUT/bench_c4.json" 2> "$OUT/bench_c4.err"; echo "rc=$?" >> "$OUT/bench_c4.err"
fi
echo done > "$OUT/DONE"
