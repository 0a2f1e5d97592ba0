#!/usr/bin/env bash
# Bench lines of every workload on one B200 + the predictor comparison:
#   gpurun --timeout 3600 -- bash tools/gpu_bench_all.sh TAG
set -u
OUT=gpurun_out/${1:-bench}
mkdir -p "$OUT"
nproc > "$OUT/nproc.txt"
timeout 900 python bench.py > "$OUT/bench_c2.json" 2> "$OUT/bench_c2.err"; echo "rc=$?" >> "$OUT/bench_c2.err"
timeout 600 python bench.py --workload c1 > "$OUT/bench_c1.json" 2> "$OUT/bench_c1.err"; echo "rc=$?" >> "$OUT/bench_c1.err"
timeout 900 python bench.py --workload c5 --steps 2 --warmup 1 > "$OUT/bench_c5.json" 2> "$OUT/bench_c5.err"; echo "rc=$?" >> "$OUT/bench_c5.err"
timeout 1200 python bench.py --workload c4 --steps 1 --warmup 0 > "$OUT/bench_c4.json" 2> "$OUT/bench_c4.err"; echo "rc=$?" >> "$OUT/bench_c4.err"
timeout 900 python bench.py --workload c3 --steps 2 --warmup 1 > "$OUT/bench_c3.json" 2> "$OUT/bench_c3.err"; echo "rc=$?" >> "$OUT/bench_c3.err"
timeout 900 python tools/bench_predictor.py > "$OUT/predictor.jsonl" 2> "$OUT/predictor.err"; echo "rc=$?" >> "$OUT/predictor.err"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > "$OUT/bench_ref.json" 2> "$OUT/bench_ref.err"
echo done > "$OUT/DONE"
