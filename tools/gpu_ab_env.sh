#!/usr/bin/env bash
# Same-box A/B of runtime settings (environment assignments) by the engine /
# pipeline times of tools/engine_times.py, 3 interleaved rounds:
#   gpurun -- bash tools/gpu_ab_env.sh TAG "WORKLOADS" "NAME:VAR=V VAR2=W" ...
set -u
OUT=gpurun_out/$1; shift
W=$1; shift
mkdir -p "$OUT"
for r in 1 2 3; do
  for spec in "$@"; do
    name=${spec%%:*}; envs=${spec#*:}
    env $envs timeout 300 python tools/engine_times.py $W 2>/dev/null | sed "s/^/$name /" >> "$OUT/ab.log"
  done
done
echo done > "$OUT/DONE"
