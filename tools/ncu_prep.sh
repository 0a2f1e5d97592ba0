mkdir -p gpurun_out/n1
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"count_kernel|gather_kernel|seed_kernel|tables_draw" -c 4 \
  -o gpurun_out/n1/prep -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-sweeps > gpurun_out/n1/ncu.log 2>&1
