mkdir -p gpurun_out/st1
for v in 0 1; do LT_STAGED=$v timeout 600 python bench.py --no-cpu-baseline --no-sweeps --steps 5 --warmup 3 > gpurun_out/st1/bench_$v.json 2> gpurun_out/st1/bench_$v.err; done
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/st1/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-sweeps > /dev/null 2>&1
