mkdir -p gpurun_out/d12
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/d12/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/d12/pytest.log
timeout 300 python tools/c2_full_parity.py > gpurun_out/d12/c2_parity.log 2>&1
timeout 300 python tools/heavy_batch.py 2 > gpurun_out/d12/heavy.log 2>&1
timeout 300 python tools/diag_c4_phase.py > gpurun_out/d12/c4phase.log 2>&1
timeout 600 python tools/bench_configs.py c3 c4 --c4-conditions 256 > gpurun_out/d12/cfg.jsonl 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/d12/bench.json 2> gpurun_out/d12/bench.err
