timeout 900 python -m pytest tests -m gpu -x -q -s 2>&1 | grep -E "^\[cfg|passed|failed|FAILED" | tee gpurun_out/r02_pytest_gpu_full_parity.txt
timeout 300 python tools/gpu_variant_sweep.py 1 100000 nowarm 2>&1 | tail -1 | cut -c1-250
timeout 900 python bench.py --workload cfg5 --instances 256 --steps 1 --warmup 0 > gpurun_out/r02_bench_cfg5_x256.json 2> gpurun_out/r02_bench_cfg5_x256.err; tail -c 900 gpurun_out/r02_bench_cfg5_x256.json; tail -3 gpurun_out/r02_bench_cfg5_x256.err
