set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --workload cfg5 --instances 32 --steps 1 --warmup 0 > gpurun_out/r02_cfg5_x32_slots.json 2> gpurun_out/r02_cfg5_x32_slots.err; tail -c 1200 gpurun_out/r02_cfg5_x32_slots.json; tail -3 gpurun_out/r02_cfg5_x32_slots.err
PDSDP_B200_LIB=$PWD/paper_1810_05231_b200/libpdsdp_b200_trace.so timeout 300 python tools/gpu_trace_ctas.py 1 20000 400 > gpurun_out/r02_trace_r10.txt 2>&1; tail -45 gpurun_out/r02_trace_r10.txt
