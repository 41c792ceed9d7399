timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python tools/gpu_trace_ctas.py 1 29000 2 > gpurun_out/trace_r20.txt 2>&1
timeout 300 python tools/gpu_trace_ctas.py 1 20000 2 > gpurun_out/trace_r10.txt 2>&1
grep -A16 "transition totals" gpurun_out/trace_r20.txt; grep "total us" -A1 gpurun_out/trace_r20.txt gpurun_out/trace_r10.txt
