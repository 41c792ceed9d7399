timeout 900 python -m pytest tests -m gpu -x -q -s 2>&1 | grep -v "^$" | tail -8
timeout 400 python tools/gpu_variant_sweep.py 3 100000 nowarm 2>&1 | tail -1 | cut -c1-330 | tee gpurun_out/r02_cfg4_adaptive.txt
