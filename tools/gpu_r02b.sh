timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in var_g1 var_g3 var_g6 var_g10; do PDSDP_B200_LIB=$PWD/build/$v.so timeout 300 python tools/gpu_variant_sweep.py 3 8000 nowarm 2>&1 | tail -1; done | tee gpurun_out/r02_cfg4_guard_sweep.txt
bash tools/gpu_sanitize.sh cluster
