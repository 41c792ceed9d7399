for v in var_g3 var_g6; do PDSDP_B200_LIB=$PWD/build/$v.so timeout 400 python tools/gpu_variant_sweep.py 3 100000 nowarm 2>&1 | tail -1; done | tee gpurun_out/r02_cfg4_guard_full.txt
