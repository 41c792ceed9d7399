for v in var_g1 var_g3; do PDSDP_B200_LIB=$PWD/build/$v.so timeout 300 python tools/gpu_variant_sweep.py 4 100000 nowarm 2>&1 | tail -1 | cut -c1-330; done | tee gpurun_out/r02_cfg5_guard.txt
for v in var_cur var_d7 var_g3; do PDSDP_B200_LIB=$PWD/build/$v.so timeout 300 python tools/gpu_variant_sweep.py 1 100000 nowarm 2>&1 | tail -1 | cut -c1-330; done | tee gpurun_out/r02_cfg2_guard.txt
