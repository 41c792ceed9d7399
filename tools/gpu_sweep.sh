for v in "$@"; do PDSDP_B200_LIB=build/$v.so timeout 300 python tools/gpu_variant_sweep.py 1 2>&1 | tail -1; done
