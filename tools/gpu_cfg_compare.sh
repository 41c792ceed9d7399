# Time to tolerance per config (1, 4, one config-5 instance) with two library builds.
for idx in 0 3 4; do for v in "$@"; do
  echo "cfg idx $idx $v: $(PDSDP_B200_LIB=build/$v.so timeout 600 python tools/gpu_variant_sweep.py $idx 2>&1 | tail -1)"
done; done
