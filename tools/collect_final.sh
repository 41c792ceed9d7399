#!/bin/bash
# After tools/gpu_r02_final.sh on the GPU box: turn gpurun_out/ into the committed profiles/r02_* files.
cd gpurun_out
for K in 5000 28000; do r=$([ $K = 5000 ] && echo 10 || echo 20)
  ncu -i r02_iter_k$K.ncu-rep --page details > ../profiles/r02_iterate_kernel_ncu_details_r$r.txt 2>/dev/null
  ncu -i r02_iter_k$K.ncu-rep --page raw --csv > ../profiles/r02_iterate_kernel_ncu_raw_r$r.csv 2>/dev/null
  python ../tools/ncu_lines.py r02_iter_k$K.ncu-rep 45 > ../profiles/r02_iterate_kernel_stall_lines_r$r.txt 2>/dev/null
done
cd ..
cp gpurun_out/r02_bench_cfg2.json gpurun_out/r02_bench_reference_arm.json gpurun_out/r02_ncu_launches_cfg2_2500it.txt gpurun_out/r02_dense_path_hbm.txt profiles/
tools/sass_summary.sh > profiles/r02_sass_opcode_summary.txt
