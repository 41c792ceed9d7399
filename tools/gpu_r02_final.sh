# Round-2 measurement pass: smoke, both bench arms, ncu launch list, full captures.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_bench_reference_arm.json 2> gpurun_out/r02_bench_reference_arm.err; echo "ref exit $?"
timeout 1800 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_cfg2.json 2> gpurun_out/r02_bench_cfg2.err; echo "bench exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches.csv python tools/ncu_target.py 1 2500 > gpurun_out/ncu.log 2>&1; echo "ncu list exit $?"
python tools/ncu_launch_summary.py gpurun_out/r02_launches.csv > gpurun_out/r02_ncu_launches_cfg2_2500it.txt 2>&1; head -12 gpurun_out/r02_ncu_launches_cfg2_2500it.txt
for K0 in 5000 28000; do
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:lrpdhg_iterate -c 1 -o gpurun_out/r02_iter_k$K0 -f python tools/ncu_late.py 1 $K0 > gpurun_out/ncu_full_$K0.log 2>&1; echo "ncu full $K0 exit $?"
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2500 --csv --log-file gpurun_out/r02_dense_path_metrics.csv python tools/ncu_dense_target.py 2048 > gpurun_out/ncu_dense.log 2>&1; echo "ncu dense exit $?"
python tools/ncu_dense_summary.py gpurun_out/r02_dense_path_metrics.csv > gpurun_out/r02_dense_path_hbm.txt 2>&1; cat gpurun_out/r02_dense_path_hbm.txt
