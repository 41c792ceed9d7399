# Phase profiles at rank 10 / 20 and the ncu launch list of the first 2500 iterations.
for K0 in 5000 26000; do timeout 600 python tools/gpu_prof_late.py 1 $K0 100 2>&1 | tail -20; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/launches.csv python tools/ncu_target.py 1 2500 > gpurun_out/ncu.log 2>&1; echo "ncu exit $?"
python tools/ncu_launch_summary.py gpurun_out/launches.csv > gpurun_out/launch_summary.txt 2>&1; head -8 gpurun_out/launch_summary.txt
