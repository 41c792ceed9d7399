timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python tools/ncu_target.py 1 2500 > gpurun_out/ncu.log 2>&1; echo "ncu list exit $?"
python tools/ncu_launch_summary.py gpurun_out/launches.csv > gpurun_out/launch_summary.txt 2>&1
for K0 in 5000 28000; do
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:lrpdhg_iterate -c 1 -o gpurun_out/iter_k$K0 -f python tools/ncu_late.py 1 $K0 > gpurun_out/ncu_full_$K0.log 2>&1; echo "ncu full $K0 exit $?"
done
