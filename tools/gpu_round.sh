timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for K0 in 2000 26000 29000; do timeout 300 python tools/gpu_prof_late.py 1 $K0 40 2>&1 | grep "n=2000"; done
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_hint.json 2>gpurun_out/bench_hint.err
python - <<'PY'
import json; d=json.load(open('gpurun_out/bench_hint.json'))
print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['iterate_kernel_us'], d['config']['iterations_per_solve'], d['config']['time_to_tol_s'], d['config']['eig_matvecs_per_iter'], d['config']['eig_passes_per_iter'])
PY
