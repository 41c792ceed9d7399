timeout 120 python -m pytest tests/test_gpu_parity.py -x -q -k "aproj_psd_matches_reference" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/gpu_prof_late.py 1 29000 300 2>&1 | head -3
timeout 300 python tools/gpu_prof_late.py 1 20000 300 2>&1 | head -3
