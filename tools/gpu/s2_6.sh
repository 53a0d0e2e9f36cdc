timeout 300 python tools/gpu_given_diag.py 2>&1 | tail -30
