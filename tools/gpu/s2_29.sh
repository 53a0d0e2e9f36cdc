TQ_STRESS_REPS=60 timeout 600 python -m pytest tests/test_gpu_shapes.py -x -q -k stress 2>&1 | grep -E "^E |Error|assert|rep, B" | head -12
