CUDA_LAUNCH_BLOCKING=1 TQ_STRESS_REPS=30 timeout 600 python -m pytest tests/test_gpu_shapes.py -x -q -k stress 2>&1 | grep -E "^E |^>|test_gpu_shapes.py:[0-9]+" | head -12
TQ_STRESS_REPS=30 timeout 600 python -m pytest tests/test_gpu_shapes.py -x -q -k stress 2>&1 | grep -E "^>|test_gpu_shapes.py:[0-9]+" | head -5
