CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/gpu_fwd_sweep.py c2 1 2 4 8 16 32 64 2>&1 | tail -12
