timeout 300 python tools/gpu_determinism.py c2 64 65 100 128 200 256 > gpurun_out/p29.log 2>&1; cat gpurun_out/p29.log | tail -8
