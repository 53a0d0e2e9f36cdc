cd tools/micro; timeout 60 ./hmma_dq 2>&1 | tail -14; cd ../..
timeout 120 python tools/gpu_gemm_time.py c2 1 8 64 2>&1 | tail -5
TQ_GRAPHS=0 timeout 300 ./integration/_build/test_gpu_shim 2>&1 | tail -12
timeout 300 ./integration/_build/test_gpu_shim 2>&1 | tail -12
