TILEQ_SHIM_DEBUG=1 timeout 300 ./integration/_build/test_gpu_shim 2>&1 | grep -v "cached" | tail -20
