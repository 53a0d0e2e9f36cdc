timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -8
timeout 900 python -m pytest tests/test_gpu_shapes.py -x -q -k decode_shapes 2>&1 | tail -8
timeout 120 python tools/gpu_gemm_time.py c2 1 2 8 16 32 64 2>&1 | tail -8
timeout 300 ./integration/_build/test_gpu_shim 2>&1 | tail -8
