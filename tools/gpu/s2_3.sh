timeout 300 python tools/gpu_gate_diag2.py c1 folded 700 5 2>&1 | tail -12
timeout 900 python -m pytest tests/test_gpu_shapes.py -x -q -k "prefill" 2>&1 | tail -15
timeout 600 ./integration/_build/test_gpu_shim 2>&1 | tail -30
