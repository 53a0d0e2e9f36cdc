SECONDS=0
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shim.py tests/test_gpu_vq.py -q -x > gpurun_out/s2_57_tests.log 2>&1; echo "tests rc=$? wall ${SECONDS}s"; tail -3 gpurun_out/s2_57_tests.log
