SECONDS=0
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s2_58_tests.log 2>&1; echo "tests rc=$? wall ${SECONDS}s"; tail -3 gpurun_out/s2_58_tests.log
