SECONDS=0
timeout 900 python -m pytest tests/test_gpu_producer.py tests/test_gpu_shim.py -q -x > gpurun_out/s2_68_tests.log 2>&1; echo "tests rc=$? wall ${SECONDS}s"; tail -3 gpurun_out/s2_68_tests.log
SECONDS=0; timeout 900 python tools/producer_bench.py --no-cpu > gpurun_out/s2_68_pb.log 2>&1; echo "pb c2 rc=$? ${SECONDS}s"; tail -1 gpurun_out/s2_68_pb.log
SECONDS=0; timeout 900 python tools/load_bench.py > gpurun_out/s2_68_load.log 2>&1; echo "load rc=$? ${SECONDS}s"; tail -1 gpurun_out/s2_68_load.log
