SECONDS=0
timeout 900 python -m pytest tests/test_gpu_producer.py -q -x > gpurun_out/s2_65_tests.log 2>&1; echo "tests rc=$? wall ${SECONDS}s"; tail -2 gpurun_out/s2_65_tests.log
SECONDS=0; timeout 900 python tools/producer_bench.py --no-cpu > gpurun_out/s2_65_pb.log 2>&1; echo "pb c2 rc=$? ${SECONDS}s"; tail -1 gpurun_out/s2_65_pb.log
