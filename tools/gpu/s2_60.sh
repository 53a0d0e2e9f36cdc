SECONDS=0
timeout 900 python -m pytest tests/test_gpu_producer.py -q -x > gpurun_out/s2_60_tests.log 2>&1; echo "tests rc=$? wall ${SECONDS}s"; tail -15 gpurun_out/s2_60_tests.log
SECONDS=0; timeout 600 python tools/producer_bench.py --rows 2048 --dim 1024 --tokens 256 --cpu-rows 4 > gpurun_out/s2_60_pb_small.log 2>&1; echo "pb small rc=$? ${SECONDS}s"; tail -3 gpurun_out/s2_60_pb_small.log
SECONDS=0; timeout 900 python tools/producer_bench.py --no-cpu > gpurun_out/s2_60_pb.log 2>&1; echo "pb c2 rc=$? ${SECONDS}s"; tail -3 gpurun_out/s2_60_pb.log
