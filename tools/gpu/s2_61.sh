SECONDS=0
timeout 900 python -m pytest tests/test_gpu_producer.py -q -x > gpurun_out/s2_61_tests.log 2>&1; echo "tests rc=$? wall ${SECONDS}s"; tail -3 gpurun_out/s2_61_tests.log
SECONDS=0; timeout 900 python tools/producer_bench.py --no-cpu > gpurun_out/s2_61_pb.log 2>&1; echo "pb c2 rc=$? ${SECONDS}s"; tail -1 gpurun_out/s2_61_pb.log
SECONDS=0; timeout 1200 python tools/producer_bench.py --rows 512 --cpu-rows 2 > gpurun_out/s2_61_pb_cpu.log 2>&1; echo "pb cpu rc=$? ${SECONDS}s"; tail -1 gpurun_out/s2_61_pb_cpu.log
nproc; lscpu | grep "Model name"
