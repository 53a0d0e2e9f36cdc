SECONDS=0
timeout 600 python -m pytest tests/test_gpu_producer.py -q -x -k sketch > gpurun_out/s2_86_tests.log 2>&1; echo "tests rc=$? wall ${SECONDS}s"; tail -2 gpurun_out/s2_86_tests.log
timeout 600 python tools/producer_bench.py --no-cpu --rows 512 > gpurun_out/s2_86_pb.log 2>&1; grep -o '"sketch_lowrank_ms": [0-9.]*\|"sketch_gbs": [0-9.]*' gpurun_out/s2_86_pb.log
