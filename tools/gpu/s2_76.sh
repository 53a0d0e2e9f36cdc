SECONDS=0
timeout 900 python -m pytest tests/test_gpu_producer.py -q -x > gpurun_out/s2_76_tests.log 2>&1; echo "tests rc=$? wall ${SECONDS}s"; tail -2 gpurun_out/s2_76_tests.log
timeout 600 python tools/producer_bench.py --no-cpu --sketch '' > gpurun_out/s2_76_pb1024.log 2>&1; echo "1024:"; grep -o '"quantize_gptq_ms": [0-9.]*' gpurun_out/s2_76_pb1024.log
TQ_LIB_PATH=$PWD/paper_2605_09281_b200/libtileq_b200_tq_gptq_threads=512.so timeout 600 python tools/producer_bench.py --no-cpu --sketch '' > gpurun_out/s2_76_pb512.log 2>&1; echo "512:"; grep -o '"quantize_gptq_ms": [0-9.]*' gpurun_out/s2_76_pb512.log
