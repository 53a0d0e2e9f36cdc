SECONDS=0
timeout 900 python -m pytest tests/test_gpu_producer.py -q -x > gpurun_out/s2_96_tests.log 2>&1; echo "tests rc=$? wall ${SECONDS}s"; tail -2 gpurun_out/s2_96_tests.log
timeout 600 python tools/producer_bench.py --no-cpu --sketch '' > gpurun_out/s2_96_pb.log 2>&1; grep -o '"quantize_gptq_ms": [0-9.]*\|"proxy_loss_ms": [0-9.]*\|"spd_inverse_ms": [0-9.]*' gpurun_out/s2_96_pb.log
