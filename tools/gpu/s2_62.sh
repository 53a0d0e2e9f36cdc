SECONDS=0
timeout 900 python -m pytest tests/test_gpu_producer.py -q -x > gpurun_out/s2_62_tests.log 2>&1; echo "tests rc=$? wall ${SECONDS}s"; tail -2 gpurun_out/s2_62_tests.log
SECONDS=0; timeout 900 python tools/producer_bench.py --no-cpu > gpurun_out/s2_62_pb.log 2>&1; echo "pb c2 rc=$? ${SECONDS}s"; tail -1 gpurun_out/s2_62_pb.log
SECONDS=0; timeout 900 ncu --set full --clock-control none -k regex:"proxy_he|gptq_kernel|hinv_kernel|chol_update" -c 4 -o gpurun_out/s2_62_prod python tools/producer_bench.py --no-cpu --rows 2048 > gpurun_out/s2_62_ncu.log 2>&1; echo "ncu rc=$? ${SECONDS}s"; tail -2 gpurun_out/s2_62_ncu.log
