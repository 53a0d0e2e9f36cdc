nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader
SECONDS=0; timeout 900 python tools/producer_bench.py --no-cpu > gpurun_out/s2_75_pb.log 2>&1; echo "pb rc=$? ${SECONDS}s"; tail -1 gpurun_out/s2_75_pb.log
SECONDS=0; timeout 900 python tools/load_bench.py > gpurun_out/s2_75_load.log 2>&1; echo "load rc=$? ${SECONDS}s"; tail -1 gpurun_out/s2_75_load.log
