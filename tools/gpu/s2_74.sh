SECONDS=0; timeout 1700 python tools/producer_bench.py --cpu-rows 2 > gpurun_out/s2_74_pb.log 2>&1; echo "pb rc=$? ${SECONDS}s"; tail -1 gpurun_out/s2_74_pb.log
