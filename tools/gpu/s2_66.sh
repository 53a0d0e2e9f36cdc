SECONDS=0; timeout 1500 python tools/producer_bench.py --cpu-rows 2 > gpurun_out/s2_66_pb.log 2>&1; echo "pb rc=$? ${SECONDS}s"; tail -1 gpurun_out/s2_66_pb.log
