SECONDS=0
timeout 900 python -m pytest tests/test_gpu_producer.py -q -x -k sketch > gpurun_out/s2_73_tests.log 2>&1; echo "tests rc=$? wall ${SECONDS}s"; tail -2 gpurun_out/s2_73_tests.log
SECONDS=0; timeout 900 python tools/producer_bench.py --no-cpu --rows 1024 > gpurun_out/s2_73_pb.log 2>&1; echo "pb rc=$? ${SECONDS}s"; tail -1 gpurun_out/s2_73_pb.log
SECONDS=0; timeout 900 ncu --metrics gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/s2_73_launches.csv -k regex:"matvec|mattvec|norm2|deflate" python tools/producer_bench.py --no-cpu --rows 128 --dim 256 --tokens 64 --sketch-rank 2 > gpurun_out/s2_73_l.log 2>&1; echo "launches rc=$? ${SECONDS}s"
