SECONDS=0
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s2_1_tests.log 2>&1; echo "tests rc=$? wall ${SECONDS}s"; tail -3 gpurun_out/s2_1_tests.log
SECONDS=0; timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/s2_1_bench.log 2> gpurun_out/s2_1_bench.err; echo "bench rc=$? wall ${SECONDS}s"; tail -3 gpurun_out/s2_1_bench.err
timeout 300 python tools/prof_sweep.py c2 1 8 64 > gpurun_out/s2_1_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s2_1_launches_decode.csv python tools/prof_sweep.py c2 1 8 64 > gpurun_out/s2_1_ncu1.log 2>&1; echo "launches rc=$?"
