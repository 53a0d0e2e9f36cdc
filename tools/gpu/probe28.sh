timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/p28_gpu.log 2>&1; echo "gpu rc=$?"; tail -3 gpurun_out/p28_gpu.log
timeout 1500 python -m pytest tests/test_gpu_shapes.py -x -q -s -p no:cacheprovider > gpurun_out/p28_shapes.log 2>&1; echo "shapes rc=$?"
grep -E "rel_frob|passed|failed|Error" gpurun_out/p28_shapes.log | tail -30
for i in 1 2; do timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/p28_bench$i.log 2>&1; echo "bench $i rc=$? $(grep -m1 'Error' gpurun_out/p28_bench$i.log)"; done
