for i in 1 2 3 4; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/p23_bench$i.log 2>&1; echo "bench $i rc=$? $(grep -m1 'Error' gpurun_out/p23_bench$i.log)"
done
REPRO_CHECK=1 REPRO_STEPS=100 timeout 300 python tools/gpu_bench_repro.py > gpurun_out/p23_repro.log 2>&1; echo "repro rc=$?"; grep -m5 "nonzero\|Error" gpurun_out/p23_repro.log
