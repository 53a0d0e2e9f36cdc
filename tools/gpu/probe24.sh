for i in 1 2 3; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/p24_bench$i.log 2>&1; echo "minb1 bench $i rc=$? $(grep -m1 'Error' gpurun_out/p24_bench$i.log)"
done
