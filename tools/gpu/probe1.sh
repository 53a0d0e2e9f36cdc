set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for m in mma_tput dq_rate tmem_st tmem_contend mma_lat; do echo "== $m"; timeout 60 ./tools/micro/$m; done > gpurun_out/r2_micro.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest0.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench0.log 2>&1; echo "bench rc=$?"
tail -3 gpurun_out/r2_gputest0.log
