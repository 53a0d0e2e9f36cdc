timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/p3_bench.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
l=[x for x in open('gpurun_out/p3_bench.log') if x.startswith('{')][-1]; d=json.loads(l)
print("value", d["value"], "ms/step", d["ms_per_step"], "roof", d["roofline"]["frac"], d["roofline"]["avg_launch_ms"], "launches/fwd", d["gpu_launches_per_forward"])
for b,v in d["per_batch"].items(): print(b, round(v["us"],1), round(v["layer_hbm_frac"],3))
print("e2e", d["e2e"]["value"])
PY
timeout 300 python tools/gpu_gemm_time.py c2 1 2 4 8 16 32 64 > gpurun_out/p3_gemm.log 2>&1; cat gpurun_out/p3_gemm.log | tail -8
timeout 300 python tools/prof_sweep.py c2 1 8 64 > gpurun_out/p3_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/p3_launches.csv python tools/prof_sweep.py c2 1 8 64 > gpurun_out/p3_ncu.log 2>&1; echo "ncu rc=$?"
