timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py -x -q -k "decode or forward_matches or stress or given" 2>&1 | tail -2
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-prefill --no-cpu-baseline > gpurun_out/s2_50_bench.log 2> gpurun_out/s2_50_bench.err; echo "bench rc=$?"; tail -2 gpurun_out/s2_50_bench.err
python - <<'PY'
import json
d=json.loads([x for x in open('gpurun_out/s2_50_bench.log') if x.startswith('{')][-1])
print("decode", round(d["value"]), "roof", round(d["roofline"]["frac"],3), d["clocks"])
print({k: round(v["us"],1) for k,v in d["per_batch"].items()})
PY
timeout 300 python tools/prof_sweep.py c2 1 8 64 > gpurun_out/s2_50_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s2_50_launches_decode.csv python tools/prof_sweep.py c2 1 8 64 > gpurun_out/s2_50_ncu.log 2>&1; echo "launches rc=$?"
