timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py -x -q -k "not stress and not prefill_shapes" 2>&1 | tail -2
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/s2_22_bench.log 2> gpurun_out/s2_22_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads([x for x in open('gpurun_out/s2_22_bench.log') if x.startswith('{')][-1])
print("decode", round(d["value"]), "roof", round(d["roofline"]["frac"],3), "e2e", round(d["e2e"]["value"]))
print({k: round(v["us"],1) for k,v in d["per_batch"].items()})
p=d["prefill"]; print("prefill", round(p["value"]), "roof", round(p["roofline"]["frac"],3))
PY
timeout 300 python tools/prof_sweep.py c2 1 8 64 > gpurun_out/s2_22_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2_22_launches.csv python tools/prof_sweep.py c2 1 8 64 > gpurun_out/s2_22_ncu.log 2>&1; echo "launches rc=$?"
