SR_B="1" SR_REPS=1 SR_PN=120 timeout 600 python tools/gpu_stress_repro.py 2>&1 | tail -2 | sed "s/^/tile-router prefill: /"
SR_B="1" SR_REPS=1 SR_P=1000 SR_PN=200 timeout 600 python tools/gpu_stress_repro.py 2>&1 | tail -1 | sed "s/^/tile-router 1000: /"
timeout 900 python -m pytest tests/test_gpu_shapes.py tests/test_gpu_parity.py -x -q -k "prefill or route" 2>&1 | tail -2
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/s2_47_bench.log 2> gpurun_out/s2_47_bench.err; echo "bench rc=$?"; tail -2 gpurun_out/s2_47_bench.err
python - <<'PY'
import json
d=json.loads([x for x in open('gpurun_out/s2_47_bench.log') if x.startswith('{')][-1])
print("decode", round(d["value"]), "roof", round(d["roofline"]["frac"],3), "e2e", round(d["e2e"]["value"]), d["clocks"])
print({k: round(v["us"],1) for k,v in d["per_batch"].items()})
p=d["prefill"]; print("prefill", round(p["value"]), "roof", round(p["roofline"]["frac"],3), "e2e", round(p["e2e"]["value"]))
PY
timeout 300 python tools/prof_sweep.py c2 4096 > gpurun_out/s2_47_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s2_47_launches_prefill.csv python tools/prof_sweep.py c2 4096 > gpurun_out/s2_47_ncu.log 2>&1; echo "launches rc=$?"
