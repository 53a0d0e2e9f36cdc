timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py -x -q -k "decode or forward_matches or stress" 2>&1 | tail -2
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-prefill --no-cpu-baseline > gpurun_out/s2_49_bench.log 2> gpurun_out/s2_49_bench.err; echo "bench rc=$?"; tail -2 gpurun_out/s2_49_bench.err
python - <<'PY'
import json
d=json.loads([x for x in open('gpurun_out/s2_49_bench.log') if x.startswith('{')][-1])
print("decode", round(d["value"]), "roof", round(d["roofline"]["frac"],3), d["clocks"])
print({k: round(v["us"],1) for k,v in d["per_batch"].items()})
PY
