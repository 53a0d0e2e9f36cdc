timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py tests/test_gpu_create.py -x -q -k "decode or forward_matches or stress or given or route or ep_ or create" 2>&1 | tail -2
for t in 1 2 3; do SCAN_BATCHES=1,2,4,8,12,16,24,31,32,33,48,64,100,256 timeout 300 python tools/gpu_stress_scan.py 2>&1 | grep -E "done|Error:" | head -2 | sed "s/^/scan$t: /"; done
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-prefill --no-cpu-baseline > gpurun_out/s2_53_bench.log 2> gpurun_out/s2_53_bench.err; echo "bench rc=$?"; tail -2 gpurun_out/s2_53_bench.err
python - <<'PY'
import json
d=json.loads([x for x in open('gpurun_out/s2_53_bench.log') if x.startswith('{')][-1])
print("decode", round(d["value"]), "roof", round(d["roofline"]["frac"],3), "e2e", round(d["e2e"]["value"]), d["clocks"])
print({k: round(v["us"],1) for k,v in d["per_batch"].items()})
PY
