timeout 300 python -m pytest tests/test_gpu_vq.py -x -q 2>&1 | grep -E "^E |FAILED|passed|failed|Error" | head -8
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/s2_26_bench.log 2> gpurun_out/s2_26_bench.err; echo "bench rc=$?"; tail -3 gpurun_out/s2_26_bench.err
python - <<'PY'
import json
d=json.loads([x for x in open('gpurun_out/s2_26_bench.log') if x.startswith('{')][-1])
print("decode", round(d["value"]), "roof", round(d["roofline"]["frac"],3), "e2e", round(d["e2e"]["value"]))
print({k: round(v["us"],1) for k,v in d["per_batch"].items()})
p=d["prefill"]; print("prefill", round(p["value"]), "roof", round(p["roofline"]["frac"],3))
PY
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s2_26_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s2_26_tests.log
