SECONDS=0
timeout 900 python -m pytest tests/test_gpu_exp.py tests/test_gpu_parity.py tests/test_gpu_shim.py -q -s -x > gpurun_out/s2_56_tests.log 2>&1; echo "tests rc=$? wall ${SECONDS}s"; grep "exp vs glibc" gpurun_out/s2_56_tests.log; tail -3 gpurun_out/s2_56_tests.log
SECONDS=0; timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/s2_56_bench.log 2> gpurun_out/s2_56_bench.err; echo "bench rc=$? wall ${SECONDS}s"; tail -2 gpurun_out/s2_56_bench.err
python - <<'PY'
import json
d=json.loads([x for x in open('gpurun_out/s2_56_bench.log') if x.startswith('{')][-1])
print("decode", round(d["value"]), "roof", round(d["roofline"]["frac"],3), "e2e", round(d["e2e"]["value"]), d["clocks"], "launches", d.get("gpu_launches"))
print({k: round(v["us"],1) for k,v in d["per_batch"].items()})
p=d["prefill"]; print("prefill", round(p["value"]), "roof", round(p["roofline"]["frac"],3), "e2e", round(p["e2e"]["value"]))
PY
