SECONDS=0
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s2_89_tests.log 2>&1; echo "tests rc=$? wall ${SECONDS}s"; tail -3 gpurun_out/s2_89_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
SECONDS=0; timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/s2_89_bench.log 2> gpurun_out/s2_89_bench.err; echo "bench rc=$? wall ${SECONDS}s"; tail -2 gpurun_out/s2_89_bench.err
python - <<'PY'
import json
d=json.loads([x for x in open('gpurun_out/s2_89_bench.log') if x.startswith('{')][-1])
print("decode", round(d["value"]), "roof", round(d["roofline"]["frac"],3), "e2e", round(d["e2e"]["value"]), d["clocks"], "launches", d.get("gpu_launches"), d.get("gpu_launches_per_forward"))
print({k: round(v["us"],1) for k,v in d["per_batch"].items()})
p=d["prefill"]; print("prefill", round(p["value"]), "roof", round(p["roofline"]["frac"],3), "e2e", round(p["e2e"]["value"]))
PY
