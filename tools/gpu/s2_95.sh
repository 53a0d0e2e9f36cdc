SECONDS=0; timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --no-prefill > gpurun_out/s2_95_bench.log 2> gpurun_out/s2_95_bench.err; echo "bench rc=$? wall ${SECONDS}s"; tail -2 gpurun_out/s2_95_bench.err
python - <<'PY'
import json
d=json.loads([x for x in open('gpurun_out/s2_95_bench.log') if x.startswith('{')][-1])
print("decode", round(d["value"]), "roof", round(d["roofline"]["frac"],3), "e2e", round(d["e2e"]["value"]))
print({k: round(v["us"],1) for k,v in d["per_batch"].items()})
PY
