SECONDS=0
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s2_46_tests.log 2>&1; echo "tests rc=$? wall ${SECONDS}s"; tail -3 gpurun_out/s2_46_tests.log
SECONDS=0; timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/s2_46_bench.log 2> gpurun_out/s2_46_bench.err; echo "bench rc=$? wall ${SECONDS}s"; tail -2 gpurun_out/s2_46_bench.err
python - <<'PY'
import json
d=json.loads([x for x in open('gpurun_out/s2_46_bench.log') if x.startswith('{')][-1])
print("decode", round(d["value"]), "roof", round(d["roofline"]["frac"],3), "e2e", round(d["e2e"]["value"]), d["clocks"])
print({k: round(v["us"],1) for k,v in d["per_batch"].items()})
p=d["prefill"]; print("prefill", round(p["value"]), "roof", round(p["roofline"]["frac"],3), "e2e", round(p["e2e"]["value"]))
PY
timeout 300 python tools/prof_sweep.py c2 1 8 64 > gpurun_out/s2_46_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s2_46_launches_decode.csv python tools/prof_sweep.py c2 1 8 64 > gpurun_out/s2_46_ncu1.log 2>&1; echo "launches rc=$?"
