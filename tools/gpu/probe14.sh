timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/p14_gputest.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/p14_gputest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/p14_bench.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
l=[x for x in open('gpurun_out/p14_bench.log') if x.startswith('{')][-1]; d=json.loads(l)
print("value", round(d["value"]), "roof", round(d["roofline"]["frac"],3), "gemm_ms", d["roofline"]["avg_launch_ms"], "clk", d["clocks"])
print({b: round(v["us"],1) for b,v in d["per_batch"].items()}, "e2e", round(d["e2e"]["value"]))
PY
timeout 300 python tools/prof_sweep.py c2 1 8 64 > gpurun_out/p14_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p14_launches.csv python tools/prof_sweep.py c2 1 8 64 > gpurun_out/p14_ncu.log 2>&1; echo "ncu rc=$?"
