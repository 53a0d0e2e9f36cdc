export TQ_LIB_PATH=$PWD/paper_2605_09281_b200/libtileq_b200_tq_route_trace.so
timeout 120 python tools/route_trace.py c2 1 64 > gpurun_out/p16_rtrace.log 2>&1; echo rc=$?; head -20 gpurun_out/p16_rtrace.log; grep -A 12 "B=64" gpurun_out/p16_rtrace.log
unset TQ_LIB_PATH
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/p16_gputest.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/p16_gputest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/p16_bench.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
l=[x for x in open('gpurun_out/p16_bench.log') if x.startswith('{')][-1]; d=json.loads(l)
print("value", round(d["value"]), "roof", round(d["roofline"]["frac"],3), "gemm_ms", d["roofline"]["avg_launch_ms"], "clk", d["clocks"])
print({b: round(v["us"],1) for b,v in d["per_batch"].items()}, "e2e", round(d["e2e"]["value"]))
PY
