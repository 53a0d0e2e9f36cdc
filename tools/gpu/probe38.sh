timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -s > gpurun_out/p38_gpu.log 2>&1; echo "gpu rc=$?"; tail -3 gpurun_out/p38_gpu.log; grep "stress:" gpurun_out/p38_gpu.log
for i in 1 2; do SR_REPS=0 SR_PN=60 timeout 300 python tools/gpu_stress_repro.py > gpurun_out/p38_$i.log 2>&1; echo "prefill60 $i: $(grep -E 'Error|ok' gpurun_out/p38_$i.log | tail -1)"; done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/p38_bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --workload prefill --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/p38_bench_pre.log 2>&1; echo "bench prefill rc=$?"
python - <<'PY'
import json
for f in ("gpurun_out/p38_bench.log", "gpurun_out/p38_bench_pre.log"):
    l=[x for x in open(f) if x.startswith('{')]
    if not l: print(f, "no json"); continue
    d=json.loads(l[-1])
    print(f, "value", round(d["value"]), "roof", round(d["roofline"]["frac"],3), "gemm_ms", round(d["roofline"]["avg_launch_ms"],4), "clk", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
    print({b: round(v["us"],1) for b,v in d["per_batch"].items()}, "e2e", round(d["e2e"]["value"]))
PY
