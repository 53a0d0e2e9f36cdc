timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shapes.py -x -q -k "decode or forward_matches or stress or given or route or ep_" 2>&1 | tail -2
for t in 1 2 3; do SCAN_BATCHES=1,2,4,8,12,16,24,31,32,33,48,64 timeout 300 python tools/gpu_stress_scan.py 2>&1 | grep -E "done|Error:" | head -2 | sed "s/^/scan$t: /"; done
export TQ_LIB_PATH=$PWD/paper_2605_09281_b200/libtileq_b200_tq_route_trace.so; timeout 120 python tools/route_trace.py c2 1 > gpurun_out/s2_52_route.log 2>&1; unset TQ_LIB_PATH
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-prefill --no-cpu-baseline > gpurun_out/s2_52_bench.log 2> gpurun_out/s2_52_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads([x for x in open('gpurun_out/s2_52_bench.log') if x.startswith('{')][-1])
print("decode", round(d["value"]), "roof", round(d["roofline"]["frac"],3), d["clocks"])
print({k: round(v["us"],1) for k,v in d["per_batch"].items()})
PY
