SECONDS=0
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s2_88_tests.log 2>&1; echo "tests rc=$? wall ${SECONDS}s"; tail -3 gpurun_out/s2_88_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
SECONDS=0; timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/s2_88_bench.log 2> gpurun_out/s2_88_bench.err; echo "bench rc=$? wall ${SECONDS}s"; tail -2 gpurun_out/s2_88_bench.err
SECONDS=0; timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/s2_88_ref.log 2> gpurun_out/s2_88_ref.err; echo "ref rc=$? wall ${SECONDS}s"; tail -2 gpurun_out/s2_88_ref.err
python - <<'PY'
import json
d=json.loads([x for x in open('gpurun_out/s2_88_bench.log') if x.startswith('{')][-1])
print("decode", round(d["value"]), "roof", round(d["roofline"]["frac"],3), "e2e", round(d["e2e"]["value"]), d["clocks"], "launches", d.get("gpu_launches"))
print({k: round(v["us"],1) for k,v in d["per_batch"].items()})
p=d["prefill"]; print("prefill", round(p["value"]), "roof", round(p["roofline"]["frac"],3), "e2e", round(p["e2e"]["value"]), "cpu", p.get("cpu_baseline",{}).get("value"))
print("cpu", d["cpu_baseline"])
r=json.loads([x for x in open('gpurun_out/s2_88_ref.log') if x.startswith('{')][-1])
print("ref", r.get("value"), r.get("steps"), r.get("cpu_baseline"))
PY
SECONDS=0; TILEQ_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-prefill > gpurun_out/s2_88_ep2.log 2> gpurun_out/s2_88_ep2.err; echo "ep2 gloo rc=$? wall ${SECONDS}s"; tail -1 gpurun_out/s2_88_ep2.log | cut -c1-400; tail -3 gpurun_out/s2_88_ep2.err
