SECONDS=0; timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/p39_bench.log 2> gpurun_out/p39_bench.err; echo "bench rc=$? wall ${SECONDS}s"; tail -2 gpurun_out/p39_bench.err
SECONDS=0; timeout 1200 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/p39_ref.log 2> gpurun_out/p39_ref.err; echo "ref rc=$? wall ${SECONDS}s"; tail -2 gpurun_out/p39_ref.err
python - <<'PY'
import json
d=json.loads([x for x in open('gpurun_out/p39_bench.log') if x.startswith('{')][-1])
print("decode", round(d["value"]), "roof", round(d["roofline"]["frac"],3), "e2e", round(d["e2e"]["value"]), "clk", d["clocks"])
p=d["prefill"]; print("prefill", round(p["value"]), "roof", round(p["roofline"]["frac"],3), "e2e", round(p["e2e"]["value"]), "cpu", p.get("cpu_baseline",{}).get("value"))
print("cpu", d["cpu_baseline"])
r=json.loads([x for x in open('gpurun_out/p39_ref.log') if x.startswith('{')][-1])
print("ref", r["value"], r["steps"], r["cpu_baseline"]["cores"], r["cpu_baseline"].get("nproc"), r["cpu_baseline"].get("cpu_model"))
PY
