SECONDS=0
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_create.py tests/test_gpu_vq.py tests/test_gpu_layouts.py -q -x > gpurun_out/s2_69_tests.log 2>&1; echo "tests rc=$? wall ${SECONDS}s"; tail -3 gpurun_out/s2_69_tests.log
SECONDS=0; timeout 900 python tools/load_bench.py > gpurun_out/s2_69_load.log 2>&1; echo "load rc=$? ${SECONDS}s"; tail -1 gpurun_out/s2_69_load.log
SECONDS=0; timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/s2_69_bench.log 2> gpurun_out/s2_69_bench.err; echo "bench rc=$? ${SECONDS}s"; python -c "
import json; d=json.loads([x for x in open('gpurun_out/s2_69_bench.log') if x.startswith('{')][-1]); print(round(d['value']), round(d['roofline']['frac'],3), round(d['prefill']['value']))"
