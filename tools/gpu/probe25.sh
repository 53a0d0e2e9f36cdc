timeout 1500 python -m pytest tests/test_gpu_shapes.py -x -q -s -p no:cacheprovider > gpurun_out/p25_shapes.log 2>&1; echo "shapes rc=$?"
grep -E "rel_frob|passed|failed|Error|assert" gpurun_out/p25_shapes.log | head -40
