for t in 1 2 3 4 5 6; do
SCAN_PATHS=full SCAN_BATCHES=12,16,24,31,32 timeout 300 python tools/gpu_stress_scan.py 2>&1 | grep -E "done|Error:" | head -2 | sed "s/^/$t: /"
done
SCAN_BATCHES=33,48,63,64 timeout 300 python tools/gpu_stress_scan.py 2>&1 | grep -E "done|Error:" | head -2 | sed "s/^/33-64: /"
timeout 900 python -m pytest tests/test_gpu_shapes.py -x -q -k stress 2>&1 | tail -2
