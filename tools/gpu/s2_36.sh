for t in 1 2; do
SCAN_PATHS=full timeout 300 python tools/gpu_stress_scan.py 2>&1 | tail -2 | sed "s/^/full: /"
SCAN_BATCHES=1,2,4,8,16,32,33,48,64 timeout 300 python tools/gpu_stress_scan.py 2>&1 | tail -2 | sed "s/^/le64: /"
done
