timeout 300 python tools/gpu_stress_scan.py 2>&1 | tail -8 | sed "s/^/all: /"
SCAN_PATHS=full timeout 300 python tools/gpu_stress_scan.py 2>&1 | tail -4 | sed "s/^/full: /"
SCAN_BATCHES=1,2,4,8,16,32,33,48,64 timeout 300 python tools/gpu_stress_scan.py 2>&1 | tail -4 | sed "s/^/le64: /"
SCAN_BATCHES=65,100,128,200,256 timeout 300 python tools/gpu_stress_scan.py 2>&1 | tail -4 | sed "s/^/gt64: /"
