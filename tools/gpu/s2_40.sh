timeout 300 python tools/gpu_counter_check.py 2>&1 | grep -vE "^ +" | head -12
SCAN_PATH=lotile timeout 300 python tools/gpu_counter_check.py 2>&1 | grep -vE "^ +" | head -6 | sed "s/^/lotile: /"
