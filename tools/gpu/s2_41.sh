timeout 300 python tools/gpu_given_scan.py 2>&1 | grep -E "ok|done|Error:" | tail -2 | sed "s/^/given-full: /"
SCAN_PATH=qmoe timeout 300 python tools/gpu_given_scan.py 2>&1 | grep -E "ok|done|Error:" | tail -2 | sed "s/^/given-qmoe: /"
timeout 300 python tools/gpu_counter_check.py 2>&1 | grep -vE "^ +" | head -3 | sed "s/^/routed-full: /"
