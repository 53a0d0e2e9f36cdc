for t in 1 2 3 4 5; do
TQ_GRAPHS=0 TQ_LIB_PATH=$PWD/paper_2605_09281_b200/libtileq_b200_tq_check_each.so SCAN_PATHS=full SCAN_BATCHES=12,16,24,31,32 timeout 300 python tools/gpu_stress_scan.py 2>&1 | grep -E "CHECK|done|Error" | head -3 | sed "s/^/$t: /"
done
