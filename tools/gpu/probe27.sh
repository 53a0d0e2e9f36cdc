export TQ_LIB_PATH=$PWD/paper_2605_09281_b200/libtileq_b200_tq_wait_trap.so
CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/gpu_one.py c5 general 65 > gpurun_out/p27.log 2>&1; echo rc=$?; grep -E "TQ_WAIT|^ok|Error" gpurun_out/p27.log | head -8
unset TQ_LIB_PATH
for B in 65 300; do TQ_NO_XR=1 CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/gpu_one.py c2 general $B 2>&1 | grep -E "^ok|Error" | head -1 | sed "s/^/c2 general B=$B /"; done
