for B in 700 300 128 65; do
CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/gpu_one.py c5 general $B 2>&1 | grep -E "^ok|Error" | head -2 | sed "s/^/B=$B /"
done
CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/gpu_one.py c5 folded 700 2>&1 | grep -E "^ok|Error" | head -2 | sed "s/^/folded /"
CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/gpu_one.py c4 general 700 2>&1 | grep -E "^ok|Error" | head -2 | sed "s/^/c4 general /"
