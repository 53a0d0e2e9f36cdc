for i in 1 2 3 4 5 6; do SR_REPS=0 timeout 120 python tools/gpu_stress_repro.py 2>&1 | grep -E "ok|Error" | tail -1 | sed "s/^/prefill only $i: /"; done
for i in 1 2 3; do SR_REPS=0 CUDA_LAUNCH_BLOCKING=1 TQ_GRAPHS=0 timeout 120 python tools/gpu_stress_repro.py 2>&1 | grep -E "ok|Error" | tail -1 | sed "s/^/prefill only blocking $i: /"; done
