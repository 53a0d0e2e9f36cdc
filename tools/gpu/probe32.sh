for i in 1 2 3; do SR_B="1 64" timeout 120 python tools/gpu_stress_repro.py 2>&1 | grep -E "ok|Error" | tail -2 | sed "s/^/B<=64 run $i: /"; done
for i in 1 2; do SR_B="1 64" TQ_GRAPHS=0 timeout 120 python tools/gpu_stress_repro.py 2>&1 | grep -E "ok|Error" | tail -1 | sed "s/^/B<=64 nographs $i: /"; done
for i in 1 2; do SR_B="1 64" SR_P=1024 timeout 120 python tools/gpu_stress_repro.py 2>&1 | grep -E "ok|Error" | tail -1 | sed "s/^/B<=64 P=1024 $i: /"; done
for i in 1 2; do SR_B="64" SR_PATHS=full timeout 120 python tools/gpu_stress_repro.py 2>&1 | grep -E "ok|Error" | tail -1 | sed "s/^/B=64 full $i: /"; done
