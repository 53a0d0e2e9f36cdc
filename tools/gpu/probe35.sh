for i in 1 2 3 4 5 6 7 8; do SR_REPS=0 timeout 120 python tools/gpu_stress_repro.py > gpurun_out/p35_$i.log 2>&1; echo "run $i: $(grep -E 'Error|prefill 3 ok' gpurun_out/p35_$i.log | head -1)"; done
for i in 1 2 3; do SR_B="1 64" timeout 120 python tools/gpu_stress_repro.py 2>&1 | grep -E "Error|prefill 3 ok" | head -1 | sed "s/^/decode+prefill $i: /"; done
