for i in 1 2 3; do SR_REPS=0 SR_PN=60 timeout 300 python tools/gpu_stress_repro.py > gpurun_out/p36_$i.log 2>&1; echo "plain $i: $(grep -E 'Error|ok' gpurun_out/p36_$i.log | tail -1)"; done
export TQ_LIB_PATH=$PWD/paper_2605_09281_b200/libtileq_b200_tq_check_each.so
for i in 1 2 3; do SR_REPS=0 SR_PN=60 TQ_GRAPHS=0 timeout 300 python tools/gpu_stress_repro.py > gpurun_out/p36_c$i.log 2>&1; echo "check_each $i: $(grep -E 'TQ_CHECK|Error|ok' gpurun_out/p36_c$i.log | tail -1)"; done
