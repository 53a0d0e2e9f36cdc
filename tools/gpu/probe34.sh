export TQ_LIB_PATH=$PWD/paper_2605_09281_b200/libtileq_b200_tq_check_each.so
for i in 1 2 3 4 5 6 7 8; do SR_REPS=0 TQ_GRAPHS=0 timeout 120 python tools/gpu_stress_repro.py > gpurun_out/p34_$i.log 2>&1; echo "run $i: $(grep -E 'TQ_CHECK|prefill 3 ok' gpurun_out/p34_$i.log | head -2)"; done
