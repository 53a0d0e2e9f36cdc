TQ_STRESS_REPS=60 timeout 600 python -m pytest tests/test_gpu_shapes.py -x -q -k stress 2>&1 | tail -2 | sed "s/^/default: /"
TQ_LIB_PATH=$PWD/paper_2605_09281_b200/libtileq_b200_tq_route_no256.so TQ_STRESS_REPS=60 timeout 600 python -m pytest tests/test_gpu_shapes.py -x -q -k stress 2>&1 | tail -2 | sed "s/^/no256: /"
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "slab" 2>&1 | tail -2
