for c in a96ea7f 8f9a1da; do (cd .bisect/$c && TQ_STRESS_REPS=60 timeout 600 python -m pytest tests/test_gpu_shapes.py -x -q -k stress 2>&1 | tail -2 | sed "s/^/$c: /"); done
