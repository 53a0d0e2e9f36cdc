TQ_STRESS_REPS=2 timeout 900 compute-sanitizer --tool memcheck --show-backtrace no --print-limit 5 python -m pytest tests/test_gpu_shapes.py -x -q -k stress > gpurun_out/s2_33_memcheck.log 2>&1; echo "rc=$?"
grep -E "Invalid|at 0x|by thread|Address|of size|kernel" gpurun_out/s2_33_memcheck.log | head -30
