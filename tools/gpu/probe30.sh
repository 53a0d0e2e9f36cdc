timeout 900 python -m pytest tests/test_gpu_shapes.py -x -q -s -p no:cacheprovider -k stress > gpurun_out/p30.log 2>&1; echo "rc=$?"; tail -4 gpurun_out/p30.log
