export TQ_LIB_PATH=$PWD/paper_2605_09281_b200/libtileq_b200_tq_wait_trap.so
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "forward_matches or paths_match or launch_count" > gpurun_out/p10_trap.log 2>&1; echo "parity trap rc=$?"; tail -3 gpurun_out/p10_trap.log
unset TQ_LIB_PATH
timeout 120 python tools/gpu_gemm_time.py c2 1 2 4 8 16 32 64 2>&1 | grep gemm
export TQ_LIB_PATH=$PWD/paper_2605_09281_b200/libtileq_b200_tq_dec_trace.so
timeout 120 python tools/dec_trace.py c2 1 64 5 > gpurun_out/p10_trace.log 2>&1; echo rc=$?
