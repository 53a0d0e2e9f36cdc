timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | grep -E "^E |FAILED|passed|failed" | head -8
TQ_LIB_PATH=$PWD/paper_2605_09281_b200/libtileq_b200_tq_check_each.so timeout 120 python tools/gpu_gemm_time.py c2 8 32 64 2>&1 | tail -4
