TQ_GRAPHS=0 TQ_LIB_PATH=$PWD/paper_2605_09281_b200/libtileq_b200_tq_check_each.so timeout 120 python tools/gpu_gemm_time.py c2 8 32 64 2>&1 | tail -4
timeout 120 python tools/gpu_gemm_time.py c2 1 8 32 64 2>&1 | tail -4
