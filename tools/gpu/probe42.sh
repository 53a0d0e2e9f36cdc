timeout 120 python tools/gpu_gemm_time.py c2 1 8 32 64 2>&1 | grep gemm | sed "s/^/NI=4 /"
for n in 2 1; do TQ_LIB_PATH=$PWD/paper_2605_09281_b200/libtileq_b200_tq_dec_ni32=$n.so timeout 120 python tools/gpu_gemm_time.py c2 1 8 32 64 2>&1 | grep gemm | sed "s/^/NI=$n /"; done
