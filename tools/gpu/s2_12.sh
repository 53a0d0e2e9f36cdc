timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
export TQ_LIB_PATH=$PWD/paper_2605_09281_b200/libtileq_b200_tq_dec_trace.so; timeout 120 python tools/dec_trace.py c2 1 64 5 > gpurun_out/s2_12_dec.log 2>&1; echo dec rc=$?
