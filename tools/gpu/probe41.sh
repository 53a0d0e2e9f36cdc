export TQ_LIB_PATH=$PWD/paper_2605_09281_b200/libtileq_b200_tq_dec_trace.so; timeout 120 python tools/dec_trace.py c2 1 64 5 > gpurun_out/p41.log 2>&1; echo rc=$?
