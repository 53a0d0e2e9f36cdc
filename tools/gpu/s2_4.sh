timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "K6 or K4" 2>&1 | tail -25
export TQ_LIB_PATH=$PWD/paper_2605_09281_b200/libtileq_b200_tq_route_trace.so; timeout 120 python tools/route_trace.py c2 1 8 64 > gpurun_out/s2_4_route.log 2>&1; echo route rc=$?
export TQ_LIB_PATH=$PWD/paper_2605_09281_b200/libtileq_b200_tq_dec_trace.so; timeout 120 python tools/dec_trace.py c2 1 64 5 > gpurun_out/s2_4_dec.log 2>&1; echo dec rc=$?
