export TQ_LIB_PATH=$PWD/paper_2605_09281_b200/libtileq_b200_tq_route_trace.so; timeout 120 python tools/route_trace.py c2 1 8 > gpurun_out/s2_51_route.log 2>&1; echo route rc=$?
