export TQ_LIB_PATH=$PWD/paper_2605_09281_b200/libtileq_b200_tq_route_trace.so; timeout 120 python tools/route_trace.py c2 1 > gpurun_out/p17.log 2>&1; cat gpurun_out/p17.log
