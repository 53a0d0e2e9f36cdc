export TQ_LIB_PATH=$PWD/paper_2605_09281_b200/libtileq_b200_tq_route_trace.so
timeout 120 python tools/route_trace.py c2 1 64 > gpurun_out/p15_rtrace.log 2>&1; echo rc=$?; head -40 gpurun_out/p15_rtrace.log
