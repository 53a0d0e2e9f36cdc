#!/bin/bash
# mbarrier wait strategies: try_wait loop vs try_wait + nanosleep backoff
for v in tq_wait_backoff=64 tq_wait_backoff=256; do
  export TQ_LIB_PATH=$PWD/paper_2605_09281_b200/libtileq_b200_$v.so
  for f in 8 235; do
    TQ_DEBUG=$f TRACE_TAG=_${v}_f$f python tools/gpu_trace.py c2 1 64 > /dev/null 2>&1
  done
  python tools/gpu_perf.py c2 > gpurun_out/perf_$v.log 2>&1
done
