#!/bin/bash
# try_wait (suspending) vs test_wait (spinning) mbarrier waits
export TQ_LIB_PATH=$PWD/paper_2605_09281_b200/libtileq_b200_tq_spin_wait.so
for f in 8 235 40; do
  TQ_DEBUG=$f TRACE_TAG=_spin_f$f python tools/gpu_trace.py c2 1 64 > gpurun_out/trs_f$f.log 2>&1
done
python tools/gpu_perf.py c2 > gpurun_out/perf_spin.log 2>&1
