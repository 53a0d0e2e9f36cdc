#!/bin/bash
# CTA-0 traces with the TQ_TRACE build (flag 8 = record)
export TQ_LIB_PATH=$PWD/paper_2605_09281_b200/libtileq_b200_tq_experiment_tq_trace.so
for f in ${FLAGS:-8 235}; do
  TQ_DEBUG=$f TRACE_TAG=_t$f python tools/gpu_trace.py c2 1 64 > gpurun_out/trt_f$f.log 2>&1
done
