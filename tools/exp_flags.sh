#!/bin/bash
# pipeline experiments: CTA-0 traces of the B=1 / B=64 expert GEMM under TQ_DEBUG flag sets
for f in 8 40 43 47 107 235 171; do
  TQ_DEBUG=$f TRACE_TAG=_f$f python tools/gpu_trace.py c2 1 64 > gpurun_out/tr_f$f.log 2>&1
done
