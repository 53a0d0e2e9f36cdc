#!/bin/bash
# per-role wait profile of the expert GEMM (TQ_PROFILE build), one file per batch size
export TQ_LIB_PATH=$PWD/paper_2605_09281_b200/libtileq_b200_tq_profile.so
for B in ${BS:-1 64}; do
  TQ_DEBUG=8 TRACE_TAG=_prof python tools/gpu_trace.py c2 $B > /dev/null 2>&1
done
