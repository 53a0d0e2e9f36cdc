#!/bin/bash
# expert-GEMM time: production build, then the experiment build under TQ_DEBUG skip flags
# (1 no dequant, 2 no MMA, 4 no stores, 32 no X, 64 no STTM, 128 no code copies)
BS=${BS:-1 8 64}
python tools/gpu_gemm_time.py c2 $BS 2>&1 | grep gemm | sed "s/^/prod /"
export TQ_LIB_PATH=$PWD/paper_2605_09281_b200/libtileq_b200_tq_experiment.so
for f in ${FLAGS:-227 3 35}; do
  TQ_DEBUG=$f python tools/gpu_gemm_time.py c2 $BS 2>&1 | grep gemm | sed "s/^/exp /"
done
