#!/bin/bash
# expert-GEMM time of compile-time ablation builds (TQ_DBG_CONST=<flags>; see exp_dbg.sh for the bits)
BS=${BS:-1 8 64}
python tools/gpu_gemm_time.py c2 $BS 2>&1 | grep gemm | sed "s/^/prod /"
for f in ${FLAGS:-128 195 3 1 2 64}; do
  TQ_LIB_PATH=$PWD/paper_2605_09281_b200/libtileq_b200_tq_dbg_const=$f.so python tools/gpu_gemm_time.py c2 $BS 2>&1 | grep gemm | sed "s/^/const=$f /"
done
