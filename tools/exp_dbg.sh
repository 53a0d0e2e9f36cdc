#!/bin/bash
# expert-GEMM time under TQ_DEBUG skip flags (1 no dequant, 2 no MMA, 32 no X, 64 no STTM, 128 no code copies)
for f in 0 227 3 35; do
  TQ_DEBUG=$f python tools/gpu_gemm_time.py c2 1 64 2>&1 | grep gemm
done
