for f in 0 1 2 4 8 9 6 15; do
  if [ $f = 0 ]; then unset TQ_LIB_PATH; else export TQ_LIB_PATH=$PWD/paper_2605_09281_b200/libtileq_b200_tq_dec_abl=$f.so; fi
  timeout 120 python tools/gpu_gemm_time.py c2 1 8 64 2>&1 | sed "s/^/abl=$f /" | grep gemm
done
