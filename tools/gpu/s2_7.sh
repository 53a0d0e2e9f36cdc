cd tools/micro; for f in mma_tput mma_acc tmem_contend dq_rate; do echo "== $f"; timeout 60 ./$f 2>&1 | tail -24; done; cd ../..
for a in 0 2 4 6; do
  if [ $a = 0 ]; then unset TQ_LIB_PATH; else export TQ_LIB_PATH=$PWD/paper_2605_09281_b200/libtileq_b200_tq_dec_abl=$a.so; fi
  timeout 120 python tools/gpu_gemm_time.py c2 1 2 8 32 64 2>&1 | grep gemm | sed "s/^/ABL=$a /"
done
timeout 300 ./integration/_build/test_gpu_shim 2>&1 | tail -30
