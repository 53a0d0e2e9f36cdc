for f in 0 1 2 4 8 9 15; do
  if [ $f = 0 ]; then unset TQ_LIB_PATH; else export TQ_LIB_PATH=$PWD/paper_2605_09281_b200/libtileq_b200_tq_dec_abl=$f.so; fi
  timeout 120 python tools/gpu_gemm_time.py c2 1 8 64 2>&1 | sed "s/^/abl=$f /" | grep gemm
done > gpurun_out/p4_abl.log 2>&1
unset TQ_LIB_PATH
cat gpurun_out/p4_abl.log
timeout 300 python tools/prof_sweep.py c2 1 64 > gpurun_out/p4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"dec_" -c 6 -o gpurun_out/p4_dec python tools/prof_sweep.py c2 1 64 > gpurun_out/p4_ncu.log 2>&1; echo "ncu rc=$?"
