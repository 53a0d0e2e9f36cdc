timeout 300 python tools/prof_sweep.py c2 1 8 64 > gpurun_out/p40_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_launches_decode.csv python tools/prof_sweep.py c2 1 8 64 > gpurun_out/p40_ncu1.log 2>&1; echo "launches rc=$?"
timeout 300 python tools/prof_sweep.py c2 4096 > gpurun_out/p40_plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_launches_prefill.csv python tools/prof_sweep.py c2 4096 > gpurun_out/p40_ncu2.log 2>&1; echo "launches prefill rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"dec_gemm|dec_route" -c 6 -o gpurun_out/r02_dec python tools/prof_sweep.py c2 1 8 64 > gpurun_out/p40_ncu3.log 2>&1; echo "full decode rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel" -s 1 -c 1 -o gpurun_out/r02_pre python tools/prof_sweep.py c2 4096 > gpurun_out/p40_ncu4.log 2>&1; echo "full prefill rc=$?"
