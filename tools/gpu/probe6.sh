timeout 60 ./tools/micro/pipe2 > gpurun_out/p6_pipe2.log 2>&1; echo rc=$?
timeout 60 ./tools/micro/pipe_empty > gpurun_out/p6_pipe_empty.log 2>&1; echo rc=$?
cat gpurun_out/p6_pipe2.log gpurun_out/p6_pipe_empty.log
