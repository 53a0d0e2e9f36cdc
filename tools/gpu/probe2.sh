# first run of the decode path: bounded-wait build first, then production
export TQ_LIB_PATH=$PWD/paper_2605_09281_b200/libtileq_b200_tq_wait_trap.so
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/p2_smoke_trap.log 2>&1; echo "smoke trap rc=$?"
tail -5 gpurun_out/p2_smoke_trap.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "forward_matches or paths_match or underflow" > gpurun_out/p2_par_trap.log 2>&1; echo "parity trap rc=$?"
tail -15 gpurun_out/p2_par_trap.log
unset TQ_LIB_PATH
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/p2_gputest.log 2>&1; echo "gpu tests rc=$?"
tail -15 gpurun_out/p2_gputest.log
