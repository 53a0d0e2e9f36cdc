python -c "import __graft_entry__" 
timeout 600 python tools/gpu_gate_diag.py c1 folded 700 30 2>&1 | tail -12
timeout 600 python tools/gpu_gate_diag.py c1 general 700 10 2>&1 | tail -6
timeout 600 python tools/gpu_gate_diag.py c1 folded 300 10 2>&1 | tail -6
timeout 600 python tools/gpu_gate_diag.py c2 folded 700 5 2>&1 | tail -6
