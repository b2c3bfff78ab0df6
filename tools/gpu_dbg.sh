timeout 300 python tools/sweep_heavy.py c3 16 > gpurun_out/sweep.log 2>&1
timeout 300 python tools/jit_runs.py c4 0 | tail -2 >> gpurun_out/sweep.log 2>&1
timeout 300 python tools/e2e_sweep.py c3 >> gpurun_out/sweep.log 2>&1
