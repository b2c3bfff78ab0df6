for cfg in c3 c4; do timeout 300 python tools/jit_sweep.py $cfg 100000 -1 2>&1 | sed "s/^/interp /"; done > gpurun_out/sweep.log
