mkdir -p gpurun_out
timeout 600 python tools/dbg_black.py > gpurun_out/j118.log 2>&1
