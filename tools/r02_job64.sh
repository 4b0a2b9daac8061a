mkdir -p gpurun_out
J=j64
TMG_TAIL=0 timeout 300 python tools/tail_ab.py > gpurun_out/${J}_off.log 2>&1; echo "rc=$?" >> gpurun_out/${J}_off.log
timeout 300 python tools/tail_ab.py > gpurun_out/${J}_on.log 2>&1; echo "rc=$?" >> gpurun_out/${J}_on.log
timeout 300 python tools/vcycle_sizes.py 8 32 128 256 1024 2048 > gpurun_out/${J}_sizes.log 2>&1
