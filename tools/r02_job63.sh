mkdir -p gpurun_out
J=j63
timeout 600 python tools/vcycle_sizes.py > gpurun_out/${J}_sizes.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --print-units base --csv python tools/vcycle_once.py config1 > gpurun_out/${J}_c1.csv 2>&1
