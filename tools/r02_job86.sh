mkdir -p gpurun_out
J=j86
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${J}_launches.csv python tools/vcycle_once.py > gpurun_out/${J}_ncu.log 2>&1
