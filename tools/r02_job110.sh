mkdir -p gpurun_out
J=j110
timeout 900 ncu --set full --import-source on --clock-control none -k regex:prolong2 -s 15 -c 1 -o gpurun_out/${J}_prolong python tools/vcycle_once.py > gpurun_out/${J}_ncu.log 2>&1
timeout 300 python tools/transfer_time.py > gpurun_out/${J}_transfer_time.log 2>&1
