mkdir -p gpurun_out
J=j83
timeout 300 python tools/legk_time.py > gpurun_out/${J}_time.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:leg_sweep -s 2 -c 2 -o gpurun_out/${J}_legk python tools/legk_once.py > gpurun_out/${J}_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/${J}_ncu.log
