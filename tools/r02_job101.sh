mkdir -p gpurun_out
J=j101
timeout 900 ncu --set full --import-source on --clock-control none -k regex:prolong2 -s 16 -c 1 -o gpurun_out/${J}_prolong python tools/vcycle_once.py > gpurun_out/${J}_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:restrict3 -s 8 -c 1 -o gpurun_out/${J}_restrict python tools/vcycle_once.py >> gpurun_out/${J}_ncu.log 2>&1
