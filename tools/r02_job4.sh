mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:leg_sweep -s 2 -c 1 -o gpurun_out/j4_legk python tools/legk_once.py > gpurun_out/j4_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/j4_ncu.log
