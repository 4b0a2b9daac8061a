mkdir -p gpurun_out
timeout 300 python tests/legk_worker.py default > gpurun_out/j5_default.log 2>&1; echo "rc=$?" >> gpurun_out/j5_default.log
TMG_LEGK_NMIN=16 TMG_LEGK_K0=3 timeout 300 python tests/legk_worker.py small > gpurun_out/j5_small.log 2>&1; echo "rc=$?" >> gpurun_out/j5_small.log
TMG_LEGK_NMIN=16 TMG_LEGK_K0=9 timeout 300 python tests/legk_worker.py small > gpurun_out/j5_small9.log 2>&1; echo "rc=$?" >> gpurun_out/j5_small9.log
timeout 300 python tests/legk_worker.py split > gpurun_out/j5_split.log 2>&1; echo "rc=$?" >> gpurun_out/j5_split.log
timeout 300 python tools/legk_time.py > gpurun_out/j5_time1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:leg_sweep -s 2 -c 1 -o gpurun_out/j5_legk python tools/legk_once.py > gpurun_out/j5_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/j5_ncu.log
