mkdir -p gpurun_out
J=${J:-j10}
timeout 300 python tests/legk_worker.py default > gpurun_out/${J}_default.log 2>&1; echo "rc=$?" >> gpurun_out/${J}_default.log
TMG_LEGK_NMIN=16 TMG_LEGK_K0=3 timeout 300 python tests/legk_worker.py small > gpurun_out/${J}_small.log 2>&1; echo "rc=$?" >> gpurun_out/${J}_small.log
TMG_LEGK_NMIN=16 TMG_LEGK_K0=9 timeout 300 python tests/legk_worker.py small > gpurun_out/${J}_small9.log 2>&1; echo "rc=$?" >> gpurun_out/${J}_small9.log
timeout 300 python tests/legk_worker.py split > gpurun_out/${J}_split.log 2>&1; echo "rc=$?" >> gpurun_out/${J}_split.log
timeout 300 python tools/legk_time.py > gpurun_out/${J}_time1.log 2>&1
TMG_LIB_PATH=paper_2110_08389_b200/libtmg_b200_timing.so TMG_LEGK_TIMING=1 timeout 300 python tools/legk_phases.py > gpurun_out/${J}_phases.log 2>&1
if [ -n "$NCU" ]; then timeout 600 ncu --set full --import-source on --clock-control none -k regex:leg_sweep -s 2 -c 1 -o gpurun_out/${J}_legk python tools/legk_once.py > gpurun_out/${J}_ncu.log 2>&1; fi
