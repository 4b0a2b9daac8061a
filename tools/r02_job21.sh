mkdir -p gpurun_out
export TMG_LIB_PATH=paper_2110_08389_b200/libtmg_b200_R.so
timeout 300 python tests/legk_worker.py default > gpurun_out/j21_default.log 2>&1; echo "rc=$?" >> gpurun_out/j21_default.log
TMG_LEGK_NMIN=16 TMG_LEGK_K0=3 timeout 300 python tests/legk_worker.py small > gpurun_out/j21_small.log 2>&1; echo "rc=$?" >> gpurun_out/j21_small.log
timeout 300 python tests/legk_worker.py split > gpurun_out/j21_split.log 2>&1; echo "rc=$?" >> gpurun_out/j21_split.log
unset TMG_LIB_PATH
J=j21 bash tools/r02_ab.sh H R H R
