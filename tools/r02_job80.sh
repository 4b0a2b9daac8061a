mkdir -p gpurun_out
TMG_LIB_PATH=paper_2110_08389_b200/libtmg_b200_timing.so TMG_LEGK_TIMING=1 timeout 300 python tools/legk_phases.py > gpurun_out/j80_phases.log 2>&1
timeout 300 python tools/legk_time.py >> gpurun_out/j80_phases.log 2>&1
