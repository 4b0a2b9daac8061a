mkdir -p gpurun_out
TMG_LIB_PATH=paper_2110_08389_b200/libtmg_b200_mtime.so timeout 300 python tools/mini_once.py config1 2>&1 | head -120 > gpurun_out/j98.log
