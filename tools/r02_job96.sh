mkdir -p gpurun_out
TMG_LIB_PATH=paper_2110_08389_b200/libtmg_b200_mtime.so timeout 300 python tools/mini_once.py config1 > gpurun_out/j96.log 2>&1
TMG_LIB_PATH=paper_2110_08389_b200/libtmg_b200_mtime.so timeout 300 python tools/mini_once.py config2 >> gpurun_out/j96.log 2>&1
