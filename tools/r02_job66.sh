mkdir -p gpurun_out
J=j67
for n in 8 16 128 1024; do
TMG_LIB_PATH=paper_2110_08389_b200/libtmg_b200_tailp.so timeout 300 python tools/tail_phases.py $n >> gpurun_out/${J}.log 2>&1
TMG_TAIL=0 TMG_LIB_PATH=paper_2110_08389_b200/libtmg_b200_tailp.so timeout 300 python tools/tail_phases.py $n >> gpurun_out/${J}.log 2>&1
done
