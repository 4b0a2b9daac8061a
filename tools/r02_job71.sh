mkdir -p gpurun_out
J=j71
TMG_TAIL=0 timeout 300 python tools/tail_ab.py > gpurun_out/${J}_off.log 2>&1; echo "rc=$?" >> gpurun_out/${J}_off.log
for n in 8 128 1024; do
TMG_TAIL=0 TMG_LIB_PATH=paper_2110_08389_b200/libtmg_b200_tailp.so timeout 300 python tools/tail_phases.py $n >> gpurun_out/${J}_ph.log 2>&1
done
timeout 300 python tools/vcycle_sizes.py 8 32 128 256 1024 2048 > gpurun_out/${J}_sizes.log 2>&1
TMG_TAIL=1 timeout 300 python tools/vcycle_sizes.py 8 32 128 256 1024 2048 > gpurun_out/${J}_sizes_tail.log 2>&1
