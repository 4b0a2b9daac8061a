mkdir -p gpurun_out
J=j65
for n in 8 128; do
TMG_LIB_PATH=paper_2110_08389_b200/libtmg_b200_tailt.so timeout 300 python tools/tail_times.py $n > gpurun_out/${J}_t$n.log 2>&1
done
for c in 1 2 4 8 16 32; do
echo "ctas $c" >> gpurun_out/${J}_ctas.log
TMG_TAIL_CTAS=$c timeout 300 python tools/vcycle_sizes.py 8 128 1024 >> gpurun_out/${J}_ctas.log 2>&1
done
