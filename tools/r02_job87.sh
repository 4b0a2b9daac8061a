mkdir -p gpurun_out
J=j87
for v in nobpf main nobpf main; do
  if [ $v = main ]; then L=paper_2110_08389_b200/libtmg_b200.so; else L=paper_2110_08389_b200/libtmg_b200_$v.so; fi
  echo "== $v" >> gpurun_out/${J}_ab.log
  TMG_LIB_PATH=$L timeout 300 python tools/legk_time.py >> gpurun_out/${J}_ab.log 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:leg_sweep -s 2 -c 2 -o gpurun_out/${J}_legk python tools/legk_once.py > gpurun_out/${J}_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/${J}_ncu.log
