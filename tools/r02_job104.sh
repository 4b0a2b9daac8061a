mkdir -p gpurun_out
J=j104
for v in main pb6 pb8 main pb6 pb8; do
  if [ $v = main ]; then L=paper_2110_08389_b200/libtmg_b200.so; else L=paper_2110_08389_b200/libtmg_b200_$v.so; fi
  echo "== $v" >> gpurun_out/${J}_ab.log
  TMG_LIB_PATH=$L timeout 300 python tools/transfer_time.py >> gpurun_out/${J}_ab.log 2>&1
done
