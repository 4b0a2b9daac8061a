mkdir -p gpurun_out
J=j81
for v in main l2pf stag l2pfstag main l2pf; do
  if [ $v = main ]; then L=paper_2110_08389_b200/libtmg_b200.so; else L=paper_2110_08389_b200/libtmg_b200_$v.so; fi
  echo "== $v" >> gpurun_out/${J}_ab.log
  TMG_LIB_PATH=$L timeout 300 python tools/legk_time.py >> gpurun_out/${J}_ab.log 2>&1
done
echo "== timing main" >> gpurun_out/${J}_ab.log
TMG_LIB_PATH=paper_2110_08389_b200/libtmg_b200_timing.so TMG_LEGK_TIMING=1 timeout 300 python tools/legk_phases.py >> gpurun_out/${J}_ab.log 2>&1
echo "== timing l2pf" >> gpurun_out/${J}_ab.log
TMG_LIB_PATH=paper_2110_08389_b200/libtmg_b200_tl2pf.so TMG_LEGK_TIMING=1 timeout 300 python tools/legk_phases.py >> gpurun_out/${J}_ab.log 2>&1
