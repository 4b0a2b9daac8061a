mkdir -p gpurun_out
J=j82
for v in ns main l2pfns l2pf ns l2pf; do
  if [ $v = main ]; then L=paper_2110_08389_b200/libtmg_b200.so; else L=paper_2110_08389_b200/libtmg_b200_$v.so; fi
  echo "== $v" >> gpurun_out/${J}_ab.log
  TMG_LIB_PATH=$L timeout 300 python tools/legk_time.py >> gpurun_out/${J}_ab.log 2>&1
done
echo "== timing l2pf" >> gpurun_out/${J}_ab.log
TMG_LIB_PATH=paper_2110_08389_b200/libtmg_b200_tl2pf.so TMG_LEGK_TIMING=1 timeout 300 python tools/legk_phases.py >> gpurun_out/${J}_ab.log 2>&1
echo "== pytest legk (l2pf lib)" >> gpurun_out/${J}_ab.log
TMG_LIB_PATH=paper_2110_08389_b200/libtmg_b200_l2pf.so timeout 900 python -m pytest tests/test_gpu_legk.py tests/test_gpu_golden.py -m gpu -x -q -p no:cacheprovider >> gpurun_out/${J}_ab.log 2>&1
