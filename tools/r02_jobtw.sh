mkdir -p gpurun_out
O=gpurun_out/jtw.log; VARS=${VARS:-main tw0 main tw0}
timeout 900 python -m pytest tests/test_gpu_legk.py tests/test_gpu_golden.py -q -x -p no:cacheprovider > gpurun_out/jtw_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/jtw_pytest.log
for v in $VARS; do
  if [ $v = main ]; then L=paper_2110_08389_b200/libtmg_b200.so; else L=paper_2110_08389_b200/libtmg_b200_$v.so; fi
  echo "== $v" >> $O
  TMG_LIB_PATH=$L timeout 300 python tools/legk_time.py >> $O 2>&1
done
