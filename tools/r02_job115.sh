mkdir -p gpurun_out
J=j115
for v in noserp main noserp main; do
  if [ $v = main ]; then L=paper_2110_08389_b200/libtmg_b200.so; else L=paper_2110_08389_b200/libtmg_b200_$v.so; fi
  echo "== $v" >> gpurun_out/${J}.log
  TMG_LIB_PATH=$L timeout 300 python tools/legk_time.py >> gpurun_out/${J}.log 2>&1
done
echo "== pytest legk" >> gpurun_out/${J}.log
timeout 900 python -m pytest tests/test_gpu_legk.py tests/test_gpu_golden.py -m gpu -x -q -p no:cacheprovider >> gpurun_out/${J}.log 2>&1
