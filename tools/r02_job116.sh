mkdir -p gpurun_out
J=j116
for v in 0 1 0 1; do
  echo "== serp $v" >> gpurun_out/${J}.log
  TMG_LEGK_SERP=$v timeout 300 python tools/legk_time.py >> gpurun_out/${J}.log 2>&1
done
echo "== pytest legk" >> gpurun_out/${J}.log
timeout 900 python -m pytest tests/test_gpu_legk.py tests/test_gpu_golden.py -m gpu -x -q -p no:cacheprovider >> gpurun_out/${J}.log 2>&1
