mkdir -p gpurun_out
J=j88
for v in 0 1 0 1; do
  echo "== walign $v" >> gpurun_out/${J}_ab.log
  TMG_LEGK_WALIGN=$v timeout 300 python tools/legk_time.py >> gpurun_out/${J}_ab.log 2>&1
done
echo "== pytest legk" >> gpurun_out/${J}_ab.log
timeout 900 python -m pytest tests/test_gpu_legk.py -m gpu -x -q -p no:cacheprovider >> gpurun_out/${J}_ab.log 2>&1
