mkdir -p gpurun_out
J=j123
timeout 1800 python -m pytest tests/test_gpu_black.py tests/test_gpu_golden.py tests/test_gpu_parity.py tests/test_gpu_hybrid.py tests/test_gpu_legk.py -m gpu -x -q -p no:cacheprovider > gpurun_out/${J}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${J}_pytest.log
for v in 0 1 0 1; do
  echo "== black64 $v" >> gpurun_out/${J}.log
  TMG_PROLONG_BLACK64=$v timeout 300 python tools/legk_time.py >> gpurun_out/${J}.log 2>&1
done
