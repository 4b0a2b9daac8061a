mkdir -p gpurun_out
J=j103
timeout 1500 python -m pytest tests/test_gpu_transfers.py tests/test_gpu_hybrid.py tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_tail.py -m gpu -x -q -p no:cacheprovider > gpurun_out/${J}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${J}_pytest.log
for v in pslow main pslow main; do
  if [ $v = main ]; then L=paper_2110_08389_b200/libtmg_b200.so; else L=paper_2110_08389_b200/libtmg_b200_$v.so; fi
  echo "== $v" >> gpurun_out/${J}_ab.log
  TMG_LIB_PATH=$L timeout 300 python tools/legk_time.py >> gpurun_out/${J}_ab.log 2>&1
  TMG_LIB_PATH=$L timeout 300 python tools/transfer_time.py >> gpurun_out/${J}_ab.log 2>&1
done
